/* Compiled-C caller of the boundary (include/dpr.h): plain C99, no Python, no torch.
 *   abi_smoke host   -- host-only calls: the exchange planner, error reporting
 *   abi_smoke gpu    -- one rank on cuda:0 (NULL stream, NULL allocator): a ground quad lit
 *                       from above with AO rays that cannot be occluded renders the closed form
 *                       rho*(E*(n.l) + A) (SURVEY 8(c).4 P6 pin) at every covered pixel; the
 *                       frame descriptor is filled over garbage padding bytes (the digest /
 *                       copy are field-wise). */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "dpr.h"

#define CHECK(x)                                                                              \
    do {                                                                                      \
        int rc_ = (x);                                                                        \
        if (rc_ != DPR_OK) {                                                                  \
            fprintf(stderr, "%s:%d %s -> %d (%s)\n", __FILE__, __LINE__, #x, rc_, dpr_last_error(NULL)); \
            return 1;                                                                         \
        }                                                                                     \
    } while (0)

static int host_part(void) {
    /* 3 ranks, counts[src][dst]; rank 1's next input = [self 7 | from 0: 1 | from 2: 6] */
    const int64_t counts[9] = {5, 1, 2, 3, 7, 0, 4, 6, 9};
    int64_t off[3], tin = 0, gt = 0;
    CHECK(dpr_exchange_plan(3, 1, counts, 100, off, &tin, &gt));
    if (tin != 14 || gt != 37 || off[0] != 7 || off[2] != 8 || off[1] != 0) {
        fprintf(stderr, "exchange plan wrong: %lld %lld\n", (long long)tin, (long long)gt);
        return 1;
    }
    if (dpr_exchange_plan(3, 1, counts, 13, off, &tin, &gt) != DPR_ERR_QUEUE_OVERFLOW) return 1;
    if (dpr_exchange_plan(3, 7, counts, 100, off, &tin, &gt) != DPR_ERR_INVALID_ARG) return 1;
    if (strlen(dpr_last_error(NULL)) == 0) return 1;
    if (dpr_create_device(0, 1, 0, NULL, NULL, NULL, NULL) != DPR_ERR_INVALID_ARG) return 1;
    printf("host ok: sizeof(dpr_frame_desc)=%zu sizeof(dpr_stats)=%zu\n", sizeof(dpr_frame_desc), sizeof(dpr_stats));
    return 0;
}

static int gpu_part(void) {
    dpr_device dev = NULL;
    CHECK(dpr_create_device(0, 1, 0, NULL, NULL, NULL, &dev));
    /* ground quad y = 0, x,z in [-4, 4] (two triangles), albedo 0.8 */
    const float verts[12] = {-4, 0, -4, 4, 0, -4, 4, 0, 4, -4, 0, 4};
    const int32_t idx[6] = {0, 1, 2, 0, 2, 3};
    dpr_part_desc p;
    memset(&p, 0, sizeof(p));
    p.kind = DPR_PART_TRIANGLES;
    p.memory = DPR_MEMORY_HOST;
    p.albedo[0] = p.albedo[1] = p.albedo[2] = 0.8f;
    p.n_verts = 4; p.verts = verts; p.n_tris = 2; p.idx = idx;
    CHECK(dpr_commit_part(dev, &p));
    CHECK(dpr_commit_world(dev));
    float b[6];
    CHECK(dpr_get_world_bounds(dev, b));
    if (b[0] != -4.0f || b[4] != 0.0f || b[5] != 4.0f) { fprintf(stderr, "bounds\n"); return 1; }
    /* camera at (0, 3, 0.5) looking straight down (fovy 60 deg, square): every pixel sees the quad */
    const int W = 32, H = 32;
    const double h = tan(60.0 * M_PI / 360.0);
    const double w[3] = {0, -1, 0}, u[3] = {1, 0, 0}, v[3] = {0, 0, -1}; /* u = w x up(0,0,-1)... */
    dpr_camera_basis cam;
    memset(&cam, 0, sizeof(cam));
    cam.E[0] = 0.0f; cam.E[1] = 3.0f; cam.E[2] = 0.5f;
    for (int c = 0; c < 3; ++c) {
        cam.U[c] = (float)(2.0 * h * u[c]);
        cam.V[c] = (float)(2.0 * h * v[c]);
        cam.L[c] = (float)(w[c] - h * u[c] - h * v[c]);
    }
    CHECK(dpr_set_camera(dev, &cam));
    dpr_frame_desc f;
    memset(&f, 0xAB, sizeof(f)); /* garbage in the padding: fields are set one by one */
    f.W = W; f.H = H; f.spp = 2; f.spp_batch = 2; f.max_depth = 1; f.ao_k = 4; f.ao_radius = 0.5f;
    f.light_dir[0] = 0.0f; f.light_dir[1] = 1.0f; f.light_dir[2] = 0.0f;
    for (int c = 0; c < 3; ++c) { f.E[c] = 1.0f; f.A[c] = 0.25f; f.B[c] = 0.0f; }
    f.dt = 0.0f; f.seed = 7; f.flags = 0;
    CHECK(dpr_set_frame(dev, &f));
    CHECK(dpr_render_frame(dev));
    const float *rgba = NULL;
    int mw = 0, mh = 0, und = 1;
    CHECK(dpr_map_frame(dev, &rgba, &mw, &mh, &und));
    if (!rgba || mw != W || mh != H || und) { fprintf(stderr, "map_frame\n"); return 1; }
    float *host = (float *)malloc(sizeof(float) * 4 * W * H);
    if (cudaMemcpy(host, rgba, sizeof(float) * 4 * W * H, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
    /* closed form: 0.8 * (1 * n.l + 0.25) with n.l = 1 (the AO rays of a plane with nothing above
       it are never occluded: AO = 1 exactly) */
    const float want = 0.8f * (1.0f + 0.25f);
    double maxd = 0;
    for (int i = 0; i < W * H; ++i) {
        for (int c = 0; c < 3; ++c) maxd = fmax(maxd, fabs(host[4 * i + c] - want));
        if (host[4 * i + 3] != 1.0f) { fprintf(stderr, "coverage %d\n", i); return 1; }
    }
    dpr_stats st;
    CHECK(dpr_get_stats(dev, &st));
    CHECK(dpr_release_device(dev));
    free(host);
    if (maxd > 1e-6) { fprintf(stderr, "pixel off by %g\n", maxd); return 1; }
    printf("gpu ok: rays %lld/%lld/%lld steps %lld max|d| %.3g launches %lld\n", (long long)st.rays[0],
           (long long)st.rays[1], (long long)st.rays[2], (long long)st.steps, maxd, (long long)st.kernel_launches_local);
    return 0;
}

int main(int argc, char **argv) {
    if (argc > 1 && strcmp(argv[1], "gpu") == 0) return gpu_part();
    return host_part();
}
