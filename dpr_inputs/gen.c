/*
 * dpr_inputs/gen.c -- seeded, deterministic SYNTHETIC INPUT generators shared by the
 * oracle tests and the CUDA product path.  Holds none of the method's arithmetic
 * (no ray tracing, routing or shading): only scene geometry and volume fields shaped
 * like the paper's workloads (SURVEY 8(d) "Concrete synthetic inputs").
 *
 *   dpri_gyroid_mt: gyroid iso-surface sin(kx)cos(ky)+sin(ky)cos(kz)+sin(kz)cos(kx)=0 on
 *     [-1,1]^3 extracted by marching tetrahedra (Kuhn 6-tet split of each grid cell),
 *     vertices by linear interpolation on cut edges -- the "~10M-triangle mesh" of
 *     BASELINE configs[1] (an iso-surface like the paper's DNS / Mars-lander meshes,
 *     P:1260-1286).  Indexed mesh (one shared vertex per cut grid edge), float32;
 *     exact-zero-area triangles are dropped.
 *   dpri_volume_field: the procedural 1024^3-class scalar field of config 3
 *     (a stand-in for the paper's thunderstorm / DNS volumes).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

static double gyroid(double x, double y, double z, double k)
{
    return sin(k * x) * cos(k * y) + sin(k * y) * cos(k * z) + sin(k * z) * cos(k * x);
}

/* Kuhn decomposition: 6 tets along the main diagonal 0-7 of the cube.  Corner c has
 * offset (c&1, (c>>1)&1, (c>>2)&1). */
static const int TETS[6][4] = {
    {0, 1, 3, 7}, {0, 3, 2, 7}, {0, 2, 6, 7}, {0, 6, 4, 7}, {0, 4, 5, 7}, {0, 5, 1, 7}};

/* Indexed mesh: one vertex per cut grid edge, shared by every tet using that edge.  In
 * the Kuhn split every tet edge joins a corner to a corner whose offset bits are a superset,
 * so each edge is (low grid point p, direction d in 1..7; offset bits x=1, y=2, z=4) and its
 * vertex is interpolated from low to high endpoint: bit-identical wherever it is used.
 * Vertex numbering: z-plane of the low point, then (y, x, d) -- independent of threads. */
typedef struct {
    int G;
    double k;
    int z0, z1;            /* cube-z range [z0, z1); vertex planes owned: [z0, z1) (+G-1 if last) */
    int last;
    int64_t *plane_cnt;    /* count pass: cut edges per owned plane */
    const int64_t *plane_off;
    float *verts;          /* NULL = count only */
    int32_t *idx;
    int64_t tri_off;
    int64_t n;             /* triangles produced */
} MTJob;

static int is_cut(double fa, double fb) { return (fa > 0.0) != (fb > 0.0); }

static void edge_point(int G, double h, int x, int y, int z, int d, double fa, double fb, float out[3])
{
    (void)G;
    const double pa[3] = {-1 + x * h, -1 + y * h, -1 + z * h};
    const double pb[3] = {-1 + (x + (d & 1)) * h, -1 + (y + ((d >> 1) & 1)) * h, -1 + (z + ((d >> 2) & 1)) * h};
    double w = fa / (fa - fb);
    for (int c = 0; c < 3; ++c) out[c] = (float)(pa[c] + w * (pb[c] - pa[c]));
}

static void fill_plane(double *pl, int G, double h, int z, double k)
{
    for (int y = 0; y < G; ++y)
        for (int x = 0; x < G; ++x) pl[y * G + x] = gyroid(-1 + x * h, -1 + y * h, -1 + z * h, k);
}

/* Cut edges whose low point lies in plane q (fq1 = plane q+1, NULL for the top plane).
 * map (optional): vertex id per (y, x, d-1), -1 if not cut; verts (optional): positions. */
static int64_t plane_edges(int G, double h, int q, const double *fq, const double *fq1, int32_t *map,
                           int64_t base, float *verts)
{
    int64_t k = 0;
    for (int y = 0; y < G; ++y)
        for (int x = 0; x < G; ++x)
            for (int d = 1; d < 8; ++d) {
                int dx = d & 1, dy = (d >> 1) & 1, dz = (d >> 2) & 1;
                int32_t id = -1;
                if (x + dx < G && y + dy < G && (!dz || fq1)) {
                    double fa = fq[y * G + x], fb = (dz ? fq1 : fq)[(y + dy) * G + x + dx];
                    if (is_cut(fa, fb)) {
                        id = (int32_t)(base + k);
                        if (verts) edge_point(G, h, x, y, q, d, fa, fb, verts + 3 * (base + k));
                        ++k;
                    }
                }
                if (map) map[(y * G + x) * 7 + d - 1] = id;
            }
    return k;
}

static int tri_nonzero(const float a[3], const float b[3], const float c[3])
{
    /* exact-zero-area triangles (f32 cross product == 0) are dropped */
    float e1[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
    float e2[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
    float nx = e1[1] * e2[2] - e1[2] * e2[1];
    float ny = e1[2] * e2[0] - e1[0] * e2[2];
    float nz = e1[0] * e2[1] - e1[1] * e2[0];
    return !(nx == 0.0f && ny == 0.0f && nz == 0.0f);
}

static void *mt_worker(void *arg)
{
    MTJob *J = (MTJob *)arg;
    const int G = J->G;
    const double h = 2.0 / (double)(G - 1);
    const size_t P = (size_t)G * G;
    double *f0 = (double *)malloc(sizeof(double) * P), *f1 = (double *)malloc(sizeof(double) * P),
           *f2 = (double *)malloc(sizeof(double) * P);
    int32_t *m0 = NULL, *m1 = NULL;
    const int emit = J->verts != NULL;
    if (emit) { m0 = (int32_t *)malloc(sizeof(int32_t) * P * 7); m1 = (int32_t *)malloc(sizeof(int32_t) * P * 7); }
    fill_plane(f0, G, h, J->z0, J->k);
    fill_plane(f1, G, h, J->z0 + 1, J->k);
    if (emit)
        plane_edges(G, h, J->z0, f0, f1, m0, J->plane_off[J->z0], J->verts);
    else
        J->plane_cnt[J->z0] = plane_edges(G, h, J->z0, f0, f1, NULL, 0, NULL);
    for (int z = J->z0; z < J->z1; ++z) {
        /* plane z+1 (low points of the top-face edges of the cubes at z) */
        const int q = z + 1;
        const double *fq2 = NULL;
        if (q + 1 < G) { fill_plane(f2, G, h, q + 1, J->k); fq2 = f2; }
        const int owned = q < J->z1 || (J->last && q == G - 1);
        if (emit)
            plane_edges(G, h, q, f1, fq2, m1, J->plane_off[q], owned ? J->verts : NULL);
        else if (owned)
            J->plane_cnt[q] = plane_edges(G, h, q, f1, fq2, NULL, 0, NULL);
        for (int y = 0; y + 1 < G; ++y) {
            for (int x = 0; x + 1 < G; ++x) {
                double f[8];
                for (int c = 0; c < 8; ++c)
                    f[c] = ((c >> 2) ? f1 : f0)[(y + ((c >> 1) & 1)) * G + (x + (c & 1))];
                for (int t = 0; t < 6; ++t) {
                    const int *v = TETS[t];
                    int in[4], nin = 0;
                    for (int i = 0; i < 4; ++i) { in[i] = f[v[i]] > 0.0; nin += in[i]; }
                    if (nin == 0 || nin == 4) continue;
                    /* the cut edges of the tet, as corner pairs, in the emission order */
                    int ea[4][2], ne;
                    if (nin == 1 || nin == 3) {
                        int want = nin == 1 ? 1 : 0, a = 0, m = 0;
                        for (int i = 0; i < 4; ++i) if (in[i] == want) a = i;
                        for (int i = 0; i < 4; ++i) if (i != a) { ea[m][0] = v[a]; ea[m][1] = v[i]; ++m; }
                        ne = 3;
                    } else {
                        int ins[2], outs[2], ni = 0, no = 0;
                        for (int i = 0; i < 4; ++i) { if (in[i]) ins[ni++] = v[i]; else outs[no++] = v[i]; }
                        ea[0][0] = ins[0]; ea[0][1] = outs[0];
                        ea[1][0] = ins[0]; ea[1][1] = outs[1];
                        ea[2][0] = ins[1]; ea[2][1] = outs[1];
                        ea[3][0] = ins[1]; ea[3][1] = outs[0];
                        ne = 4;
                    }
                    float qp[4][3];
                    int32_t qi[4];
                    for (int e = 0; e < ne; ++e) {
                        int ca = ea[e][0], cb = ea[e][1];
                        int lo = (ca & cb) == ca ? ca : cb, hi = lo == ca ? cb : ca;
                        int d = hi ^ lo;
                        int lx = x + (lo & 1), ly = y + ((lo >> 1) & 1), lz = (lo >> 2) & 1;
                        edge_point(G, h, lx, ly, z + lz, d, f[lo], f[hi], qp[e]);
                        if (emit) qi[e] = (lz ? m1 : m0)[((size_t)ly * G + lx) * 7 + d - 1];
                    }
                    const int tris[2][3] = {{0, 1, 2}, {0, 2, 3}};
                    for (int tt = 0; tt < (ne == 3 ? 1 : 2); ++tt) {
                        const int *c = tris[tt];
                        if (!tri_nonzero(qp[c[0]], qp[c[1]], qp[c[2]])) continue;
                        if (emit) {
                            int32_t *o = J->idx + 3 * (J->tri_off + J->n);
                            o[0] = qi[c[0]]; o[1] = qi[c[1]]; o[2] = qi[c[2]];
                        }
                        J->n++;
                    }
                }
            }
        }
        double *t = f0; f0 = f1; f1 = f2; f2 = t;
        if (emit) { int32_t *tm = m0; m0 = m1; m1 = tm; }
    }
    free(f0); free(f1); free(f2); free(m0); free(m1);
    return NULL;
}

/* Indexed gyroid mesh.  Call with verts == NULL to count (*nv_out, return = triangles),
 * then with buffers of the counted sizes (verts: 3 floats per vertex, idx: 3 int32 per
 * triangle).  Returns the number of triangles, or -1 on error. */
EXPORT int64_t dpri_gyroid_mt(int G, double k, float *verts, int32_t *idx, int64_t nv_cap, int64_t nt_cap,
                              int nthreads, int64_t *nv_out)
{
    if (G < 2) return -1;
    if (nthreads < 1) nthreads = 1;
    int nz = G - 1;
    if (nthreads > nz) nthreads = nz;
    MTJob *jobs = (MTJob *)calloc((size_t)nthreads, sizeof(MTJob));
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    int64_t *cnt = (int64_t *)calloc((size_t)G, sizeof(int64_t)), *off = (int64_t *)calloc((size_t)G + 1, sizeof(int64_t));
    /* pass 1: cut edges per plane and triangles per thread */
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].G = G; jobs[t].k = k;
        jobs[t].z0 = (int)((int64_t)nz * t / nthreads);
        jobs[t].z1 = (int)((int64_t)nz * (t + 1) / nthreads);
        jobs[t].last = t == nthreads - 1;
        jobs[t].plane_cnt = cnt;
        pthread_create(&th[t], NULL, mt_worker, &jobs[t]);
    }
    int64_t total = 0;
    for (int t = 0; t < nthreads; ++t) { pthread_join(th[t], NULL); total += jobs[t].n; }
    for (int z = 0; z < G; ++z) off[z + 1] = off[z] + cnt[z];
    if (nv_out) *nv_out = off[G];
    int rc = 0;
    if (verts) {
        if (nv_cap < off[G] || nt_cap < total || !idx || off[G] > INT32_MAX) rc = -1;
        else {
            int64_t toff = 0;
            for (int t = 0; t < nthreads; ++t) {
                int64_t c = jobs[t].n;
                jobs[t].verts = verts; jobs[t].idx = idx; jobs[t].plane_off = off;
                jobs[t].tri_off = toff; jobs[t].n = 0;
                toff += c;
                pthread_create(&th[t], NULL, mt_worker, &jobs[t]);
            }
            for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
        }
    }
    free(jobs); free(th); free(cnt); free(off);
    return rc ? -1 : total;
}

/* Procedural field on a G^3 grid over [-1,1]^3 (x fastest), computed in double, stored
 * f32:  f = clamp(1-|x|^2, 0, 1) * (0.5 + 0.25 sin9x sin7y sin8z
 *                                    + 0.25 sin(23x+1) sin(19y+2) sin(29z+3)).
 * Writes the sub-box [lo, hi] (inclusive) of the grid into out (x fastest). */
typedef struct { int G; int lo[3], hi[3]; int z0, z1; float *out; } VJob;

static void *vol_worker(void *arg)
{
    VJob *J = (VJob *)arg;
    const double h = 2.0 / (double)(J->G - 1);
    int nx = J->hi[0] - J->lo[0] + 1, ny = J->hi[1] - J->lo[1] + 1;
    double *ax = (double *)malloc(sizeof(double) * nx), *bx = (double *)malloc(sizeof(double) * nx);
    double *x2 = (double *)malloc(sizeof(double) * nx);
    for (int i = 0; i < nx; ++i) {
        double x = -1 + (J->lo[0] + i) * h;
        ax[i] = sin(9 * x); bx[i] = sin(23 * x + 1); x2[i] = x * x;
    }
    for (int z = J->z0; z < J->z1; ++z) {
        double zz = -1 + z * h;
        double cz = sin(8 * zz), dz = sin(29 * zz + 3);
        for (int j = 0; j < ny; ++j) {
            double y = -1 + (J->lo[1] + j) * h;
            double cy = sin(7 * y), dy = sin(19 * y + 2);
            float *row = J->out + ((int64_t)(z - J->lo[2]) * ny + j) * nx;
            for (int i = 0; i < nx; ++i) {
                double r = 1.0 - (x2[i] + y * y + zz * zz);
                if (r < 0) r = 0;
                if (r > 1) r = 1;
                row[i] = (float)(r * (0.5 + 0.25 * ax[i] * cy * cz + 0.25 * bx[i] * dy * dz));
            }
        }
    }
    free(ax); free(bx); free(x2);
    return NULL;
}

EXPORT int dpri_volume_field(int G, const int lo[3], const int hi[3], float *out, int nthreads)
{
    if (nthreads < 1) nthreads = 1;
    int nz = hi[2] - lo[2] + 1;
    if (nthreads > nz) nthreads = nz;
    VJob *jobs = (VJob *)calloc((size_t)nthreads, sizeof(VJob));
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].G = G;
        memcpy(jobs[t].lo, lo, sizeof(int) * 3);
        memcpy(jobs[t].hi, hi, sizeof(int) * 3);
        jobs[t].z0 = lo[2] + (int)((int64_t)nz * t / nthreads);
        jobs[t].z1 = lo[2] + (int)((int64_t)nz * (t + 1) / nthreads);
        jobs[t].out = out;
        pthread_create(&th[t], NULL, vol_worker, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(jobs); free(th);
    return 0;
}
