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
 *     P:1260-1286).  Triangle soup, float32; exact-zero-area triangles are dropped.
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

typedef struct {
    int G;
    double k;
    int z0, z1;
    float *out;        /* triangles, 9 floats each; NULL = count only */
    int64_t n;         /* produced */
    int64_t cap;
} MTJob;

static void edge_point(const double pa[3], const double pb[3], double fa, double fb, float out[3])
{
    double w = fa / (fa - fb);
    for (int c = 0; c < 3; ++c) out[c] = (float)(pa[c] + w * (pb[c] - pa[c]));
}

static int emit(MTJob *J, const float a[3], const float b[3], const float c[3])
{
    /* drop exact-zero-area triangles (f32 cross product == 0) */
    float e1[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
    float e2[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
    float nx = e1[1] * e2[2] - e1[2] * e2[1];
    float ny = e1[2] * e2[0] - e1[0] * e2[2];
    float nz = e1[0] * e2[1] - e1[1] * e2[0];
    if (nx == 0.0f && ny == 0.0f && nz == 0.0f) return 0;
    if (J->out) {
        if (J->n >= J->cap) return -1;
        float *o = J->out + 9 * J->n;
        memcpy(o, a, 12); memcpy(o + 3, b, 12); memcpy(o + 6, c, 12);
    }
    J->n++;
    return 0;
}

static void *mt_worker(void *arg)
{
    MTJob *J = (MTJob *)arg;
    const int G = J->G;
    const double h = 2.0 / (double)(G - 1);
    double *plane0 = (double *)malloc(sizeof(double) * G * G);
    double *plane1 = (double *)malloc(sizeof(double) * G * G);
    for (int y = 0; y < G; ++y)
        for (int x = 0; x < G; ++x) plane0[y * G + x] = gyroid(-1 + x * h, -1 + y * h, -1 + J->z0 * h, J->k);
    for (int z = J->z0; z < J->z1; ++z) {
        for (int y = 0; y < G; ++y)
            for (int x = 0; x < G; ++x) plane1[y * G + x] = gyroid(-1 + x * h, -1 + y * h, -1 + (z + 1) * h, J->k);
        for (int y = 0; y + 1 < G; ++y) {
            for (int x = 0; x + 1 < G; ++x) {
                double f[8], p[8][3];
                for (int c = 0; c < 8; ++c) {
                    int dx = c & 1, dy = (c >> 1) & 1, dz = (c >> 2) & 1;
                    f[c] = (dz ? plane1 : plane0)[(y + dy) * G + (x + dx)];
                    p[c][0] = -1 + (x + dx) * h; p[c][1] = -1 + (y + dy) * h; p[c][2] = -1 + (z + dz) * h;
                }
                for (int t = 0; t < 6; ++t) {
                    const int *v = TETS[t];
                    int in[4], nin = 0;
                    for (int i = 0; i < 4; ++i) { in[i] = f[v[i]] > 0.0; nin += in[i]; }
                    if (nin == 0 || nin == 4) continue;
                    if (nin == 1 || nin == 3) {
                        int want = nin == 1 ? 1 : 0, a = 0;
                        for (int i = 0; i < 4; ++i) if (in[i] == want) a = i;
                        float q[3][3];
                        int m = 0;
                        for (int i = 0; i < 4; ++i) {
                            if (i == a) continue;
                            edge_point(p[v[a]], p[v[i]], f[v[a]], f[v[i]], q[m++]);
                        }
                        emit(J, q[0], q[1], q[2]);
                    } else {
                        int ins[2], outs[2], ni = 0, no = 0;
                        for (int i = 0; i < 4; ++i) { if (in[i]) ins[ni++] = i; else outs[no++] = i; }
                        float q[4][3];
                        edge_point(p[v[ins[0]]], p[v[outs[0]]], f[v[ins[0]]], f[v[outs[0]]], q[0]);
                        edge_point(p[v[ins[0]]], p[v[outs[1]]], f[v[ins[0]]], f[v[outs[1]]], q[1]);
                        edge_point(p[v[ins[1]]], p[v[outs[1]]], f[v[ins[1]]], f[v[outs[1]]], q[2]);
                        edge_point(p[v[ins[1]]], p[v[outs[0]]], f[v[ins[1]]], f[v[outs[0]]], q[3]);
                        emit(J, q[0], q[1], q[2]);
                        emit(J, q[0], q[2], q[3]);
                    }
                }
            }
        }
        double *t = plane0; plane0 = plane1; plane1 = t;
    }
    free(plane0); free(plane1);
    return NULL;
}

/* Two-pass: call with out == NULL to count, then with a buffer of the counted size.
 * Returns the number of triangles (9 floats each, soup), or -1 on error. */
EXPORT int64_t dpri_gyroid_mt(int G, double k, float *out, int64_t cap, int nthreads)
{
    if (G < 2) return -1;
    if (nthreads < 1) nthreads = 1;
    int nz = G - 1;
    if (nthreads > nz) nthreads = nz;
    MTJob *jobs = (MTJob *)calloc((size_t)nthreads, sizeof(MTJob));
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    /* pass 1: count per slab range (needed to place each thread's output) */
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].G = G; jobs[t].k = k;
        jobs[t].z0 = (int)((int64_t)nz * t / nthreads);
        jobs[t].z1 = (int)((int64_t)nz * (t + 1) / nthreads);
        jobs[t].out = NULL;
        pthread_create(&th[t], NULL, mt_worker, &jobs[t]);
    }
    int64_t total = 0;
    for (int t = 0; t < nthreads; ++t) { pthread_join(th[t], NULL); total += jobs[t].n; }
    if (out) {
        if (cap < total) { free(jobs); free(th); return -1; }
        int64_t off = 0;
        for (int t = 0; t < nthreads; ++t) {
            int64_t cnt = jobs[t].n;
            jobs[t].out = out + 9 * off;
            jobs[t].cap = cnt;
            jobs[t].n = 0;
            off += cnt;
            pthread_create(&th[t], NULL, mt_worker, &jobs[t]);
        }
        for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    }
    free(jobs); free(th);
    return total;
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
