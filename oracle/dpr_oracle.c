/*
 * oracle/dpr_oracle.c -- CPU ORACLE for the data-parallel wavefront path tracer.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / `--impl reference` legs may load this library.  It shares no code,
 * header, table or helper with paper_2407_00179_b200/ (the CUDA product path), and the
 * product path never loads it.
 *
 * What it computes (PAPER.md = P:<line>, SURVEY.md section 8(c) = the pinned reading):
 *   - or_render_union: a plain, slow path tracer over the merged UNION of all ranks'
 *     parts -- the "distributed world" of P:357-363 (S3.1.2) rendered as if it were one
 *     world.  P:657-659 (S5.2): "each ray will always find its respectively closest
 *     intersection no matter which rank ... holds that respective geometry".
 *   - or_render_dp: the same estimator, but every ray is traced rank by rank over the
 *     per-rank parts following the ray-forwarding visit rule (P:180-182 S2.2; P:655-659
 *     S5.2; pinned as P8 in SURVEY 8(c)) with the lock-step wavefront schedule of
 *     P:204-216 (S2.2; pinned as P8b).  It records the routing matrices S[kind][src][dst],
 *     visit counts V[kind][rank] and the number of wavefront steps per spp batch.
 *   The paper's invariant: or_render_dp == or_render_union for events, occlusion bits and
 *   pixels (checked in tests/test_oracle_*.py before the oracle is used as a reference).
 *
 * Arithmetic: IEEE binary32, round-to-nearest, NO contraction (build with
 * -ffp-contract=off, no fast-math), denormals kept, written C evaluation order.  The only
 * double-precision code is the oracle's own BVH box test (padded, conservative; it only
 * decides what to skip, never a result) and the pixel accumulator (P11: "the oracle
 * accumulates in double").
 *
 * Pin status of each function: see DESIGN.md "Oracle pins".  Every function below is
 * pinned by a test in tests/test_oracle_*.py.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define OR_EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------------------------ */
/* Public structs (mirrored by oracle/__init__.py with ctypes).                          */
/* ------------------------------------------------------------------------------------ */
enum { OR_TRIS = 0, OR_SPHERES = 1, OR_BRICK = 2 };

typedef struct {
    int32_t rank, kind;
    float albedo[3];
    int64_t n_verts;
    const float *verts;      /* n_verts * 3 */
    int64_t n_tris;
    const int32_t *idx;      /* n_tris * 3 */
    int64_t n_spheres;
    const float *spheres;    /* n_spheres * 4: cx cy cz r */
    int32_t gdims[3];
    float origin[3], spacing[3];
    int32_t cell_lo[3], cell_hi[3]; /* voxels [cell_lo, cell_hi] inclusive are stored */
    const float *voxels;     /* x-fastest */
    const float *tf;         /* 256 * 4 rgba */
    float tf_lo, tf_hi, density_scale;
} or_part;

typedef struct { float E[3], L[3], U[3], V[3]; float lens_radius, focus_dist; } or_camera;

typedef struct {
    int32_t W, H, spp, spp_batch, max_depth, ao_k;
    float ao_radius;
    float light_dir[3], E[3], A[3], B[3];
    float dt;
    uint64_t seed;
    int32_t flags; /* bit0: jitter fixed at 0.5; bit3: ring schedule (routing simulator);
                      bit4: delta tracking instead of the P10 march (R-DELTA);
                      bit2: no background (local render of the
                      compositing contrast device) */
} or_frame;

/* ------------------------------------------------------------------------------------ */
/* P1: Philox4x32-10 (Salmon et al., SC'11 / Random123).                                  */
/* ------------------------------------------------------------------------------------ */
static void philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        if (round < 9) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* u = (float)(x>>8) * 2^-24, in [0, 1-2^-24] exactly (P1). */
static float u01(uint32_t x) { return (float)(x >> 8) * 0x1p-24f; }

enum { PUR_CAMERA = 0, PUR_LENS = 1, PUR_AO = 2, PUR_BOUNCE = 3, PUR_VOL_PATH = 4, PUR_VOL_SHADOW = 5,
       PUR_VOL_AO = 6, PUR_ISO = 7 };

/* Counter = (p, s, (depth<<8)|purpose, sub); key = (seed lo, seed hi)  (P1). */
static void rng4(uint64_t seed, uint32_t p, uint32_t s, uint32_t depth, uint32_t purpose,
                 uint32_t sub, uint32_t out[4])
{
    uint32_t ctr[4] = {p, s, (depth << 8) | purpose, sub};
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    philox4x32_10(ctr, key, out);
}

/* ------------------------------------------------------------------------------------ */
/* float3 helpers with the pinned evaluation order.                                      */
/* ------------------------------------------------------------------------------------ */
typedef struct { float x, y, z; } v3;
static v3 V3(float x, float y, float z) { v3 r; r.x = x; r.y = y; r.z = z; return r; }
static v3 vsub(v3 a, v3 b) { return V3(a.x - b.x, a.y - b.y, a.z - b.z); }
static v3 vmul(v3 a, v3 b) { return V3(a.x * b.x, a.y * b.y, a.z * b.z); }
static v3 vscale(v3 a, float s) { return V3(a.x * s, a.y * s, a.z * s); }
static float vdot(v3 a, v3 b) { float r = a.x * b.x + a.y * b.y; r = r + a.z * b.z; return r; }
static v3 vcross(v3 a, v3 b)
{
    return V3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static float vget(v3 a, int c) { return c == 0 ? a.x : (c == 1 ? a.y : a.z); }
static v3 vload(const float *p) { return V3(p[0], p[1], p[2]); }

/* ------------------------------------------------------------------------------------ */
/* P3: Moeller-Trumbore, double-sided, no epsilon.  Returns 1 and t if valid.            */
/* ------------------------------------------------------------------------------------ */
static int tri_hit(v3 o, v3 d, float tmax, v3 v0, v3 e1, v3 e2, float *t_out)
{
    v3 pv = vcross(d, e2);
    float det = vdot(e1, pv);
    if (det == 0.0f) return 0;
    float inv = 1.0f / det;
    v3 tv = vsub(o, v0);
    float u = vdot(tv, pv) * inv;
    if (u < 0.0f || u > 1.0f) return 0;
    v3 qv = vcross(tv, e1);
    float v = vdot(d, qv) * inv;
    if (v < 0.0f || u + v > 1.0f) return 0;
    float t = vdot(e2, qv) * inv;
    if (!(t > 0.0f && t < tmax)) return 0;
    *t_out = t;
    return 1;
}

/* Edges of a committed triangle (P3 precompute e1 = v1-v0, e2 = v2-v0), with reading
 * R-DEGEN: a triangle whose binary32 cross(e1, e2) is exactly the zero vector has
 * no area and no normal; it is stored with e1 = e2 = 0, so P3's det == 0 test always rejects
 * it (otherwise rounding can make MT report a hit whose normal is 0/0). */
static void tri_edges(v3 v0, v3 v1, v3 v2, v3 *e1, v3 *e2)
{
    *e1 = vsub(v1, v0);
    *e2 = vsub(v2, v0);
    v3 ng = vcross(*e1, *e2);
    if (ng.x == 0.0f && ng.y == 0.0f && ng.z == 0.0f) { *e1 = V3(0, 0, 0); *e2 = V3(0, 0, 0); }
}

/* Orient a unit normal against the ray: negate if dot(n,d) > 0 (P3). */
static v3 orient(v3 n, v3 d)
{
    if (vdot(n, d) > 0.0f) return V3(-n.x, -n.y, -n.z);
    return n;
}

static v3 tri_normal(v3 e1, v3 e2, v3 d)
{
    v3 ng = vcross(e1, e2);
    float len = sqrtf(vdot(ng, ng));
    v3 n = V3(ng.x / len, ng.y / len, ng.z / len);
    return orient(n, d);
}

/* P4: sphere, reading R-SPHERE: the discriminant is taken from the perpendicular
 * distance, disc = r^2 - |f - b d|^2 (cancellation-free, Ray Tracing Gems I ch. 7), instead
 * of b^2 - (|f|^2 - r^2), whose rounding error (~ulp(|f|^2)) rivals r^2 for small distant
 * spheres and reports "hits" outside the sphere's own bounding box. */
static int sphere_hit(v3 o, v3 d, float tmax, v3 c, float r, float *t_out)
{
    v3 f = vsub(o, c);
    float b = vdot(f, d);
    v3 q = V3(f.x - b * d.x, f.y - b * d.y, f.z - b * d.z);
    float disc = r * r - vdot(q, q);
    if (disc < 0.0f) return 0;
    float sq = sqrtf(disc);
    float t = -b - sq;
    if (!(t > 0.0f)) t = -b + sq;
    if (!(t > 0.0f && t < tmax)) return 0;
    *t_out = t;
    return 1;
}

static v3 sphere_normal(v3 o, v3 d, float t, v3 c, float r)
{
    v3 p = V3(o.x + t * d.x, o.y + t * d.y, o.z + t * d.z);
    v3 n = V3((p.x - c.x) / r, (p.y - c.y) / r, (p.z - c.z) / r);
    return orient(n, d);
}

/* ------------------------------------------------------------------------------------ */
/* P8: slab test against a box, minNum semantics (C99 fminf/fmaxf drop NaN).             */
/* ------------------------------------------------------------------------------------ */
static int slab(const float lo[3], const float hi[3], v3 o, v3 d, float tmax, float *t0_out,
                float *t1_out)
{
    float oo[3] = {o.x, o.y, o.z}, dd[3] = {d.x, d.y, d.z};
    float nr[3], fr[3];
    for (int c = 0; c < 3; ++c) {
        float inv = 1.0f / dd[c];
        float ta = (lo[c] - oo[c]) * inv;
        float tb = (hi[c] - oo[c]) * inv;
        nr[c] = fminf(ta, tb);
        fr[c] = fmaxf(ta, tb);
    }
    float t0 = fmaxf(fmaxf(fmaxf(0.0f, nr[0]), nr[1]), nr[2]);
    float t1 = fminf(fminf(fminf(tmax, fr[0]), fr[1]), fr[2]);
    *t0_out = t0;
    if (t1_out) *t1_out = t1;
    return t0 <= t1;
}

/* ------------------------------------------------------------------------------------ */
/* P10: structured bricks -- trilinear + transfer function.                               */
/* ------------------------------------------------------------------------------------ */
typedef struct {
    int rank;
    int32_t gd[3], lo[3], hi[3];
    float O[3], h[3];
    const float *vox;
    const float *tf;
    float tf_lo, tf_hi, dscale;
    float box_lo[3], box_hi[3]; /* world box of the cell domain [cell_lo, cell_hi] */
} OBrick;

static float lerpf(float a, float b, float w) { return a + w * (b - a); }

static float brick_voxel(const OBrick *b, int x, int y, int z)
{
    int64_t nx = b->hi[0] - b->lo[0] + 1, ny = b->hi[1] - b->lo[1] + 1;
    int64_t i = (int64_t)(x - b->lo[0]) + nx * ((int64_t)(y - b->lo[1]) + ny * (int64_t)(z - b->lo[2]));
    return b->vox[i];
}

/* Grid coordinate g.c = (p.c - O.c)/h.c against the GLOBAL origin/spacing (P10). */
static v3 grid_coord(const OBrick *b, v3 p)
{
    return V3((p.x - b->O[0]) / b->h[0], (p.y - b->O[1]) / b->h[1], (p.z - b->O[2]) / b->h[2]);
}

/* Ownership: cell_lo <= g < cell_hi per axis (half-open). */
static int brick_owns(const OBrick *b, v3 g)
{
    for (int c = 0; c < 3; ++c) {
        float gc = vget(g, c);
        if (!(gc >= (float)b->lo[c] && gc < (float)b->hi[c])) return 0;
    }
    return 1;
}

static float brick_trilinear(const OBrick *b, v3 g)
{
    float fx0 = floorf(g.x), fy0 = floorf(g.y), fz0 = floorf(g.z);
    int ix = (int)fx0, iy = (int)fy0, iz = (int)fz0;
    float fx = g.x - fx0, fy = g.y - fy0, fz = g.z - fz0;
    float v000 = brick_voxel(b, ix, iy, iz), v100 = brick_voxel(b, ix + 1, iy, iz);
    float v010 = brick_voxel(b, ix, iy + 1, iz), v110 = brick_voxel(b, ix + 1, iy + 1, iz);
    float v001 = brick_voxel(b, ix, iy, iz + 1), v101 = brick_voxel(b, ix + 1, iy, iz + 1);
    float v011 = brick_voxel(b, ix, iy + 1, iz + 1), v111 = brick_voxel(b, ix + 1, iy + 1, iz + 1);
    float c00 = lerpf(v000, v100, fx), c10 = lerpf(v010, v110, fx);
    float c01 = lerpf(v001, v101, fx), c11 = lerpf(v011, v111, fx);
    float c0 = lerpf(c00, c10, fy), c1 = lerpf(c01, c11, fy);
    return lerpf(c0, c1, fz);
}

/* TF: 256 entries over [lo,hi]; returns rgba, alpha = min(1, a*densityScale). */
static void tf_eval(const float *tf, float lo, float hi, float dscale, float s, float rgba[4])
{
    float x = fminf(fmaxf((s - lo) / (hi - lo), 0.0f), 1.0f) * 255.0f;
    int j = (int)floorf(x);
    if (j > 254) j = 254;
    float w = x - (float)j;
    for (int c = 0; c < 4; ++c) rgba[c] = tf[4 * j + c] + w * (tf[4 * (j + 1) + c] - tf[4 * j + c]);
    rgba[3] = fminf(1.0f, rgba[3] * dscale);
}

/* Sample i: t_i = ((float)i + 0.5f)*dt, p.c = o.c + t_i*d.c (P10). */
static float sample_t(int64_t i, float dt) { return ((float)i + 0.5f) * dt; }
static v3 sample_p(v3 o, v3 d, float t)
{
    return V3(o.x + t * d.x, o.y + t * d.y, o.z + t * d.z);
}

/* March range for a box padded by one voxel (reading R-VOL-RANGE):
 * i in [max(0, floor(t0/dt - 0.5) - 1), ceil(t1/dt) + 1]. */
static int march_range(const float blo[3], const float bhi[3], const float h[3], v3 o, v3 d,
                       float tmax, float dt, int64_t *i0, int64_t *i1)
{
    float plo[3], phi[3];
    for (int c = 0; c < 3; ++c) { plo[c] = blo[c] - h[c]; phi[c] = bhi[c] + h[c]; }
    float t0, t1;
    if (!slab(plo, phi, o, d, tmax, &t0, &t1)) return 0;
    float a = floorf(t0 / dt - 0.5f);
    float bb = ceilf(t1 / dt);
    if (bb > 1.0e9f) bb = 1.0e9f;
    int64_t s0 = (int64_t)a - 1;
    if (s0 < 0) s0 = 0;
    *i0 = s0;
    *i1 = (int64_t)bb + 1;
    return 1;
}

/* ------------------------------------------------------------------------------------ */
/* Scene: prims with global ids (P12), per-rank + union BVHs (oracle's own median split). */
/* ------------------------------------------------------------------------------------ */
typedef struct {
    int type;      /* 0 tri, 1 sphere */
    uint32_t id;   /* global id */
    int32_t part;  /* global part index -> albedo */
    v3 a, b, c;    /* tri: v0, e1, e2; sphere: centre, (r,0,0) */
    float lo[3], hi[3];
} OPrim;

typedef struct {
    double lo[3], hi[3];
    int64_t left, right; /* internal: children */
    int64_t start, count; /* leaf: count > 0 */
} ONode;

typedef struct {
    int64_t *ref; /* prim indices */
    int64_t n;
    ONode *nodes;
    int64_t nn, cap;
} OBVH;

typedef struct {
    int nranks;
    OPrim *prims;          /* union, in global id order */
    int64_t nprims;
    float (*albedo)[3];    /* per global part */
    int nparts;
    OBrick *bricks;
    int nbricks;
    OBVH ubvh;             /* union */
    OBVH *rbvh;            /* per rank */
    float (*rbox)[6];      /* padded rank boxes lo3 hi3 */
    int *rank_nonempty;
    float ubox[6];         /* union brick domain box (unpadded) */
    int has_volume;
    float amax;            /* delta tracking majorant: max TF alpha over all bricks */
    float gdom[6];         /* global grid domain O .. O + (gdims-1) h */
} OScene;

static double centroid(const OPrim *p, int axis)
{
    return 0.5 * ((double)p->lo[axis] + (double)p->hi[axis]);
}

typedef struct { double key; int64_t idx; } KeyIdx;

static int ki_less(const KeyIdx *a, const KeyIdx *b)
{
    return a->key < b->key || (a->key == b->key && a->idx < b->idx);
}

/* Quickselect: place the k-th smallest (by (key, idx)) at position k. */
static void kselect(KeyIdx *v, int64_t n, int64_t k)
{
    int64_t lo = 0, hi = n - 1;
    while (hi > lo) {
        KeyIdx pivot = v[lo + (hi - lo) / 2];
        int64_t i = lo, j = hi;
        while (i <= j) {
            while (ki_less(&v[i], &pivot)) ++i;
            while (ki_less(&pivot, &v[j])) --j;
            if (i <= j) { KeyIdx t = v[i]; v[i] = v[j]; v[j] = t; ++i; --j; }
        }
        if (k <= j) hi = j;
        else if (k >= i) lo = i;
        else return;
    }
}

static int64_t bvh_push(OBVH *b)
{
    if (b->nn == b->cap) {
        b->cap = b->cap ? 2 * b->cap : 1024;
        b->nodes = (ONode *)realloc(b->nodes, (size_t)b->cap * sizeof(ONode));
    }
    return b->nn++;
}

/* Box padding of the oracle's BVH (conservative). */
static double pad_of(double x) { return 1e-6 + 1e-6 * fabs(x); }

static int64_t bvh_build_rec(OBVH *b, const OPrim *prims, KeyIdx *tmp, int64_t first, int64_t count)
{
    int64_t ni = bvh_push(b);
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    double clo[3] = {INFINITY, INFINITY, INFINITY}, chi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = first; i < first + count; ++i) {
        const OPrim *p = &prims[b->ref[i]];
        for (int c = 0; c < 3; ++c) {
            if (p->lo[c] < lo[c]) lo[c] = p->lo[c];
            if (p->hi[c] > hi[c]) hi[c] = p->hi[c];
            double cc = centroid(p, c);
            if (cc < clo[c]) clo[c] = cc;
            if (cc > chi[c]) chi[c] = cc;
        }
    }
    ONode nd;
    for (int c = 0; c < 3; ++c) { nd.lo[c] = lo[c] - pad_of(lo[c]); nd.hi[c] = hi[c] + pad_of(hi[c]); }
    if (count <= 4) {
        nd.left = nd.right = -1; nd.start = first; nd.count = count;
        b->nodes[ni] = nd;
        return ni;
    }
    int axis = 0;
    double ext = chi[0] - clo[0];
    for (int c = 1; c < 3; ++c) if (chi[c] - clo[c] > ext) { ext = chi[c] - clo[c]; axis = c; }
    for (int64_t i = 0; i < count; ++i) {
        tmp[i].key = centroid(&prims[b->ref[first + i]], axis);
        tmp[i].idx = b->ref[first + i];
    }
    int64_t half = count / 2;
    kselect(tmp, count, half);
    /* After kselect, [0,half) <= tmp[half] <= (half,count) -- partition by comparing. */
    KeyIdx pivot = tmp[half];
    int64_t w = first;
    for (int64_t i = 0; i < count; ++i) if (ki_less(&tmp[i], &pivot)) b->ref[w++] = tmp[i].idx;
    for (int64_t i = 0; i < count; ++i) if (!ki_less(&tmp[i], &pivot)) b->ref[w++] = tmp[i].idx;
    nd.start = -1; nd.count = 0;
    int64_t l = bvh_build_rec(b, prims, tmp, first, half);
    int64_t r = bvh_build_rec(b, prims, tmp, first + half, count - half);
    nd.left = l; nd.right = r;
    b->nodes[ni] = nd;
    return ni;
}

static void bvh_build(OBVH *b, const OPrim *prims, const int64_t *sel, int64_t n)
{
    memset(b, 0, sizeof(*b));
    b->n = n;
    b->ref = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) b->ref[i] = sel[i];
    if (n == 0) return;
    KeyIdx *tmp = (KeyIdx *)malloc((size_t)n * sizeof(KeyIdx));
    bvh_build_rec(b, prims, tmp, 0, n);
    free(tmp);
}

static void bvh_free(OBVH *b) { free(b->ref); free(b->nodes); memset(b, 0, sizeof(*b)); }

/* Double-precision box entry; conservative: returns 0 only if the ray surely misses the
 * padded box within [0, tbound]. */
static int box_enter(const ONode *nd, const double o[3], const double d[3], double tbound,
                     double *tnear)
{
    double t0 = 0.0, t1 = tbound;
    for (int c = 0; c < 3; ++c) {
        if (d[c] == 0.0) {
            if (o[c] < nd->lo[c] || o[c] > nd->hi[c]) return 0;
            continue;
        }
        double ta = (nd->lo[c] - o[c]) / d[c], tb = (nd->hi[c] - o[c]) / d[c];
        if (ta > tb) { double t = ta; ta = tb; tb = t; }
        if (ta > t0) t0 = ta;
        if (tb < t1) t1 = tb;
    }
    double slack = 1e-6 * (1.0 + fabs(t1));
    if (t0 > t1 + slack) return 0;
    *tnear = t0;
    return 1;
}

typedef struct { float t; uint32_t id; v3 n; } OHit; /* id 0xffffffff: no event */

static void hit_none(OHit *h) { h->t = INFINITY; h->id = 0xffffffffu; h->n = V3(0, 0, 0); }

/* P9 rule: t < bestT or (t == bestT and id < bestId). */
static int better(float t, uint32_t id, const OHit *h)
{
    return t < h->t || (t == h->t && id < h->id);
}

static void prim_closest(const OPrim *p, v3 o, v3 d, float tmax, OHit *best)
{
    float t;
    if (p->type == 0) {
        if (tri_hit(o, d, tmax, p->a, p->b, p->c, &t) && better(t, p->id, best)) {
            best->t = t; best->id = p->id; best->n = tri_normal(p->b, p->c, d);
        }
    } else {
        if (sphere_hit(o, d, tmax, p->a, p->b.x, &t) && better(t, p->id, best)) {
            best->t = t; best->id = p->id; best->n = sphere_normal(o, d, t, p->a, p->b.x);
        }
    }
}

static int prim_any(const OPrim *p, v3 o, v3 d, float tmax)
{
    float t;
    if (p->type == 0) return tri_hit(o, d, tmax, p->a, p->b, p->c, &t);
    return sphere_hit(o, d, tmax, p->a, p->b.x, &t);
}

/* Test switch: trace by brute force over the BVH's prim list instead of the BVH (the P9
 * definition itself); used by tests to pin the BVH on large scenes. */
static int g_brute = 0;
OR_EXPORT void or_set_brute(int on) { g_brute = on; }

/* Closest hit through the oracle BVH (equals brute force; pinned by tests). */
static void bvh_closest(const OBVH *b, const OPrim *prims, v3 o, v3 d, float tmax, OHit *best)
{
    if (b->n == 0) return;
    if (g_brute) {
        for (int64_t i = 0; i < b->n; ++i) prim_closest(&prims[b->ref[i]], o, d, tmax, best);
        return;
    }
    double od[3] = {o.x, o.y, o.z}, dd[3] = {d.x, d.y, d.z};
    int64_t stack[128];
    int sp = 0;
    stack[sp++] = 0;
    while (sp) {
        const ONode *nd = &b->nodes[stack[--sp]];
        double bound = (double)fminf(tmax, best->t);
        double tn;
        if (!box_enter(nd, od, dd, isinf(bound) ? INFINITY : bound * (1.0 + 1e-6) + 1e-6, &tn)) continue;
        if (nd->count > 0) {
            for (int64_t i = nd->start; i < nd->start + nd->count; ++i)
                prim_closest(&prims[b->ref[i]], o, d, tmax, best);
        } else {
            stack[sp++] = nd->right;
            stack[sp++] = nd->left;
        }
    }
}

static int bvh_any(const OBVH *b, const OPrim *prims, v3 o, v3 d, float tmax)
{
    if (b->n == 0) return 0;
    if (g_brute) {
        for (int64_t i = 0; i < b->n; ++i) if (prim_any(&prims[b->ref[i]], o, d, tmax)) return 1;
        return 0;
    }
    double od[3] = {o.x, o.y, o.z}, dd[3] = {d.x, d.y, d.z};
    int64_t stack[128];
    int sp = 0;
    stack[sp++] = 0;
    double bound = isinf(tmax) ? INFINITY : (double)tmax * (1.0 + 1e-6) + 1e-6;
    while (sp) {
        const ONode *nd = &b->nodes[stack[--sp]];
        double tn;
        if (!box_enter(nd, od, dd, bound, &tn)) continue;
        if (nd->count > 0) {
            for (int64_t i = nd->start; i < nd->start + nd->count; ++i)
                if (prim_any(&prims[b->ref[i]], o, d, tmax)) return 1;
        } else {
            stack[sp++] = nd->right;
            stack[sp++] = nd->left;
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------------------ */
/* Volume marching.                                                                      */
/* ------------------------------------------------------------------------------------ */
static float vol_u(uint64_t seed, uint32_t p, uint32_t s, uint32_t depth, uint32_t purpose,
                   uint32_t subhi, int64_t i)
{
    uint32_t x[4];
    rng4(seed, p, s, depth, purpose, subhi | (uint32_t)(i >> 2), x);
    return u01(x[i & 3]);
}

typedef struct {
    uint64_t seed;
    uint32_t p, s, depth, purpose, subhi; /* purpose 4/5/6, subhi = k<<24 for AO */
} VolKey;

/* Sample i against a brick: returns 1 and alpha/rgb if the brick owns the sample. */
static int brick_sample(const OBrick *b, v3 pt, float rgba[4])
{
    v3 g = grid_coord(b, pt);
    if (!brick_owns(b, g)) return 0;
    float s = brick_trilinear(b, g);
    tf_eval(b->tf, b->tf_lo, b->tf_hi, b->dscale, s, rgba);
    return 1;
}

/* Per-brick march, path ray: first collision with t_i < best->t becomes the event. */
static void brick_march_path(const OBrick *b, v3 o, v3 d, float dt, const VolKey *k, OHit *best)
{
    int64_t i0, i1;
    if (!march_range(b->box_lo, b->box_hi, b->h, o, d, INFINITY, dt, &i0, &i1)) return;
    for (int64_t i = i0; i <= i1; ++i) {
        float ti = sample_t(i, dt);
        if (!(ti < best->t)) return;
        v3 pt = sample_p(o, d, ti);
        float rgba[4];
        if (!brick_sample(b, pt, rgba)) continue;
        float u = vol_u(k->seed, k->p, k->s, k->depth, k->purpose, k->subhi, i);
        if (u < rgba[3]) {
            best->t = ti; best->id = 0x80000000u | (uint32_t)i; best->n = V3(rgba[0], rgba[1], rgba[2]);
            return;
        }
    }
}

static int brick_march_any(const OBrick *b, v3 o, v3 d, float tmax, float dt, const VolKey *k)
{
    int64_t i0, i1;
    if (!march_range(b->box_lo, b->box_hi, b->h, o, d, tmax, dt, &i0, &i1)) return 0;
    for (int64_t i = i0; i <= i1; ++i) {
        float ti = sample_t(i, dt);
        if (!(ti < tmax)) return 0;
        v3 pt = sample_p(o, d, ti);
        float rgba[4];
        if (!brick_sample(b, pt, rgba)) continue;
        float u = vol_u(k->seed, k->p, k->s, k->depth, k->purpose, k->subhi, i);
        if (u < rgba[3]) return 1;
    }
    return 0;
}

/* ------------------------------------------------------------------------------------ */
/* Delta tracking (NEXT f4; readings R-DELTA and R-LOG).                        */
/* ------------------------------------------------------------------------------------ */
/* R-LOG: natural logarithm of x in (0, 1] in binary32, operation by operation (the
 * fdlibm/Cephes logf reduction; no contraction):
 *   x = m*2^e, m in [1,2) (from the bits); if m > sqrt2 (0x3fb504f3) then m = m*0.5, e = e+1;
 *   f = m - 1; s = f/(2+f); z = s*s; w = z*z;
 *   R = z*(Lg1 + w*Lg3) + w*(Lg2 + w*Lg4);  hfsq = (0.5*f)*f;
 *   ln x = e*ln2_hi - ((hfsq - (s*(hfsq + R) + e*ln2_lo)) - f). */
static float pln(float x)
{
    const float Lg1 = 0x1.555554p-1f, Lg2 = 0x1.999c26p-2f, Lg3 = 0x1.23d3dcp-2f, Lg4 = 0x1.f13c4cp-3f;
    const float ln2_hi = 0x1.62e3p-1f, ln2_lo = 0x1.2fefa2p-17f;
    uint32_t bits;
    memcpy(&bits, &x, 4);
    int e = (int)((bits >> 23) & 0xff) - 127;
    uint32_t mb = (bits & 0x007fffffu) | 0x3f800000u;
    float m;
    memcpy(&m, &mb, 4);
    if (mb > 0x3fb504f3u) { m = m * 0.5f; e = e + 1; }
    float f = m - 1.0f;
    float s = f / (2.0f + f);
    float z = s * s, w = z * z;
    float R = z * (Lg1 + w * Lg3) + w * (Lg2 + w * Lg4);
    float hfsq = (0.5f * f) * f;
    float fe = (float)e;
    return fe * ln2_hi - ((hfsq - (s * (hfsq + R) + fe * ln2_lo)) - f);
}

/* R-DELTA (Woodcock tracking with one global majorant).  Extinction mu(x) = alpha(x)/dt
 * (alpha = the TF opacity of P10, per dt of path); majorant mu_bar = amax/dt.  Tentative
 * points: t = t_start (entry into the global grid domain, P8 slab, clamped at 0); for
 * k = 0, 1, ...: (xi_k, zeta_k) = lanes 2(k&1), 2(k&1)+1 of Philox(p, s, depth<<8|purpose,
 * subhi | k>>1); t += ((0 - ln(1 - xi_k)) * dt) / amax; stop when !(t < min(limit, t_exit));
 * x = o + t d; the owner brick (half-open) decides: real collision iff zeta_k*amax < alpha(x).
 * A collision is event VOL_BIT | k with the TF rgb.  Points are generated identically on
 * every rank; a rank evaluates only the points its own bricks own (rank < 0: all bricks). */
static int delta_track(const OScene *sc, int rank, v3 o, v3 d, float limit, float dt, const VolKey *k,
                       OHit *best)
{
    if (!sc->has_volume || !(sc->amax > 0.0f)) return 0;
    float t, t1;
    if (!slab(sc->gdom, sc->gdom + 3, o, d, INFINITY, &t, &t1)) return 0;
    float tend = fminf(t1, limit);
    for (uint32_t kk = 0; kk < (1u << 25); ++kk) {
        uint32_t x[4];
        rng4(k->seed, k->p, k->s, k->depth, k->purpose, k->subhi | (kk >> 1), x);
        float xi = u01(x[2 * (kk & 1)]), zeta = u01(x[2 * (kk & 1) + 1]);
        float L = 0.0f - pln(1.0f - xi);
        t = t + (L * dt) / sc->amax;
        if (!(t < tend)) return 0;
        v3 pt = sample_p(o, d, t);
        for (int b = 0; b < sc->nbricks; ++b) {
            if (rank >= 0 && sc->bricks[b].rank != rank) continue;
            float rgba[4];
            if (!brick_sample(&sc->bricks[b], pt, rgba)) continue;
            if (zeta * sc->amax < rgba[3]) {
                if (best) { best->t = t; best->id = 0x80000000u | kk; best->n = V3(rgba[0], rgba[1], rgba[2]); }
                return 1;
            }
            break;  /* one owner per point */
        }
    }
    return 0;
}

/* Union march: one march over the whole volume domain, the owner brick looked up per
 * sample (the merged world of P:357-363 as ONE grid). */
static const OBrick *union_owner(const OScene *sc, v3 pt)
{
    for (int b = 0; b < sc->nbricks; ++b) {
        v3 g = grid_coord(&sc->bricks[b], pt);
        if (brick_owns(&sc->bricks[b], g)) return &sc->bricks[b];
    }
    return NULL;
}

static void union_march_path(const OScene *sc, v3 o, v3 d, float dt, const VolKey *k, OHit *best)
{
    if (!sc->has_volume) return;
    int64_t i0, i1;
    if (!march_range(sc->ubox, sc->ubox + 3, sc->bricks[0].h, o, d, INFINITY, dt, &i0, &i1)) return;
    for (int64_t i = i0; i <= i1; ++i) {
        float ti = sample_t(i, dt);
        if (!(ti < best->t)) return;
        v3 pt = sample_p(o, d, ti);
        const OBrick *b = union_owner(sc, pt);
        if (!b) continue;
        float rgba[4];
        brick_sample(b, pt, rgba);
        float u = vol_u(k->seed, k->p, k->s, k->depth, k->purpose, k->subhi, i);
        if (u < rgba[3]) {
            best->t = ti; best->id = 0x80000000u | (uint32_t)i; best->n = V3(rgba[0], rgba[1], rgba[2]);
            return;
        }
    }
}

static int union_march_any(const OScene *sc, v3 o, v3 d, float tmax, float dt, const VolKey *k)
{
    if (!sc->has_volume) return 0;
    int64_t i0, i1;
    if (!march_range(sc->ubox, sc->ubox + 3, sc->bricks[0].h, o, d, tmax, dt, &i0, &i1)) return 0;
    for (int64_t i = i0; i <= i1; ++i) {
        float ti = sample_t(i, dt);
        if (!(ti < tmax)) return 0;
        v3 pt = sample_p(o, d, ti);
        const OBrick *b = union_owner(sc, pt);
        if (!b) continue;
        float rgba[4];
        brick_sample(b, pt, rgba);
        float u = vol_u(k->seed, k->p, k->s, k->depth, k->purpose, k->subhi, i);
        if (u < rgba[3]) return 1;
    }
    return 0;
}

/* ------------------------------------------------------------------------------------ */
/* Scene construction.                                                                   */
/* ------------------------------------------------------------------------------------ */
static void fbox_grow(float lo[3], float hi[3], const float plo[3], const float phi[3])
{
    for (int c = 0; c < 3; ++c) {
        lo[c] = fminf(lo[c], plo[c]);
        hi[c] = fmaxf(hi[c], phi[c]);
    }
}

OR_EXPORT void or_scene_free(OScene *sc)
{
    if (!sc) return;
    free(sc->prims);
    free(sc->albedo);
    free(sc->bricks);
    bvh_free(&sc->ubvh);
    if (sc->rbvh) for (int r = 0; r < sc->nranks; ++r) bvh_free(&sc->rbvh[r]);
    free(sc->rbvh);
    free(sc->rbox);
    free(sc->rank_nonempty);
    free(sc);
}

/* Parts are listed in any order; global ids follow P12: concatenation in rank order, and
 * within a rank the order in which parts appear in the list (the commit order). */
OR_EXPORT OScene *or_scene_build(const or_part *parts, int nparts, int nranks)
{
    OScene *sc = (OScene *)calloc(1, sizeof(OScene));
    sc->nranks = nranks;
    sc->nparts = nparts;
    sc->albedo = (float (*)[3])calloc((size_t)(nparts > 0 ? nparts : 1), sizeof(float[3]));
    int64_t np = 0;
    int nb = 0;
    for (int i = 0; i < nparts; ++i) {
        if (parts[i].rank < 0 || parts[i].rank >= nranks) { or_scene_free(sc); return NULL; }
        if (parts[i].kind == OR_TRIS) np += parts[i].n_tris;
        else if (parts[i].kind == OR_SPHERES) np += parts[i].n_spheres;
        else nb++;
    }
    sc->prims = (OPrim *)malloc((size_t)(np > 0 ? np : 1) * sizeof(OPrim));
    sc->bricks = (OBrick *)calloc((size_t)(nb > 0 ? nb : 1), sizeof(OBrick));
    sc->rbox = (float (*)[6])malloc((size_t)nranks * sizeof(float[6]));
    sc->rank_nonempty = (int *)calloc((size_t)nranks, sizeof(int));
    int64_t *rank_first = (int64_t *)calloc((size_t)nranks + 1, sizeof(int64_t));
    int64_t gid = 0;
    for (int r = 0; r < nranks; ++r) {
        float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        rank_first[r] = gid;
        for (int i = 0; i < nparts; ++i) {
            const or_part *pt = &parts[i];
            if (pt->rank != r) continue;
            for (int c = 0; c < 3; ++c) sc->albedo[i][c] = pt->albedo[c];
            if (pt->kind == OR_TRIS) {
                for (int64_t t = 0; t < pt->n_tris; ++t) {
                    OPrim *p = &sc->prims[gid];
                    v3 v0 = vload(pt->verts + 3 * (int64_t)pt->idx[3 * t + 0]);
                    v3 v1 = vload(pt->verts + 3 * (int64_t)pt->idx[3 * t + 1]);
                    v3 v2 = vload(pt->verts + 3 * (int64_t)pt->idx[3 * t + 2]);
                    p->type = 0; p->id = (uint32_t)gid; p->part = i;
                    if (!isfinite(v0.x) || !isfinite(v0.y) || !isfinite(v0.z) || !isfinite(v1.x) ||
                        !isfinite(v1.y) || !isfinite(v1.z) || !isfinite(v2.x) || !isfinite(v2.y) ||
                        !isfinite(v2.z))
                        goto invalid; /* the GPU path rejects it too (DPR_ERR_INVALID_ARG) */
                    p->a = v0;
                    tri_edges(v0, v1, v2, &p->b, &p->c);
                    for (int c = 0; c < 3; ++c) {
                        p->lo[c] = fminf(fminf(vget(v0, c), vget(v1, c)), vget(v2, c));
                        p->hi[c] = fmaxf(fmaxf(vget(v0, c), vget(v1, c)), vget(v2, c));
                    }
                    fbox_grow(lo, hi, p->lo, p->hi);
                    gid++;
                }
            } else if (pt->kind == OR_SPHERES) {
                for (int64_t s = 0; s < pt->n_spheres; ++s) {
                    OPrim *p = &sc->prims[gid];
                    const float *q = pt->spheres + 4 * s;
                    if (!isfinite(q[0]) || !isfinite(q[1]) || !isfinite(q[2]) || !isfinite(q[3]) || !(q[3] > 0.0f))
                        goto invalid; /* radius must be > 0 and finite (dpr.h) */
                    p->type = 1; p->id = (uint32_t)gid; p->part = i;
                    p->a = V3(q[0], q[1], q[2]); p->b = V3(q[3], 0, 0); p->c = V3(0, 0, 0);
                    for (int c = 0; c < 3; ++c) { p->lo[c] = q[c] - q[3]; p->hi[c] = q[c] + q[3]; }
                    fbox_grow(lo, hi, p->lo, p->hi);
                    gid++;
                }
            } else {
                OBrick *b = &sc->bricks[sc->nbricks++];
                b->rank = r;
                for (int c = 0; c < 3; ++c) {
                    b->gd[c] = pt->gdims[c]; b->lo[c] = pt->cell_lo[c]; b->hi[c] = pt->cell_hi[c];
                    b->O[c] = pt->origin[c]; b->h[c] = pt->spacing[c];
                    b->box_lo[c] = pt->origin[c] + (float)pt->cell_lo[c] * pt->spacing[c];
                    b->box_hi[c] = pt->origin[c] + (float)pt->cell_hi[c] * pt->spacing[c];
                }
                b->vox = pt->voxels; b->tf = pt->tf;
                b->tf_lo = pt->tf_lo; b->tf_hi = pt->tf_hi; b->dscale = pt->density_scale;
                fbox_grow(lo, hi, b->box_lo, b->box_hi);
            }
        }
        int nonempty = lo[0] <= hi[0];
        sc->rank_nonempty[r] = nonempty;
        for (int c = 0; c < 3; ++c) {
            sc->rbox[r][c] = lo[c] - 1e-4f;     /* P8 pad */
            sc->rbox[r][3 + c] = hi[c] + 1e-4f;
        }
    }
    rank_first[nranks] = gid;
    sc->nprims = gid;
    /* union brick domain */
    sc->has_volume = sc->nbricks > 0;
    for (int c = 0; c < 3; ++c) { sc->ubox[c] = INFINITY; sc->ubox[3 + c] = -INFINITY; }
    for (int b = 0; b < sc->nbricks; ++b) fbox_grow(sc->ubox, sc->ubox + 3, sc->bricks[b].box_lo, sc->bricks[b].box_hi);
    /* delta tracking (R-DELTA): majorant = max over bricks and TF entries of min(1, a*dscale);
     * the tentative-point sequence starts where the ray enters the GLOBAL grid domain */
    sc->amax = 0.0f;
    for (int b = 0; b < sc->nbricks; ++b)
        for (int j = 0; j < 256; ++j) {
            float a = fminf(1.0f, sc->bricks[b].tf[4 * j + 3] * sc->bricks[b].dscale);
            if (a > sc->amax) sc->amax = a;
        }
    if (sc->nbricks > 0)
        for (int c = 0; c < 3; ++c) {
            const OBrick *b0 = &sc->bricks[0];
            sc->gdom[c] = b0->O[c];
            sc->gdom[3 + c] = b0->O[c] + (float)(b0->gd[c] - 1) * b0->h[c];
        }
    /* BVHs */
    int64_t *sel = (int64_t *)malloc((size_t)(gid > 0 ? gid : 1) * sizeof(int64_t));
    for (int64_t i = 0; i < gid; ++i) sel[i] = i;
    bvh_build(&sc->ubvh, sc->prims, sel, gid);
    sc->rbvh = (OBVH *)calloc((size_t)nranks, sizeof(OBVH));
    for (int r = 0; r < nranks; ++r)
        bvh_build(&sc->rbvh[r], sc->prims, sel + rank_first[r], rank_first[r + 1] - rank_first[r]);
    free(sel);
    free(rank_first);
    return sc;
invalid:
    free(rank_first);
    or_scene_free(sc);
    return NULL;
}

OR_EXPORT int64_t or_scene_nprims(const OScene *sc) { return sc->nprims; }
OR_EXPORT void or_scene_rank_box(const OScene *sc, int r, float out[6], int *nonempty)
{
    memcpy(out, sc->rbox[r], sizeof(float[6]));
    *nonempty = sc->rank_nonempty[r];
}

/* ------------------------------------------------------------------------------------ */
/* P2 camera, P7 directions.                                                             */
/* ------------------------------------------------------------------------------------ */
static void camera_ray(const or_camera *cam, const or_frame *fr, uint32_t p, uint32_t s, v3 *o, v3 *d)
{
    int x = (int)(p % (uint32_t)fr->W), y = (int)(p / (uint32_t)fr->W);
    float jx = 0.5f, jy = 0.5f;
    if (!(fr->flags & 1)) {
        uint32_t r[4];
        rng4(fr->seed, p, s, 0, PUR_CAMERA, 0, r);
        jx = u01(r[0]); jy = u01(r[1]);
    }
    float sx = ((float)x + jx) / (float)fr->W;
    float sy = ((float)y + jy) / (float)fr->H;
    v3 L = vload(cam->L), U = vload(cam->U), Vv = vload(cam->V);
    v3 q = V3((L.x + sx * U.x) + sy * Vv.x, (L.y + sx * U.y) + sy * Vv.y, (L.z + sx * U.z) + sy * Vv.z);
    v3 E = vload(cam->E);
    if (!(cam->lens_radius > 0.0f)) {
        /* pinhole (P2) */
        float len = sqrtf(vdot(q, q));
        *d = V3(q.x / len, q.y / len, q.z / len);
        *o = E;
        return;
    }
    /* Thin lens ("rendered with depth of field"; reading R-DOF).
     * 1. lens point (lx, ly) uniform in the unit disc: the first of 16 Philox draws
     *    (purpose 1, sub = attempt) with lx^2 + ly^2 <= 1, else the centre;
     * 2. lens axes: U and V normalised;
     * 3. origin o = E + (r*lx) Uhat + (r*ly) Vhat;
     * 4. the pinhole ray's point on the focal plane F = E + focus_dist * q (q has unit
     *    component along the view axis, so F lies focus_dist in front of the lens);
     * 5. direction d = normalize(F - o). */
    float lx = 0.0f, ly = 0.0f;
    for (uint32_t a = 0; a < 16; ++a) {
        uint32_t r[4];
        rng4(fr->seed, p, s, 0, PUR_LENS, a, r);
        float ax = 2.0f * u01(r[0]) - 1.0f, ay = 2.0f * u01(r[1]) - 1.0f;
        if (ax * ax + ay * ay <= 1.0f) { lx = ax; ly = ay; break; }
    }
    float lu = sqrtf(vdot(U, U)), lv = sqrtf(vdot(Vv, Vv));
    v3 Uh = V3(U.x / lu, U.y / lu, U.z / lu), Vh = V3(Vv.x / lv, Vv.y / lv, Vv.z / lv);
    float a = cam->lens_radius * lx, b = cam->lens_radius * ly;
    v3 oo = V3((E.x + a * Uh.x) + b * Vh.x, (E.y + a * Uh.y) + b * Vh.y, (E.z + a * Uh.z) + b * Vh.z);
    v3 F = V3(E.x + cam->focus_dist * q.x, E.y + cam->focus_dist * q.y, E.z + cam->focus_dist * q.z);
    v3 g = V3(F.x - oo.x, F.y - oo.y, F.z - oo.z);
    float lg = sqrtf(vdot(g, g));
    *d = V3(g.x / lg, g.y / lg, g.z / lg);
    *o = oo;
}

/* Cosine-weighted direction about n by rejection (P7) + Duff et al. 2017 frame. */
static v3 cosine_dir(v3 n, uint64_t seed, uint32_t p, uint32_t s, uint32_t depth, uint32_t purpose,
                     uint32_t subhi)
{
    for (uint32_t a = 0; a < 16; ++a) {
        uint32_t r[4];
        rng4(seed, p, s, depth, purpose, subhi | a, r);
        float x = 2.0f * u01(r[0]) - 1.0f;
        float y = 2.0f * u01(r[1]) - 1.0f;
        float r2 = x * x + y * y;
        if (!(r2 < 1.0f)) continue;
        float z = sqrtf(1.0f - r2);
        float sg = copysignf(1.0f, n.z);
        float aa = -1.0f / (sg + n.z);
        float b = (n.x * n.y) * aa;
        v3 t1 = V3(1.0f + ((sg * n.x) * n.x) * aa, sg * b, -sg * n.x);
        v3 t2 = V3(b, sg + (n.y * n.y) * aa, -n.y);
        return V3((x * t1.x + y * t2.x) + z * n.x, (x * t1.y + y * t2.y) + z * n.y,
                  (x * t1.z + y * t2.z) + z * n.z);
    }
    return n;
}

static v3 iso_dir(uint64_t seed, uint32_t p, uint32_t s, uint32_t depth)
{
    for (uint32_t a = 0; a < 16; ++a) {
        uint32_t r[4];
        rng4(seed, p, s, depth, PUR_ISO, a, r);
        v3 v = V3(2.0f * u01(r[0]) - 1.0f, 2.0f * u01(r[1]) - 1.0f, 2.0f * u01(r[2]) - 1.0f);
        float r2 = vdot(v, v);
        if (!(r2 > 0.0f && r2 < 1.0f)) continue;
        float l = sqrtf(r2);
        return V3(v.x / l, v.y / l, v.z / l);
    }
    return V3(0.0f, 0.0f, 1.0f);
}

/* P1 call sites.  Each RNG consumer of the renderer goes through
 * one of these, and each is exported for the counter-layout pins (tests/test_oracle_rng.py):
 *   AO ray k of the vertex at depth d:   purpose 2, sub = (k<<4) | attempt
 *   bounce of the vertex at depth d:     purpose 3, sub = attempt
 *   volume sample i of a path ray:       purpose 4, sub = i>>2, lane i&3
 *   volume sample i of a shadow ray:     purpose 5, sub = i>>2, lane i&3
 *   volume sample i of AO ray k:         purpose 6, sub = (k<<24) | (i>>2), lane i&3 */
static v3 ao_dir(v3 n, uint64_t seed, uint32_t p, uint32_t s, uint32_t depth, int k)
{
    return cosine_dir(n, seed, p, s, depth, PUR_AO, (uint32_t)k << 4);
}

static v3 bounce_dir(v3 n, uint64_t seed, uint32_t p, uint32_t s, uint32_t depth)
{
    return cosine_dir(n, seed, p, s, depth, PUR_BOUNCE, 0);
}

/* ------------------------------------------------------------------------------------ */
/* Rendering: a ray tree per (pixel, sample), processed with an explicit stack.          */
/* ------------------------------------------------------------------------------------ */
enum { K_PATH = 0, K_SHADOW = 1, K_AO = 2 };

/* The Philox key of the volume samples of a ray of `kind` (P1: purpose 4/5/6; AO ray k
 * carries k<<24 in the high bits of sub; vol_u adds i>>2 and takes lane i&3). */
static VolKey vol_key(uint64_t seed, uint32_t p, uint32_t s, uint32_t depth, int kind, int k)
{
    VolKey v;
    v.seed = seed; v.p = p; v.s = s; v.depth = depth;
    v.purpose = kind == K_PATH ? PUR_VOL_PATH : (kind == K_SHADOW ? PUR_VOL_SHADOW : PUR_VOL_AO);
    v.subhi = kind == K_AO ? ((uint32_t)k << 24) : 0u;
    return v;
}

typedef struct {
    int kind;
    v3 o, d;
    float tmax;
    v3 w;        /* path: throughput beta; occlusion: contrib */
    int depth;   /* path: this ray's depth; occlusion: depth of the spawning vertex */
    int k;       /* AO index */
    int rank, step; /* dp mode: rank where it is traced next, batch-relative step */
} ORay;

typedef struct {
    const OScene *sc;
    const or_camera *cam;
    const or_frame *fr;
    const int64_t *pix;
    int64_t npix;
    int dp;               /* 0: union renderer, 1: routing simulator */
    double *rgba;
    uint32_t *events, *occl;
    float *depth;         /* optional: per listed pixel, min over samples of the primary event t */
    int64_t *S, *V, *gen, *steps; /* shared outputs, merged under lock */
    int64_t *S_step, *V_step;     /* optional per-step matrices [batch][step][3][N][N], [batch][step][3][N] */
    int max_steps;                /* steps recorded per batch (later steps accumulate into the last) */
    int64_t nbatches;
    int64_t next;         /* atomic work counter */
    pthread_mutex_t lock;
} Job;

typedef struct {
    int64_t *S, *V, gen[3], *steps;
    int64_t *S_step, *V_step;
} Local;

/* P8b per-step counters: a forward or spawn counted in S happens in the exchange of the step
 * in which its ray was traced (resolving ray's step for children), a visit in the step that
 * traces it; rays carry their batch-relative step. */
static void count_S(const Job *J, Local *L, int64_t batch, int step, int kind, int src, int dst)
{
    const int N = J->sc->nranks;
    L->S[(kind * N + src) * N + dst]++;
    if (L->S_step) {
        const int k = step < J->max_steps ? step : J->max_steps - 1;
        L->S_step[(((batch * J->max_steps + k) * 3 + kind) * N + src) * N + dst]++;
    }
}

static void count_V(const Job *J, Local *L, int64_t batch, int step, int kind, int rank)
{
    const int N = J->sc->nranks;
    L->V[kind * N + rank]++;
    if (L->V_step) {
        const int k = step < J->max_steps ? step : J->max_steps - 1;
        L->V_step[((batch * J->max_steps + k) * 3 + kind) * N + rank]++;
    }
}

#define STACK_MAX 256

static int first_candidate(const OScene *sc, v3 o, v3 d, float tmax)
{
    int best = -1;
    float bt = 0;
    for (int r = 0; r < sc->nranks; ++r) {
        if (!sc->rank_nonempty[r]) continue;
        float t0;
        if (!slab(sc->rbox[r], sc->rbox[r] + 3, o, d, tmax, &t0, NULL)) continue;
        if (best < 0 || t0 < bt) { best = r; bt = t0; } /* ties: smaller rank (ascending loop) */
    }
    return best;
}

/* next = min key (t0_r, r) > (t0_c, c) among candidates (P8).  tbound = bestT (path) or
 * tmax (occlusion); candidate iff slab(t0 <= t1 with tmax) and t0 <= tbound. */
static int next_candidate(const OScene *sc, int c, v3 o, v3 d, float tmax, float tbound)
{
    float tc;
    slab(sc->rbox[c], sc->rbox[c] + 3, o, d, INFINITY, &tc, NULL);
    int best = -1;
    float bt = 0;
    for (int r = 0; r < sc->nranks; ++r) {
        if (r == c || !sc->rank_nonempty[r]) continue;
        float t0;
        if (!slab(sc->rbox[r], sc->rbox[r] + 3, o, d, tmax, &t0, NULL)) continue;
        if (!(t0 <= tbound)) continue;
        int gt = t0 > tc || (t0 == tc && r > c);
        if (!gt) continue;
        if (best < 0 || t0 < bt || (t0 == bt && r < best)) { best = r; bt = t0; }
    }
    return best;
}

static void trace_path_at(const Job *J, int rank, const ORay *ray, const VolKey *vk, OHit *best)
{
    const OScene *sc = J->sc;
    if (rank < 0) {
        bvh_closest(&sc->ubvh, sc->prims, ray->o, ray->d, ray->tmax, best);
        if (J->fr->flags & 16) delta_track(sc, -1, ray->o, ray->d, best->t, J->fr->dt, vk, best);
        else union_march_path(sc, ray->o, ray->d, J->fr->dt, vk, best);
    } else {
        bvh_closest(&sc->rbvh[rank], sc->prims, ray->o, ray->d, ray->tmax, best);
        if (J->fr->flags & 16) {
            delta_track(sc, rank, ray->o, ray->d, best->t, J->fr->dt, vk, best);
            return;
        }
        for (int b = 0; b < sc->nbricks; ++b)
            if (sc->bricks[b].rank == rank) brick_march_path(&sc->bricks[b], ray->o, ray->d, J->fr->dt, vk, best);
    }
}

static int trace_occl_at(const Job *J, int rank, const ORay *ray, const VolKey *vk)
{
    const OScene *sc = J->sc;
    if (rank < 0) {
        if (bvh_any(&sc->ubvh, sc->prims, ray->o, ray->d, ray->tmax)) return 1;
        if (J->fr->flags & 16) return delta_track(sc, -1, ray->o, ray->d, ray->tmax, J->fr->dt, vk, NULL);
        return union_march_any(sc, ray->o, ray->d, ray->tmax, J->fr->dt, vk);
    }
    if (bvh_any(&sc->rbvh[rank], sc->prims, ray->o, ray->d, ray->tmax)) return 1;
    if (J->fr->flags & 16) return delta_track(sc, rank, ray->o, ray->d, ray->tmax, J->fr->dt, vk, NULL);
    for (int b = 0; b < sc->nbricks; ++b)
        if (sc->bricks[b].rank == rank && brick_march_any(&sc->bricks[b], ray->o, ray->d, ray->tmax, J->fr->dt, vk))
            return 1;
    return 0;
}

static void note_step(Local *L, int64_t batch, int step)
{
    if (L->steps[batch] < step + 1) L->steps[batch] = step + 1;
}

static void render_sample(const Job *J, Local *L, int64_t pi, uint32_t p, uint32_t s, double acc[4])
{
    const OScene *sc = J->sc;
    const or_frame *fr = J->fr;
    const int N = sc->nranks;
    const int dp = J->dp;
    const int64_t batch = s / (uint32_t)fr->spp_batch;
    const v3 Lt = vload(fr->light_dir), Ei = vload(fr->E), Am = vload(fr->A), Bg = vload(fr->B);
    ORay stack[STACK_MAX];
    int sp = 0;

    /* primary (P2); kept by its first candidate, or by the pixel owner (P8) */
    ORay pr;
    memset(&pr, 0, sizeof(pr));
    pr.kind = K_PATH;
    camera_ray(J->cam, fr, p, s, &pr.o, &pr.d);
    pr.tmax = INFINITY;
    pr.w = V3(1.0f, 1.0f, 1.0f);
    pr.depth = 0;
    L->gen[K_PATH]++;
    /* ring schedule (frame flag bit3; "wave-fronts are exchanged in a ring buffer";
     * reading R-RING): every ray of pixel p starts at its home rank
     * home(p) = floor(p*N/(W*H)) and is traced by home, home+1, ..., home+N-1 (mod N)
     * without culling or early-out; it resolves at the last of them and its children are
     * sent home. */
    const int ring = dp && (fr->flags & 8);
    const int home = (int)(((int64_t)p * N) / ((int64_t)fr->W * fr->H));
    pr.rank = ring ? home : dp ? first_candidate(sc, pr.o, pr.d, INFINITY) : -1;
    pr.step = 0;
    int resolved_now = dp && pr.rank < 0;
    if (resolved_now) {
        /* no candidate: resolves as a miss at the pixel owner without being traced */
        if (J->events) J->events[((int64_t)s * fr->max_depth + 0) * J->npix + pi] = 1;
        if (!(fr->flags & 4)) { acc[0] += Bg.x; acc[1] += Bg.y; acc[2] += Bg.z; }
        return;
    }
    stack[sp++] = pr;

    while (sp) {
        ORay ray = stack[--sp];
        if (ray.kind == K_PATH) {
            OHit best;
            hit_none(&best);
            VolKey vk = vol_key(fr->seed, p, s, (uint32_t)ray.depth, K_PATH, 0);
            int at = ray.rank;
            if (!dp) {
                trace_path_at(J, -1, &ray, &vk, &best);
            } else {
                for (;;) {
                    count_V(J, L, batch, ray.step, K_PATH, at);
                    note_step(L, batch, ray.step);
                    trace_path_at(J, at, &ray, &vk, &best);
                    int nx = ring ? ((at + 1) % N == home ? -1 : (at + 1) % N)
                                  : next_candidate(sc, at, ray.o, ray.d, ray.tmax, best.t);
                    if (nx < 0) break;
                    count_S(J, L, batch, ray.step, K_PATH, at, nx);
                    at = nx;
                    ray.step++;
                }
            }
            /* resolve + shade (P6) at rank `at`, step ray.step */
            uint32_t code = best.id == 0xffffffffu ? 1u : ((best.id & 0x80000000u) ? best.id : 2u + best.id);
            if (J->events) J->events[((int64_t)s * fr->max_depth + ray.depth) * J->npix + pi] = code;
            if (best.id == 0xffffffffu) {
                if (ray.depth == 0 && !(fr->flags & 4)) { acc[0] += Bg.x; acc[1] += Bg.y; acc[2] += Bg.z; }
                continue;
            }
            if (ray.depth == 0) {
                acc[3] += 1.0;
                if (J->depth && best.t < J->depth[pi]) J->depth[pi] = best.t;
            }
            ORay kids[40];
            int nk = 0;
            v3 hp = sample_p(ray.o, ray.d, best.t); /* P5: p.c = o.c + bestT*d.c */
            if (!(best.id & 0x80000000u)) {
                v3 n = best.n;
                v3 rho = vload(sc->albedo[sc->prims[best.id].part]);
                v3 org = V3(hp.x + 1e-4f * n.x, hp.y + 1e-4f * n.y, hp.z + 1e-4f * n.z);
                v3 br = vmul(ray.w, rho);
                float c = vdot(n, Lt);
                if (c > 0.0f) {
                    ORay sh; memset(&sh, 0, sizeof(sh));
                    sh.kind = K_SHADOW; sh.o = org; sh.d = Lt; sh.tmax = INFINITY;
                    sh.w = vscale(vmul(br, Ei), c); sh.depth = ray.depth; sh.k = 0;
                    kids[nk++] = sh;
                }
                for (int k = 0; k < fr->ao_k; ++k) {
                    ORay ao; memset(&ao, 0, sizeof(ao));
                    ao.kind = K_AO; ao.o = org;
                    ao.d = ao_dir(n, fr->seed, p, s, (uint32_t)ray.depth, k);
                    ao.tmax = fr->ao_radius;
                    ao.w = vscale(vmul(br, Am), 1.0f / (float)fr->ao_k);
                    ao.depth = ray.depth; ao.k = k;
                    kids[nk++] = ao;
                }
                if (ray.depth + 1 < fr->max_depth) {
                    ORay bo; memset(&bo, 0, sizeof(bo));
                    bo.kind = K_PATH; bo.o = org;
                    bo.d = bounce_dir(n, fr->seed, p, s, (uint32_t)ray.depth);
                    bo.tmax = INFINITY; bo.w = br; bo.depth = ray.depth + 1;
                    kids[nk++] = bo;
                }
            } else {
                v3 rho = best.n; /* TF rgb carried in the normal slot */
                v3 br = vmul(ray.w, rho);
                ORay sh; memset(&sh, 0, sizeof(sh));
                sh.kind = K_SHADOW; sh.o = hp; sh.d = Lt; sh.tmax = INFINITY;
                sh.w = vmul(br, Ei); sh.depth = ray.depth;
                kids[nk++] = sh;
                if (ray.depth + 1 < fr->max_depth) {
                    ORay bo; memset(&bo, 0, sizeof(bo));
                    bo.kind = K_PATH; bo.o = hp;
                    bo.d = iso_dir(fr->seed, p, s, (uint32_t)ray.depth);
                    bo.tmax = INFINITY; bo.w = br; bo.depth = ray.depth + 1;
                    kids[nk++] = bo;
                }
            }
            /* route the children (P8: first candidate from the resolving rank) */
            for (int i = nk - 1; i >= 0; --i) {
                ORay ch = kids[i];
                L->gen[ch.kind]++;
                if (dp) {
                    int first = ring ? home : first_candidate(sc, ch.o, ch.d, ch.tmax);
                    if (first < 0) {
                        /* resolves immediately at `at` */
                        if (ch.kind == K_PATH) {
                            if (J->events) J->events[((int64_t)s * fr->max_depth + ch.depth) * J->npix + pi] = 1;
                        } else {
                            acc[0] += ch.w.x; acc[1] += ch.w.y; acc[2] += ch.w.z;
                            if (J->occl) J->occl[((int64_t)s * fr->max_depth + ch.depth) * J->npix + pi] |=
                                ch.kind == K_SHADOW ? 1u : (2u << ch.k);
                        }
                        continue;
                    }
                    if (first != at) count_S(J, L, batch, ray.step, ch.kind, at, first);
                    ch.rank = first;
                    ch.step = ray.step + 1;
                }
                if (sp >= STACK_MAX) abort();
                stack[sp++] = ch;
            }
        } else {
            VolKey vk = vol_key(fr->seed, p, s, (uint32_t)ray.depth, ray.kind, ray.k);
            int occluded = 0;
            if (!dp) {
                occluded = trace_occl_at(J, -1, &ray, &vk);
            } else {
                int at = ray.rank;
                for (;;) {
                    count_V(J, L, batch, ray.step, ray.kind, at);
                    note_step(L, batch, ray.step);
                    if (!occluded && trace_occl_at(J, at, &ray, &vk)) {
                        occluded = 1;
                        if (!ring) break;   /* ring: no early-out, the ray completes the ring */
                    }
                    int nx = ring ? ((at + 1) % N == home ? -1 : (at + 1) % N)
                                  : next_candidate(sc, at, ray.o, ray.d, ray.tmax, ray.tmax);
                    if (nx < 0) break;
                    count_S(J, L, batch, ray.step, ray.kind, at, nx);
                    at = nx;
                    ray.step++;
                }
            }
            if (!occluded) {
                acc[0] += ray.w.x; acc[1] += ray.w.y; acc[2] += ray.w.z;
                if (J->occl) J->occl[((int64_t)s * fr->max_depth + ray.depth) * J->npix + pi] |=
                    ray.kind == K_SHADOW ? 1u : (2u << ray.k);
            }
        }
    }
}

static void *worker(void *arg)
{
    Job *J = (Job *)arg;
    const int N = J->sc->nranks;
    Local L;
    memset(&L, 0, sizeof(L));
    L.S = (int64_t *)calloc((size_t)3 * N * N, sizeof(int64_t));
    L.V = (int64_t *)calloc((size_t)3 * N, sizeof(int64_t));
    L.steps = (int64_t *)calloc((size_t)J->nbatches, sizeof(int64_t));
    const size_t nst = (size_t)J->nbatches * (size_t)(J->max_steps > 0 ? J->max_steps : 1) * 3;
    if (J->S_step) L.S_step = (int64_t *)calloc(nst * N * N, sizeof(int64_t));
    if (J->V_step) L.V_step = (int64_t *)calloc(nst * N, sizeof(int64_t));
    for (;;) {
        int64_t i0 = __atomic_fetch_add(&J->next, 16, __ATOMIC_RELAXED);
        if (i0 >= J->npix) break;
        int64_t i1 = i0 + 16 < J->npix ? i0 + 16 : J->npix;
        for (int64_t i = i0; i < i1; ++i) {
            uint32_t p = (uint32_t)J->pix[i];
            double acc[4] = {0, 0, 0, 0};
            for (int s = 0; s < J->fr->spp; ++s) render_sample(J, &L, i, p, (uint32_t)s, acc);
            for (int c = 0; c < 4; ++c) J->rgba[4 * i + c] = acc[c] / (double)J->fr->spp;
        }
    }
    pthread_mutex_lock(&J->lock);
    for (int i = 0; i < 3 * N * N; ++i) if (J->S) J->S[i] += L.S[i];
    for (int i = 0; i < 3 * N; ++i) if (J->V) J->V[i] += L.V[i];
    for (int i = 0; i < 3; ++i) if (J->gen) J->gen[i] += L.gen[i];
    for (int64_t b = 0; b < J->nbatches; ++b)
        if (J->steps && J->steps[b] < L.steps[b]) J->steps[b] = L.steps[b];
    if (J->S_step) for (size_t i = 0; i < nst * N * N; ++i) J->S_step[i] += L.S_step[i];
    if (J->V_step) for (size_t i = 0; i < nst * N; ++i) J->V_step[i] += L.V_step[i];
    pthread_mutex_unlock(&J->lock);
    free(L.S); free(L.V); free(L.steps); free(L.S_step); free(L.V_step);
    return NULL;
}

static int run(const OScene *sc, const or_camera *cam, const or_frame *fr, const int64_t *pix,
               int64_t npix, int dp, double *rgba, uint32_t *events, uint32_t *occl, int64_t *S,
               int64_t *V, int64_t *gen, int64_t *steps, int nthreads, float *depth,
               int64_t *S_step, int64_t *V_step, int max_steps)
{
    if (!sc || !cam || !fr || fr->W <= 0 || fr->H <= 0 || fr->spp <= 0 || fr->spp_batch <= 0 ||
        fr->max_depth <= 0 || fr->ao_k < 0 || fr->ao_k > 30)
        return -1;
    if (sc->has_volume && !(fr->dt > 0.0f)) return -1;
    Job J;
    memset(&J, 0, sizeof(J));
    J.sc = sc; J.cam = cam; J.fr = fr; J.pix = pix; J.npix = npix; J.dp = dp;
    J.rgba = rgba; J.events = events; J.occl = occl; J.S = S; J.V = V; J.gen = gen; J.steps = steps;
    J.depth = depth;
    if (depth) for (int64_t i = 0; i < npix; ++i) depth[i] = INFINITY;
    J.nbatches = (fr->spp + fr->spp_batch - 1) / fr->spp_batch;
    J.S_step = S_step; J.V_step = V_step; J.max_steps = max_steps > 0 ? max_steps : 1;
    if (S_step) memset(S_step, 0, sizeof(int64_t) * (size_t)J.nbatches * J.max_steps * 3 * sc->nranks * sc->nranks);
    if (V_step) memset(V_step, 0, sizeof(int64_t) * (size_t)J.nbatches * J.max_steps * 3 * sc->nranks);
    pthread_mutex_init(&J.lock, NULL);
    if (events) memset(events, 0, (size_t)fr->spp * fr->max_depth * npix * sizeof(uint32_t));
    if (occl) memset(occl, 0, (size_t)fr->spp * fr->max_depth * npix * sizeof(uint32_t));
    if (nthreads <= 0) nthreads = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (nthreads < 1) nthreads = 1;
    pthread_t *th = (pthread_t *)malloc((size_t)nthreads * sizeof(pthread_t));
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, worker, &J);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&J.lock);
    return 0;
}

/* Union renderer (the definition).  rgba: npix*4 doubles = sum/spp; alpha = coverage.
 * events/occl: [spp][max_depth][npix] u32 (P13), may be NULL.  gen: 3 counts. */
OR_EXPORT int or_render_union(const OScene *sc, const or_camera *cam, const or_frame *fr,
                              const int64_t *pix, int64_t npix, double *rgba, uint32_t *events,
                              uint32_t *occl, int64_t *gen, int nthreads)
{
    return run(sc, cam, fr, pix, npix, 0, rgba, events, occl, NULL, NULL, gen, NULL, nthreads, NULL, NULL, NULL, 0);
}

/* Union renderer with a per-pixel depth output (min over samples of the primary event t,
 * +inf if none): the colour + depth buffers a pass-through device hands to the compositing
 * device (S5.1.2). */
OR_EXPORT int or_render_union_depth(const OScene *sc, const or_camera *cam, const or_frame *fr,
                                    const int64_t *pix, int64_t npix, double *rgba, float *depth,
                                    int nthreads)
{
    return run(sc, cam, fr, pix, npix, 0, rgba, NULL, NULL, NULL, NULL, NULL, NULL, nthreads, depth, NULL, NULL, 0);
}

/* Routing simulator (P8/P8b).  S: 3*N*N, V: 3*N, steps: ceil(spp/spp_batch). */
OR_EXPORT int or_render_dp(const OScene *sc, const or_camera *cam, const or_frame *fr,
                           const int64_t *pix, int64_t npix, double *rgba, uint32_t *events,
                           uint32_t *occl, int64_t *S, int64_t *V, int64_t *gen, int64_t *steps,
                           int nthreads)
{
    return run(sc, cam, fr, pix, npix, 1, rgba, events, occl, S, V, gen, steps, nthreads, NULL, NULL, NULL, 0);
}

/* Routing simulator with the P8b per-step matrices: S_step [nbatches][max_steps][3][N][N] and
 * V_step [nbatches][max_steps][3][N] (batch-relative steps; steps >= max_steps accumulate into
 * the last slot).  Their sums over steps are S and V. */
OR_EXPORT int or_render_dp_steps(const OScene *sc, const or_camera *cam, const or_frame *fr,
                                 const int64_t *pix, int64_t npix, double *rgba, uint32_t *events,
                                 uint32_t *occl, int64_t *S, int64_t *V, int64_t *gen, int64_t *steps,
                                 int64_t *S_step, int64_t *V_step, int max_steps, int nthreads)
{
    return run(sc, cam, fr, pix, npix, 1, rgba, events, occl, S, V, gen, steps, nthreads, NULL, S_step, V_step,
               max_steps);
}

/* ------------------------------------------------------------------------------------ */
/* Single-operation exports for the pin tests.                                          */
/* ------------------------------------------------------------------------------------ */
OR_EXPORT void or_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    philox4x32_10(ctr, key, out);
}

OR_EXPORT float or_u01(uint32_t x) { return u01(x); }

OR_EXPORT int or_tri_hit(const float o[3], const float d[3], float tmax, const float v0[3],
                         const float v1[3], const float v2[3], float *t, float n[3])
{
    v3 a = vload(v0), e1, e2;
    tri_edges(a, vload(v1), vload(v2), &e1, &e2);
    if (!tri_hit(vload(o), vload(d), tmax, a, e1, e2, t)) return 0;
    v3 nn = tri_normal(e1, e2, vload(d));
    n[0] = nn.x; n[1] = nn.y; n[2] = nn.z;
    return 1;
}

OR_EXPORT int or_sphere_hit(const float o[3], const float d[3], float tmax, const float c[3], float r,
                            float *t, float n[3])
{
    if (!sphere_hit(vload(o), vload(d), tmax, vload(c), r, t)) return 0;
    v3 nn = sphere_normal(vload(o), vload(d), *t, vload(c), r);
    n[0] = nn.x; n[1] = nn.y; n[2] = nn.z;
    return 1;
}

OR_EXPORT int or_slab(const float lo[3], const float hi[3], const float o[3], const float d[3],
                      float tmax, float *t0, float *t1)
{
    return slab(lo, hi, vload(o), vload(d), tmax, t0, t1);
}

OR_EXPORT void or_camera_ray(const or_camera *cam, const or_frame *fr, uint32_t p, uint32_t s,
                             float o[3], float d[3])
{
    v3 oo, dd;
    camera_ray(cam, fr, p, s, &oo, &dd);
    o[0] = oo.x; o[1] = oo.y; o[2] = oo.z;
    d[0] = dd.x; d[1] = dd.y; d[2] = dd.z;
}

OR_EXPORT void or_cosine_dir(const float n[3], uint64_t seed, uint32_t p, uint32_t s, uint32_t depth,
                             uint32_t purpose, uint32_t subhi, float out[3])
{
    v3 r = cosine_dir(vload(n), seed, p, s, depth, purpose, subhi);
    out[0] = r.x; out[1] = r.y; out[2] = r.z;
}

OR_EXPORT void or_iso_dir(uint64_t seed, uint32_t p, uint32_t s, uint32_t depth, float out[3])
{
    v3 r = iso_dir(seed, p, s, depth);
    out[0] = r.x; out[1] = r.y; out[2] = r.z;
}

OR_EXPORT float or_pln(float x) { return pln(x); }

/* The renderer's RNG call sites (P1 counter layout; pinned against or_philox). */
OR_EXPORT void or_ao_dir(const float n[3], uint64_t seed, uint32_t p, uint32_t s, uint32_t depth, int k,
                         float out[3])
{
    v3 r = ao_dir(vload(n), seed, p, s, depth, k);
    out[0] = r.x; out[1] = r.y; out[2] = r.z;
}

OR_EXPORT void or_bounce_dir(const float n[3], uint64_t seed, uint32_t p, uint32_t s, uint32_t depth,
                             float out[3])
{
    v3 r = bounce_dir(vload(n), seed, p, s, depth);
    out[0] = r.x; out[1] = r.y; out[2] = r.z;
}

/* u_i of volume sample i of a ray of kind 0 path / 1 shadow / 2 AO k. */
OR_EXPORT float or_vol_u(uint64_t seed, uint32_t p, uint32_t s, uint32_t depth, int kind, int k, int64_t i)
{
    VolKey v = vol_key(seed, p, s, depth, kind, k);
    return vol_u(v.seed, v.p, v.s, v.depth, v.purpose, v.subhi, i);
}

OR_EXPORT void or_tf_eval(const float *tf, float lo, float hi, float dscale, float s, float rgba[4])
{
    tf_eval(tf, lo, hi, dscale, s, rgba);
}

/* Trilinear sample of part `pt` (a brick) at world point p; returns 0 if not owned. */
OR_EXPORT int or_brick_sample(const or_part *pt, const float p[3], float *value)
{
    OBrick b;
    memset(&b, 0, sizeof(b));
    for (int c = 0; c < 3; ++c) {
        b.gd[c] = pt->gdims[c]; b.lo[c] = pt->cell_lo[c]; b.hi[c] = pt->cell_hi[c];
        b.O[c] = pt->origin[c]; b.h[c] = pt->spacing[c];
    }
    b.vox = pt->voxels;
    v3 g = grid_coord(&b, vload(p));
    if (!brick_owns(&b, g)) return 0;
    *value = brick_trilinear(&b, g);
    return 1;
}

/* Brute-force closest hit over ALL prims of the union (no BVH): the P9 definition. */
OR_EXPORT void or_brute_closest(const OScene *sc, const float o[3], const float d[3], float tmax,
                                float *t, uint32_t *id)
{
    OHit best;
    hit_none(&best);
    for (int64_t i = 0; i < sc->nprims; ++i) prim_closest(&sc->prims[i], vload(o), vload(d), tmax, &best);
    *t = best.t; *id = best.id;
}

OR_EXPORT void or_bvh_closest(const OScene *sc, const float o[3], const float d[3], float tmax,
                              float *t, uint32_t *id)
{
    OHit best;
    hit_none(&best);
    bvh_closest(&sc->ubvh, sc->prims, vload(o), vload(d), tmax, &best);
    *t = best.t; *id = best.id;
}

OR_EXPORT int or_brute_any(const OScene *sc, const float o[3], const float d[3], float tmax)
{
    for (int64_t i = 0; i < sc->nprims; ++i) if (prim_any(&sc->prims[i], vload(o), vload(d), tmax)) return 1;
    return 0;
}

OR_EXPORT int or_bvh_any(const OScene *sc, const float o[3], const float d[3], float tmax)
{
    return bvh_any(&sc->ubvh, sc->prims, vload(o), vload(d), tmax);
}
