// common.cuh -- device-side building blocks of the product path (sm_100a).
//
// Arithmetic follows the pinned reading of the paper-silent parts (
// DESIGN.md "Readings"): IEEE binary32 round-to-nearest, no FMA contraction in anything
// that decides a result (this translation unit is compiled with -fmad=false; explicit
// __fmaf_rn appears ONLY in conservative BVH box tests, which decide what to skip, never
// a result), IEEE division/sqrt (-prec-div/-prec-sqrt default), denormals kept.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/dpr.h"

namespace dpr {

// ---------------------------------------------------------------------------------------
// Ray records in HBM (SURVEY 8(a) record layouts).  Path ray 64 B, occlusion ray 48 B,
// both float4-aligned for 128-bit loads/stores.
//   path: a=(o.xyz, bestT) b=(d.xyz, bestId) c=(beta.rgb, pixel) e=(n.xyz | vol rgb, meta)
//         meta = sample | depth<<16
//   occl: a=(o.xyz, tmax)  b=(d.xyz, pixel)  c=(contrib.rgb, meta)
//         meta = sample | depth<<16 | slot<<24, slot 0 = shadow, 1+k = AO ray k
// ---------------------------------------------------------------------------------------
struct PathRec { float4 a, b, c, e; };
struct OcclRec { float4 a, b, c; };

constexpr uint32_t NO_HIT = 0xffffffffu;
constexpr uint32_t VOL_BIT = 0x80000000u;
constexpr uint32_t SPHERE_BIT = 0x80000000u;  // in a prim record's id word

enum Kind { K_PATH = 0, K_SHADOW = 1, K_AO = 2 };
enum Purpose { PUR_CAMERA = 0, PUR_LENS = 1, PUR_AO = 2, PUR_BOUNCE = 3, PUR_VOL_PATH = 4,
               PUR_VOL_SHADOW = 5, PUR_VOL_AO = 6, PUR_ISO = 7 };

// Per-kernel work counters (kc[0] = k_trace_path, kc[1] = k_trace_occl): the inputs of the
// algorithmic-byte count of DESIGN.md "Roofline".
struct KernelCounters {
    unsigned long long nodes, tris, sphs, vols, rin, rout_path, rout_occl, pad;
};
// Per-rank device counters (one block in device memory, zeroed per frame).
struct Counters {
    unsigned long long V[3];
    unsigned long long S[3][DPR_MAX_RANKS];
    unsigned long long gen[3];
    KernelCounters kc[2];
    // records this rank appended to each destination's queue, per kind (0 path, 1 occlusion),
    // self included (cumulative over the frame): a receiver's queue is complete only when every
    // sender has finished its step, so step boundaries exchange these, never a peer's tail
    unsigned long long app[2][DPR_MAX_RANKS];
    unsigned int overflow;  // bit0 queue overflow, bit1 traversal stack overflow
    unsigned int pad;
};

// ---------------------------------------------------------------------------------------
// float3 helpers with the pinned evaluation order: dot = (x*x' + y*y') + z*z'.
// ---------------------------------------------------------------------------------------
struct f3 { float x, y, z; };
__device__ __forceinline__ f3 mk(float x, float y, float z) { f3 r; r.x = x; r.y = y; r.z = z; return r; }
__device__ __forceinline__ f3 sub(f3 a, f3 b) { return mk(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ f3 mul(f3 a, f3 b) { return mk(a.x * b.x, a.y * b.y, a.z * b.z); }
__device__ __forceinline__ f3 scale(f3 a, float s) { return mk(a.x * s, a.y * s, a.z * s); }
__device__ __forceinline__ float dot(f3 a, f3 b) { float r = a.x * b.x + a.y * b.y; return r + a.z * b.z; }
__device__ __forceinline__ f3 cross(f3 a, f3 b) {
    return mk(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ f3 xyz(float4 v) { return mk(v.x, v.y, v.z); }
__device__ __forceinline__ float comp(f3 a, int c) { return c == 0 ? a.x : (c == 1 ? a.y : a.z); }

// ---------------------------------------------------------------------------------------
// P1: Philox4x32-10 (Salmon et al. SC'11).  Counter (p, s, depth<<8|purpose, sub),
// key (seed lo, seed hi).  u = (x>>8) * 2^-24.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                        uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
        uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    return make_uint4(c0, c1, c2, c3);
}
__device__ __forceinline__ float u01(uint32_t x) { return __uint2float_rn(x >> 8) * 0x1p-24f; }
__device__ __forceinline__ uint4 rng4(uint64_t seed, uint32_t p, uint32_t s, uint32_t depth,
                                      uint32_t purpose, uint32_t sub) {
    return philox(p, s, (depth << 8) | purpose, sub, (uint32_t)seed, (uint32_t)(seed >> 32));
}

// ---------------------------------------------------------------------------------------
// P3 Moeller-Trumbore (double-sided, no epsilon), P4 sphere, orientation.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ bool tri_hit(f3 o, f3 d, float tmax, f3 v0, f3 e1, f3 e2, float &t) {
    f3 pv = cross(d, e2);
    float det = dot(e1, pv);
    if (det == 0.0f) return false;
    f3 tv = sub(o, v0);
    float un = dot(tv, pv);
    // Exact early rejects before the IEEE division (they only skip cases the pinned test
    // rejects): u = un*(1/det) has the sign of un*det when it cannot
    // underflow to zero, and |u| > 1 when |un| > |det|*(1+2^-19).
    if (fabsf(un) >= 0x1p-100f && fabsf(det) <= 0x1p40f &&
        ((__float_as_uint(un) ^ __float_as_uint(det)) & 0x80000000u))
        return false;
    if (fabsf(un) > fabsf(det) * 1.0000019f) return false;
    float inv = 1.0f / det;
    float u = un * inv;
    if (u < 0.0f || u > 1.0f) return false;
    f3 qv = cross(tv, e1);
    float v = dot(d, qv) * inv;
    if (v < 0.0f || u + v > 1.0f) return false;
    t = dot(e2, qv) * inv;
    return t > 0.0f && t < tmax;
}

__device__ __forceinline__ f3 orient(f3 n, f3 d) {
    if (dot(n, d) > 0.0f) return mk(-n.x, -n.y, -n.z);
    return n;
}

__device__ __forceinline__ f3 tri_normal(f3 e1, f3 e2, f3 d) {
    f3 ng = cross(e1, e2);
    float len = sqrtf(dot(ng, ng));
    return orient(mk(ng.x / len, ng.y / len, ng.z / len), d);
}

// P4 with reading R-SPHERE: disc = r^2 - |f - b d|^2 (cancellation-free; the
// b^2 - (|f|^2 - r^2) form reports hits outside a small distant sphere's bounding box).
__device__ __forceinline__ bool sphere_hit(f3 o, f3 d, float tmax, f3 c, float r, float &t) {
    f3 f = sub(o, c);
    float b = dot(f, d);
    f3 q = mk(f.x - b * d.x, f.y - b * d.y, f.z - b * d.z);
    float disc = r * r - dot(q, q);
    if (disc < 0.0f) return false;
    float sq = sqrtf(disc);
    t = -b - sq;
    if (!(t > 0.0f)) t = -b + sq;
    return t > 0.0f && t < tmax;
}

__device__ __forceinline__ f3 sphere_normal(f3 o, f3 d, float t, f3 c, float r) {
    f3 p = mk(o.x + t * d.x, o.y + t * d.y, o.z + t * d.z);
    return orient(mk((p.x - c.x) / r, (p.y - c.y) / r, (p.z - c.z) / r), d);
}

// ---------------------------------------------------------------------------------------
// P8 slab test against a rank box (exact, minNum semantics of fminf/fmaxf).
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ bool slab(const float *lo, const float *hi, f3 o, f3 d, float tmax,
                                     float &t0, float &t1) {
    float nr[3], fr[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        float inv = 1.0f / comp(d, c);
        float ta = (lo[c] - comp(o, c)) * inv;
        float tb = (hi[c] - comp(o, c)) * inv;
        nr[c] = fminf(ta, tb);
        fr[c] = fmaxf(ta, tb);
    }
    t0 = fmaxf(fmaxf(fmaxf(0.0f, nr[0]), nr[1]), nr[2]);
    t1 = fminf(fminf(fminf(tmax, fr[0]), fr[1]), fr[2]);
    return t0 <= t1;
}

// Routing table: N padded rank boxes (lo xyz, hi xyz) + nonempty flags (P8).
struct Routing {
    int nranks, self;
    float box[DPR_MAX_RANKS][6];
    int nonempty[DPR_MAX_RANKS];
};

// First candidate = min key (t0_r, r) over candidates (P8, new rays).  -1 if none.
__device__ __forceinline__ int first_candidate(const Routing &R, f3 o, f3 d, float tmax) {
    int best = -1;
    float bt = 0.0f;
    for (int r = 0; r < R.nranks; ++r) {
        if (!R.nonempty[r]) continue;
        float t0, t1;
        if (!slab(R.box[r], R.box[r] + 3, o, d, tmax, t0, t1)) continue;
        if (best < 0 || t0 < bt) { best = r; bt = t0; }
    }
    return best;
}

// Next candidate after tracing at rank c: min key > (t0_c, c) with t0_r <= tbound (P8).
__device__ __forceinline__ int next_candidate(const Routing &R, int c, f3 o, f3 d, float tmax,
                                              float tbound) {
    if (R.nranks == 1) return -1;
    float tc, t1c;
    slab(R.box[c], R.box[c] + 3, o, d, __int_as_float(0x7f800000), tc, t1c);
    int best = -1;
    float bt = 0.0f;
    for (int r = 0; r < R.nranks; ++r) {
        if (r == c || !R.nonempty[r]) continue;
        float t0, t1;
        if (!slab(R.box[r], R.box[r] + 3, o, d, tmax, t0, t1)) continue;
        if (!(t0 <= tbound)) continue;
        bool gt = t0 > tc || (t0 == tc && r > c);
        if (!gt) continue;
        if (best < 0 || t0 < bt) { best = r; bt = t0; }
    }
    return best;
}

// ---------------------------------------------------------------------------------------
// P7 directions (rejection sampling; no transcendentals).
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ f3 cosine_dir(f3 n, uint64_t seed, uint32_t p, uint32_t s,
                                         uint32_t depth, uint32_t purpose, uint32_t subhi) {
    for (uint32_t a = 0; a < 16; ++a) {
        uint4 r = rng4(seed, p, s, depth, purpose, subhi | a);
        float x = 2.0f * u01(r.x) - 1.0f;
        float y = 2.0f * u01(r.y) - 1.0f;
        float r2 = x * x + y * y;
        if (!(r2 < 1.0f)) continue;
        float z = sqrtf(1.0f - r2);
        float sg = copysignf(1.0f, n.z);
        float aa = -1.0f / (sg + n.z);
        float b = (n.x * n.y) * aa;
        f3 t1 = mk(1.0f + ((sg * n.x) * n.x) * aa, sg * b, -sg * n.x);
        f3 t2 = mk(b, sg + (n.y * n.y) * aa, -n.y);
        return mk((x * t1.x + y * t2.x) + z * n.x, (x * t1.y + y * t2.y) + z * n.y,
                  (x * t1.z + y * t2.z) + z * n.z);
    }
    return n;
}

__device__ __forceinline__ f3 iso_dir(uint64_t seed, uint32_t p, uint32_t s, uint32_t depth) {
    for (uint32_t a = 0; a < 16; ++a) {
        uint4 r = rng4(seed, p, s, depth, PUR_ISO, a);
        f3 v = mk(2.0f * u01(r.x) - 1.0f, 2.0f * u01(r.y) - 1.0f, 2.0f * u01(r.z) - 1.0f);
        float r2 = dot(v, v);
        if (!(r2 > 0.0f && r2 < 1.0f)) continue;
        float l = sqrtf(r2);
        return mk(v.x / l, v.y / l, v.z / l);
    }
    return mk(0.0f, 0.0f, 1.0f);
}

// ---------------------------------------------------------------------------------------
// Device world of one rank.
// ---------------------------------------------------------------------------------------
// Leaf size bound of the wide-BVH collapse (binary subtrees with <= LEAF_MAX prims become
// leaf children).
#ifndef DPR_FILL_LEAVES
#define DPR_FILL_LEAVES 1
#endif
#ifndef DPR_LEAF_MAX
#define DPR_LEAF_MAX 4
#endif
constexpr int LEAF_MAX = DPR_LEAF_MAX;  // <= 4 (2-bit count in the wide-node meta)


// Prim record in BVH leaf order, 48 B (3 x float4):
//   tri:    (v0.xyz, id) (e1.xyz, 0) (e2.xyz, 0)     id = local index
//   sphere: (c.xyz, id|SPHERE_BIT) (r, 0, 0, 0) (unused)
struct BrickDev {
    int gd[3];              // global grid points per axis
    int lo[3], hi[3];       // cell_lo, cell_hi (stored voxels [lo, hi] inclusive)
    int mc_dims[3];         // macrocell grid dims (16^3 cells each)
    float O[3], h[3];       // global origin / spacing
    float box_lo[3], box_hi[3];
    const float *vox;       // x fastest
    const uint8_t *mc;      // 1 = some sample in the macrocell may have alpha > 0
    const uint8_t *mcd;     // Chebyshev distance (macrocells, capped at MC_DIST_CAP) to the
                            // nearest macrocell with mc = 1 (0: mc = 1 here)
    const float4 *tf;       // 256 rgba
    float tf_lo, tf_hi, dscale;
    float tf_rd;            // 1/(tf_hi - tf_lo) when that difference is a power of two, else 0
};

// P10 grid coordinate g = (p - O) / h (IEEE division, global origin / spacing).  (A division-
// free form, q1 = fma(fma(-q0, h, x), RN(1/h), q0), checked exhaustively equal to x / h for
// every binary32 |x| in [2^-100, 4] at configs[2]'s h, ran slower in the march kernels at the
// 64-register cap: 2.85 vs 2.76 ms, r02.)
__device__ __forceinline__ f3 grid_coord(const BrickDev &B, f3 pt) {
    return mk((pt.x - B.O[0]) / B.h[0], (pt.y - B.O[1]) / B.h[1], (pt.z - B.O[2]) / B.h[2]);
}

constexpr int MC_SIZE = 16;
constexpr int MC_DIST_PASSES = 8, MC_DIST_CAP = MC_DIST_PASSES + 1;  // exact below the cap
constexpr int MAX_BRICKS = 8;

// Compressed 8-wide node (80 B; layout in the spirit of Ylitie, Karras, Laine 2017
// "Efficient incoherent ray traversal on GPUs through compressed wide BVHs"):
//   w0 = (p.x, p.y, p.z, bits ex | ey<<8 | ez<<16 | imask<<24)   origin + per-axis 2^(e-127)
//   w1 = (child_base | leafmask[0..3] << 28, prim_base | leafmask[4..7] << 28, meta[0..3], meta[4..7])
//   w2 = (qlo_x[0..3], qlo_x[4..7], qlo_y[0..3], qlo_y[4..7])
//   w3 = (qlo_z[0..3], qlo_z[4..7], qhi_x[0..3], qhi_x[4..7])
//   w4 = (qhi_y[0..3], qhi_y[4..7], qhi_z[0..3], qhi_z[4..7])
// child box = p + q * 2^(e-127) (quantised outward from already-padded boxes: conservative).
// imask bit s: slot s is an internal child, stored at child_base + popc(imask & ((1<<s)-1)).
// meta[s] for a leaf: 0x80 | (count-1)<<5 | offset (prims prim_base+offset .. +count-1);
// 0 = empty slot.  Slots are assigned by octant so that visiting s' = 0..7 with
// slot = s' ^ octant(ray) is approximately front to back.
struct WNode { float4 w0; uint4 w1, w2, w3, w4; };

struct WorldDev {
    uint32_t prmt_hi;  // 0x4b00 (2^23 float pattern for byte decode), passed at run time so that
                       // ptxas keeps the PRMT selector as the immediate operand
    const WNode *wnodes;
    const float4 *prims;
    const float4 *prims_in;  // the same records in input order (index = local id): the normal of a
                             // hit found by the cooperative tests, which report (t, id)
    int64_t nprims;
    int64_t nnodes;         // wide nodes (bounds checks of DPR_CHECKS builds)
    uint32_t id_base;       // global id of local prim 0 (P12)
    int nbricks;
    float amax;     // delta tracking majorant (max TF alpha over ALL ranks' bricks; R-DELTA)
    float gdom[6];  // global grid domain O .. O + (gdims-1) h (tentative points start there)
    BrickDev bricks[MAX_BRICKS];
};

// Global part table for albedo lookup at the resolving rank (id ranges sorted).
struct PartTable {
    int n;
    const uint32_t *id_lo;   // first global id of each part (ascending)
    const float4 *albedo;
};

__device__ __forceinline__ f3 part_albedo(const PartTable &T, uint32_t id) {
    int lo = 0, hi = T.n - 1;
    while (lo < hi) {  // last part with id_lo <= id
        int mid = (lo + hi + 1) >> 1;
        if (__ldg(T.id_lo + mid) <= id) lo = mid; else hi = mid - 1;
    }
    float4 a = __ldg(T.albedo + lo);
    return mk(a.x, a.y, a.z);
}

// ---------------------------------------------------------------------------------------
// P10 volume sampling helpers.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ float lerpf(float a, float b, float w) { return a + w * (b - a); }

// x / h with the division replaced by a multiplication by r = 1/h when h is a power of two
// (r != 0, set by the host): x/h and x*r are then the same real number, rounded once, so the
// result is bit-identical to the IEEE division (incl. subnormal, overflow, signed-zero cases)
__device__ __forceinline__ float div_pow2(float x, float h, float r) { return r != 0.0f ? x * r : x / h; }

__device__ __forceinline__ float tf_alpha_rgb(const BrickDev &B, float s, f3 *rgb) {
    float x = fminf(fmaxf(div_pow2(s - B.tf_lo, B.tf_hi - B.tf_lo, B.tf_rd), 0.0f), 1.0f) * 255.0f;
    int j = (int)floorf(x);
    if (j > 254) j = 254;
    float w = x - (float)j;
    float4 a = __ldg(B.tf + j), b = __ldg(B.tf + j + 1);
    if (rgb) *rgb = mk(a.x + w * (b.x - a.x), a.y + w * (b.y - a.y), a.z + w * (b.z - a.z));
    return fminf(1.0f, (a.w + w * (b.w - a.w)) * B.dscale);
}

__device__ __forceinline__ float sample_t(int64_t i, float dt) { return ((float)i + 0.5f) * dt; }

}  // namespace dpr
