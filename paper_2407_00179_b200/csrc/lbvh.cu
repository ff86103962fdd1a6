// lbvh.cu -- per-rank acceleration-structure build on the GPU.
//
// The paper's method needs only "negligible pre-processing" (S2.2): each rank
// builds a local structure over its own parts.  B200 has no RT cores, so the
// structure and its traversal are hand-written: a linear BVH (Karras 2012; built bottom-up in
// one pass after Apetrei 2014), collapsed into a compressed 8-wide BVH:
//   1. k_part_prims: prim records + exact AABBs (min/max, no rounding) of every part in one
//      launch (one block per chunk), and in the same pass each part's and the rank's box and
//      centroid box (order-preserving integer atomics after a block reduction)
//   2. k_morton_h: 30-bit Morton code of the centroid (10 bits per axis) in a 32-bit key,
//      one radix tile per block, with the first pass's tile histogram
//   3. LSD radix sort of (key u32, index u32): 4 passes of 8-bit digits, warp-ranked stable
//      scatter staged in shared memory (k_tile_hist, k_scan_digits, k_scatter_w)
//   4. k_split_delta + k_agglo_p: agglomerative radix tree (persistent, 64-bit exchange words),
//      packed 32-byte node records (k_karras + k_refit and PLOC selectable)
//   5. k_collapse_r: compressed 8-wide nodes (WNode) by greedy opening of the largest child,
//      child boxes padded outward then quantised outward (conservative traversal), octant
//      slots by a lazy greedy; one BFS level per launch
//   6. k_permute_prims: prim records into wide-leaf order
//   7. k_macrocells: per 16^3 macrocell "alpha may be > 0" flags for exact empty-space
//      skipping in bricks
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"

namespace dpr {

static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

#ifndef DPR_MORTON_BITS
#define DPR_MORTON_BITS 10  // per axis; 30-bit codes in 32-bit keys (r01: 21 bits/axis in 64-bit keys
                            // traced no faster and doubled the sort's key traffic)
#endif
static_assert(DPR_MORTON_BITS <= 10, "Morton keys are 32-bit");

__device__ __forceinline__ int f2ord(float f) {
    int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float ord2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

// ---------------------------------------------------------------------------------------
// Prim records + exact AABBs, with the part's box and centroid box reduced in the same pass:
// bounds[0..5] = box lo/hi, bounds[6..11] = centroid lo/hi (order-preserving ints), merged
// into the part's slot and the global slot by one warp reduction + atomics per warp.
struct BoundsAcc {
    int v[12];
    __device__ __forceinline__ void init() {
        for (int c = 0; c < 3; ++c) {
            v[c] = 0x7fffffff; v[3 + c] = (int)0x80000000;
            v[6 + c] = 0x7fffffff; v[9 + c] = (int)0x80000000;
        }
    }
    __device__ __forceinline__ void add(f3 lo, f3 hi) {
        float l[3] = {lo.x, lo.y, lo.z}, h[3] = {hi.x, hi.y, hi.z};
        for (int c = 0; c < 3; ++c) {
            float cen = (l[c] + h[c]) * 0.5f;
            v[c] = min(v[c], f2ord(l[c]));
            v[3 + c] = max(v[3 + c], f2ord(h[c]));
            v[6 + c] = min(v[6 + c], f2ord(cen));
            v[9 + c] = max(v[9 + c], f2ord(cen));
        }
    }
    // block-wide reduction (warp shuffles, then across warps in shared memory), then one
    // atomic per bound word into the part's slot and the global slot
    __device__ __forceinline__ void block_flush(int *bounds, int *bounds_global) {
        __shared__ int sm[32][12];
        for (int k = 0; k < 12; ++k) {
            bool isMin = (k % 6) < 3;
            for (int o = 16; o > 0; o >>= 1) {
                int w = __shfl_xor_sync(0xffffffffu, v[k], o);
                v[k] = isMin ? min(v[k], w) : max(v[k], w);
            }
        }
        const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
        if ((threadIdx.x & 31) == 0)
            for (int k = 0; k < 12; ++k) sm[warp][k] = v[k];
        __syncthreads();
        if (threadIdx.x < 12) {
            const int k = threadIdx.x;
            const bool isMin = (k % 6) < 3;
            int x = sm[0][k];
            for (int w = 1; w < nw; ++w) x = isMin ? min(x, sm[w][k]) : max(x, sm[w][k]);
            if (isMin) { atomicMin(&bounds[k], x); atomicMin(&bounds_global[k], x); }
            else { atomicMax(&bounds[k], x); atomicMax(&bounds_global[k], x); }
        }
    }
};

// One block per chunk of one part (all parts of the rank in a single launch): triangle
// records (v0, e1, e2; triangle indices validated here, on the GPU) or sphere records, their
// exact AABBs, and the part's box / centroid box.
__global__ void __launch_bounds__(256) k_part_prims(const PrimChunk *__restrict__ chunks, float4 *prims,
                                                    float4 *blo, float4 *bhi, int *bounds, int *bad_index) {
    const PrimChunk c = chunks[blockIdx.x];
    BoundsAcc acc;
    acc.init();
    for (int j = threadIdx.x; j < c.count; j += blockDim.x) {
        const int64_t t = c.start + j, g = (int64_t)c.g0 + j;
        f3 lo, hi;
        if (c.kind == DPR_PART_TRIANGLES) {
            const float *verts = (const float *)c.src;
            int64_t i0 = c.idx[3 * t], i1 = c.idx[3 * t + 1], i2 = c.idx[3 * t + 2];
            if (i0 < 0 || i0 >= c.nv || i1 < 0 || i1 >= c.nv || i2 < 0 || i2 >= c.nv) {
                atomicOr(bad_index, 1);
                i0 = i1 = i2 = 0;
            }
            f3 v0 = mk(verts[3 * i0], verts[3 * i0 + 1], verts[3 * i0 + 2]);
            f3 v1 = mk(verts[3 * i1], verts[3 * i1 + 1], verts[3 * i1 + 2]);
            f3 v2 = mk(verts[3 * i2], verts[3 * i2 + 1], verts[3 * i2 + 2]);
            f3 e1 = sub(v1, v0), e2 = sub(v2, v0);
            if (!(isfinite(v0.x) && isfinite(v0.y) && isfinite(v0.z) && isfinite(v1.x) && isfinite(v1.y) &&
                  isfinite(v1.z) && isfinite(v2.x) && isfinite(v2.y) && isfinite(v2.z)))
                atomicOr(bad_index, 2);
            // reading R-DEGEN: a zero binary32 cross(e1, e2) (no area, no normal) is stored as
            // e1 = e2 = 0, which P3's det == 0 test always rejects
            const f3 ng = cross(e1, e2);
            if (ng.x == 0.0f && ng.y == 0.0f && ng.z == 0.0f) e1 = e2 = mk(0.0f, 0.0f, 0.0f);
            prims[3 * g + 0] = make_float4(v0.x, v0.y, v0.z, __uint_as_float((uint32_t)g));
            prims[3 * g + 1] = make_float4(e1.x, e1.y, e1.z, 0.0f);
            prims[3 * g + 2] = make_float4(e2.x, e2.y, e2.z, 0.0f);
            lo = mk(fminf(fminf(v0.x, v1.x), v2.x), fminf(fminf(v0.y, v1.y), v2.y), fminf(fminf(v0.z, v1.z), v2.z));
            hi = mk(fmaxf(fmaxf(v0.x, v1.x), v2.x), fmaxf(fmaxf(v0.y, v1.y), v2.y), fmaxf(fmaxf(v0.z, v1.z), v2.z));
        } else {
            const float4 s = ((const float4 *)c.src)[t];
            if (!(isfinite(s.x) && isfinite(s.y) && isfinite(s.z) && isfinite(s.w) && s.w > 0.0f))
                atomicOr(bad_index, 2);  // radius must be > 0 and finite (dpr.h)
            prims[3 * g + 0] = make_float4(s.x, s.y, s.z, __uint_as_float((uint32_t)g | SPHERE_BIT));
            prims[3 * g + 1] = make_float4(s.w, 0.0f, 0.0f, 0.0f);
            prims[3 * g + 2] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            lo = mk(s.x - s.w, s.y - s.w, s.z - s.w);
            hi = mk(s.x + s.w, s.y + s.w, s.z + s.w);
        }
        blo[2 * g] = make_float4(lo.x, lo.y, lo.z, 0.0f);  // interleaved: bhi == blo + 1
        bhi[2 * g] = make_float4(hi.x, hi.y, hi.z, 0.0f);
        acc.add(lo, hi);
    }
    acc.block_flush(bounds + 12 * c.slot, bounds);
}

__device__ __forceinline__ uint32_t expand10(uint32_t v) {  // bit i -> bit 3i (10 bits)
    v &= 0x3ffu;
    v = (v | v << 16) & 0x030000ffu;
    v = (v | v << 8) & 0x0300f00fu;
    v = (v | v << 4) & 0x030c30c3u;
    v = (v | v << 2) & 0x09249249u;
    return v;
}


// ---------------------------------------------------------------------------------------
// LSD radix sort, 8-bit digits.
// ---------------------------------------------------------------------------------------
constexpr int RS_THREADS = 256;
#ifndef DPR_RS_ITEMS
#define DPR_RS_ITEMS 8  // r02 sweep (warp-ranked scatter, configs[3] build): 4 14.28, 6 13.76, 8 13.57, 10 13.63, 12 13.84, 16 13.72 ms
#endif
constexpr int RS_ITEMS = DPR_RS_ITEMS;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;


// Morton codes of one radix tile per block (RS_TILE keys), fused with the sort's histograms:
// the tile's digit-0 counts (the first pass's tile histogram) and all digits' totals (constant-
// digit detection and the passes' digit totals), so neither needs its own read of the keys.
__global__ void __launch_bounds__(RS_THREADS) k_morton_h(const float4 *__restrict__ blo, const float4 *__restrict__ bhi,
                                                          int64_t n, const int *__restrict__ bounds, mkey_t *keys,
                                                          uint32_t *vals, uint32_t *tile_hist0, int ntiles,
                                                          unsigned long long *hist_all) {
    __shared__ unsigned int h[MKEY_DIGITS][256];
    for (int i = threadIdx.x; i < MKEY_DIGITS * 256; i += blockDim.x) (&h[0][0])[i] = 0;
    float mn[3], sc[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        mn[a] = ord2f(bounds[6 + a]);
        sc[a] = ord2f(bounds[9 + a]) - mn[a];
    }
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * RS_TILE;
    for (int j = 0; j < RS_ITEMS; ++j) {
        const int64_t i = base + j * RS_THREADS + threadIdx.x;
        if (i >= n) break;
        const float4 lo = blo[2 * i], hi = bhi[2 * i];
        const float c[3] = {(lo.x + hi.x) * 0.5f, (lo.y + hi.y) * 0.5f, (lo.z + hi.z) * 0.5f};
        uint32_t q[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const float ext = sc[a];
            const float cells = (float)(1u << DPR_MORTON_BITS);
            float x = ext > 0.0f ? (c[a] - mn[a]) / ext * cells : 0.0f;
            x = fminf(fmaxf(x, 0.0f), cells - 1.0f);
            q[a] = (uint32_t)x;
        }
        const mkey_t k = (expand10(q[0]) << 2) | (expand10(q[1]) << 1) | expand10(q[2]);
        keys[i] = k;
        vals[i] = (uint32_t)i;
        if (hist_all) {
#pragma unroll
            for (int p = 1; p < MKEY_DIGITS; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 255], 1u);
        }
        atomicAdd(&h[0][k & 255], 1u);
    }
    __syncthreads();
    tile_hist0[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[0][threadIdx.x];
    if (hist_all) {
#pragma unroll
        for (int p = 0; p < MKEY_DIGITS; ++p)
            if (h[p][threadIdx.x]) atomicAdd(&hist_all[p * 256 + threadIdx.x], (unsigned long long)h[p][threadIdx.x]);
    }
}

__global__ void k_tile_hist(const mkey_t *__restrict__ keys, int64_t n, int shift,
                            uint32_t *tile_hist, int ntiles) {
    __shared__ unsigned int h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    int64_t base = (int64_t)blockIdx.x * RS_TILE;
    for (int j = 0; j < RS_ITEMS; ++j) {
        int64_t i = base + j * RS_THREADS + threadIdx.x;
        if (i < n) atomicAdd(&h[(keys[i] >> shift) & 255], 1u);
    }
    __syncthreads();
    tile_hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// Per-digit exclusive scan over tiles: one block per digit d scans tile_hist[d][0..ntiles)
// in place and writes the digit total.  (Replaces a single-block scan of all 256*ntiles
// counters, which cost ~0.5 ms per pass at 10M keys.)
__global__ void __launch_bounds__(1024) k_scan_digits(uint32_t *tile_hist, int ntiles, uint32_t *digit_tot) {
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t carry;
    uint32_t *row = tile_hist + (int64_t)blockIdx.x * ntiles;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < ntiles; base += 1024) {
        int i = base + threadIdx.x;
        uint32_t v = i < ntiles ? row[i] : 0;
        uint32_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sums[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = warp_sums[lane];
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            warp_sums[lane] = w;
        }
        __syncthreads();
        uint32_t excl = carry + (warp ? warp_sums[warp - 1] : 0) + x - v;
        if (i < ntiles) row[i] = excl;
        __syncthreads();
        if (threadIdx.x == 1023) carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) digit_tot[blockIdx.x] = carry;
}

__global__ void __launch_bounds__(RS_THREADS)
k_scatter(const mkey_t *__restrict__ kin, const uint32_t *__restrict__ vin, mkey_t *kout,
          uint32_t *vout, int64_t n, int shift, const uint32_t *__restrict__ tile_off, int ntiles,
          const uint32_t *__restrict__ digit_tot) {
    __shared__ uint32_t wcnt[RS_THREADS / 32][256];
    __shared__ uint32_t run[256];
    __shared__ uint32_t goff[256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    {  // exclusive scan of the 256 digit totals (thread = digit)
        uint32_t v = digit_tot[threadIdx.x], x = v;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wcnt[0][warp] = x;
        __syncthreads();
        uint32_t wp = 0;
        for (int w = 0; w < warp; ++w) wp += wcnt[0][w];
        goff[threadIdx.x] = wp + x - v + tile_off[(int64_t)threadIdx.x * ntiles + blockIdx.x];
        __syncthreads();
    }
    run[threadIdx.x] = 0;
    const unsigned lt = (1u << lane) - 1u;
    int64_t base = (int64_t)blockIdx.x * RS_TILE;
    for (int j = 0; j < RS_ITEMS; ++j) {
        for (int w = 0; w < RS_THREADS / 32; ++w) wcnt[w][threadIdx.x] = 0;
        __syncthreads();
        int64_t i = base + j * RS_THREADS + threadIdx.x;
        bool valid = i < n;
        mkey_t k = valid ? kin[i] : 0;
        uint32_t v = valid ? vin[i] : 0;
        int d = valid ? (int)((k >> shift) & 255) : 256 + lane;  // invalid lanes: unique groups
        unsigned peers = __match_any_sync(0xffffffffu, d);
        uint32_t rank = __popc(peers & lt);
        if (valid && rank == 0) wcnt[warp][d] = __popc(peers);
        __syncthreads();
        {  // thread = digit: prefix over warps
            uint32_t r = run[threadIdx.x];
            for (int w = 0; w < RS_THREADS / 32; ++w) {
                uint32_t c = wcnt[w][threadIdx.x];
                wcnt[w][threadIdx.x] = r;
                r += c;
            }
            run[threadIdx.x] = r;
        }
        __syncthreads();
        if (valid) {
            uint32_t pos = goff[d] + wcnt[warp][d] + rank;
            kout[pos] = k;
            vout[pos] = v;
        }
        __syncthreads();
    }
}

// Coalesced variant (default): the tile is first ranked into digit order in shared memory
// (stable: item order within a digit is kept), then written out digit run by digit run, so
// consecutive threads store to consecutive addresses of a bucket instead of 256 scattered
// buckets per warp store.
__global__ void __launch_bounds__(RS_THREADS)
k_scatter_c(const mkey_t *__restrict__ kin, const uint32_t *__restrict__ vin, mkey_t *kout,
            uint32_t *vout, int64_t n, int shift, const uint32_t *__restrict__ tile_off, int ntiles,
            const uint32_t *__restrict__ digit_tot) {
    __shared__ uint32_t wcnt[RS_THREADS / 32][256];
    __shared__ uint32_t goff[256], lstart[256];
    __shared__ uint16_t sidx[RS_TILE];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    {  // global exclusive offset of each digit for this tile, and the tile's local digit starts
        const uint32_t v = digit_tot[threadIdx.x];
        const uint32_t mine = tile_off[(int64_t)threadIdx.x * ntiles + blockIdx.x];
        const uint32_t cnt = (blockIdx.x + 1 < (unsigned)ntiles ? tile_off[(int64_t)threadIdx.x * ntiles + blockIdx.x + 1] : v) - mine;
        uint32_t x = v, y = cnt;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t xs = __shfl_up_sync(0xffffffffu, x, o), ys = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) { x += xs; y += ys; }
        }
        if (lane == 31) { wcnt[0][warp] = x; wcnt[1][warp] = y; }
        __syncthreads();
        uint32_t wp = 0, wl = 0;
        for (int w = 0; w < warp; ++w) { wp += wcnt[0][w]; wl += wcnt[1][w]; }
        goff[threadIdx.x] = wp + x - v + mine;
        lstart[threadIdx.x] = wl + y - cnt;
        __syncthreads();
    }
    uint32_t run = 0;  // thread = digit: items of this digit ranked so far
    const unsigned lt = (1u << lane) - 1u;
    const int64_t base = (int64_t)blockIdx.x * RS_TILE;
    for (int j = 0; j < RS_ITEMS; ++j) {
        for (int w = 0; w < RS_THREADS / 32; ++w) wcnt[w][threadIdx.x] = 0;
        __syncthreads();
        const int64_t i = base + j * RS_THREADS + threadIdx.x;
        const bool valid = i < n;
        const mkey_t k = valid ? kin[i] : 0;
        const int d = valid ? (int)((k >> shift) & 255) : 256 + lane;  // invalid lanes: unique groups
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const uint32_t rank = __popc(peers & lt);
        if (valid && rank == 0) wcnt[warp][d] = __popc(peers);
        __syncthreads();
        {  // thread = digit: prefix over warps (continuing the previous rounds)
            uint32_t r = run;
            for (int w = 0; w < RS_THREADS / 32; ++w) {
                const uint32_t c = wcnt[w][threadIdx.x];
                wcnt[w][threadIdx.x] = r;
                r += c;
            }
            run = r;
        }
        __syncthreads();
        if (valid) sidx[lstart[d] + wcnt[warp][d] + rank] = (uint16_t)(j * RS_THREADS + threadIdx.x);
        __syncthreads();  // wcnt is cleared at the top of the next round
    }
    __syncthreads();
    const int count = (int)min((int64_t)RS_TILE, n - base);
    for (int i = threadIdx.x; i < count; i += RS_THREADS) {
        const int64_t gi = base + sidx[i];
        const mkey_t k = kin[gi];
        const int d = (int)((k >> shift) & 255);
        const uint32_t pos = goff[d] + (uint32_t)(i - (int)lstart[d]);
        kout[pos] = k;
        vout[pos] = vin[gi];
    }
}

// Warp-ranked variant (default): each warp owns a contiguous 512-key slice of the tile and
// loads its 16 keys and values per lane up front (coalesced, 32 loads in flight per thread);
// keys are ranked within the warp by match_any against per-warp digit counters (no block
// barrier per round), one per-digit prefix over the 8 warps orders the warps' runs, and the
// tile is staged in digit order in shared memory and written out bucket run by bucket run (no
// global gather).  Item order inside a digit is the input order (warp slices in order, inside a
// slice key it*32 + lane): stable, the same permutation as k_scatter_c.
__global__ void __launch_bounds__(RS_THREADS)
k_scatter_w(const mkey_t *__restrict__ kin, const uint32_t *__restrict__ vin, mkey_t *kout,
            uint32_t *vout, int64_t n, int shift, const uint32_t *__restrict__ tile_off, int ntiles,
            const uint32_t *__restrict__ digit_tot) {
    constexpr int NW = RS_THREADS / 32, PER_WARP = RS_TILE / NW, IT = PER_WARP / 32;
    __shared__ uint32_t wcnt[NW][256];
    __shared__ uint32_t goff[256], lstart[256];
    __shared__ mkey_t skey[RS_TILE];
    __shared__ uint32_t sval[RS_TILE];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t base = (int64_t)blockIdx.x * RS_TILE;
    const int64_t wbase = base + (int64_t)warp * PER_WARP;
    mkey_t key[IT];
    uint32_t val[IT];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
        const int64_t i = wbase + it * 32 + lane;
        key[it] = i < n ? __ldg(kin + i) : 0;
        val[it] = i < n ? __ldg(vin + i) : 0;
    }
#pragma unroll
    for (int w = 0; w < NW; ++w) wcnt[w][threadIdx.x] = 0;
    {  // global exclusive offset of each digit for this tile, and the tile's local digit starts
        const uint32_t v = digit_tot[threadIdx.x];
        const uint32_t mine = tile_off[(int64_t)threadIdx.x * ntiles + blockIdx.x];
        const uint32_t cnt = (blockIdx.x + 1 < (unsigned)ntiles ? tile_off[(int64_t)threadIdx.x * ntiles + blockIdx.x + 1] : v) - mine;
        uint32_t x = v, y = cnt;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t xs = __shfl_up_sync(0xffffffffu, x, o), ys = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) { x += xs; y += ys; }
        }
        __shared__ uint32_t wsum[2][NW];
        if (lane == 31) { wsum[0][warp] = x; wsum[1][warp] = y; }
        __syncthreads();
        uint32_t wp = 0, wl = 0;
        for (int w = 0; w < warp; ++w) { wp += wsum[0][w]; wl += wsum[1][w]; }
        goff[threadIdx.x] = wp + x - v + mine;
        lstart[threadIdx.x] = wl + y - cnt;
    }
    // rank inside the warp (wcnt[warp][*] is private to this warp: __syncwarp ordering only);
    // the IT match_any instructions are independent and issued first (their latency overlaps)
    uint32_t lrank[IT];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
        const bool valid = wbase + it * 32 + lane < n;
        lrank[it] = __match_any_sync(0xffffffffu, valid ? (int)((key[it] >> shift) & 255) : 256 + lane);
    }
#pragma unroll
    for (int it = 0; it < IT; ++it) {
        const bool valid = wbase + it * 32 + lane < n;
        const int d = valid ? (int)((key[it] >> shift) & 255) : 256 + lane;
        const unsigned peers = lrank[it];
        const int leader = __ffs(peers) - 1;
        uint32_t before = 0;
        if (valid && lane == leader) {
            before = wcnt[warp][d];
            wcnt[warp][d] = before + __popc(peers);
        }
        before = __shfl_sync(0xffffffffu, before, leader);
        lrank[it] = before + __popc(peers & lt);
        __syncwarp();
    }
    __syncthreads();
    {  // thread = digit: exclusive prefix of the warps' counts
        uint32_t r = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const uint32_t c = wcnt[w][threadIdx.x];
            wcnt[w][threadIdx.x] = r;
            r += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < IT; ++it) {
        if (wbase + it * 32 + lane < n) {
            const int d = (int)((key[it] >> shift) & 255);
            const uint32_t li = lstart[d] + wcnt[warp][d] + lrank[it];
            skey[li] = key[it];
            sval[li] = val[it];
        }
    }
    __syncthreads();
    const int count = (int)min((int64_t)RS_TILE, n - base);
    for (int i = threadIdx.x; i < count; i += RS_THREADS) {
        const mkey_t k = skey[i];
        const int d = (int)((k >> shift) & 255);
        const uint32_t pos = goff[d] + (uint32_t)(i - (int)lstart[d]);
        kout[pos] = k;
        vout[pos] = sval[i];
    }
}

// ---------------------------------------------------------------------------------------
// Karras 2012 hierarchy.  Internal nodes 0..n-2; child c < n-1 -> internal, else leaf
// (c-(n-1)) in sorted order.
// ---------------------------------------------------------------------------------------
// common-prefix length of sorted keys i, j, augmented by the index for equal keys
__device__ __forceinline__ int delta(const mkey_t *keys, int64_t n, int64_t i, int64_t j) {
    if (j < 0 || j >= n) return -1;
    const mkey_t a = keys[i], b = keys[j];
    if (a == b) return 32 + __clz((uint32_t)(i ^ j));
    return __clz(a ^ b);
}

__global__ void k_karras(const mkey_t *__restrict__ keys, int64_t n, int *left, int *right,
                         int *parent, int *rlo, int *rhi, int *size) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    int d = delta(keys, n, i, i + 1) - delta(keys, n, i, i - 1) >= 0 ? 1 : -1;
    int dmin = delta(keys, n, i, i - d);
    int64_t lmax = 2;
    while (delta(keys, n, i, i + lmax * d) > dmin) lmax *= 2;
    int64_t l = 0;
    for (int64_t t = lmax / 2; t >= 1; t /= 2)
        if (delta(keys, n, i, i + (l + t) * d) > dmin) l += t;
    int64_t j = i + l * d;
    int dnode = delta(keys, n, i, j);
    int64_t s = 0;
    for (int64_t div = 2;; div *= 2) {
        int64_t t = (l + div - 1) / div;
        if (delta(keys, n, i, i + (s + t) * d) > dnode) s += t;
        if (t <= 1) break;
    }
    int64_t g = i + s * d + min(d, 0);
    int64_t lo = min(i, j), hi = max(i, j);
    int lc = (lo == g) ? (int)(n - 1 + g) : (int)g;
    int rc = (hi == g + 1) ? (int)(n - 1 + g + 1) : (int)(g + 1);
    left[i] = lc;
    right[i] = rc;
    parent[lc] = (int)i;
    parent[rc] = (int)i;
    rlo[i] = (int)lo;
    rhi[i] = (int)hi;
    size[i] = (int)(hi - lo + 1);
}

__global__ void k_refit(int64_t n, const int *__restrict__ left, const int *__restrict__ right,
                        const int *__restrict__ parent, const float4 *__restrict__ slo,
                        const float4 *__restrict__ shi, float4 *nlo, float4 *nhi, int *arrive) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    int node = parent[n - 1 + j];
    while (true) {
        // acq_rel arrival counter: the first arriver's box stores are released by its
        // increment and acquired by the second arriver (replaces two full fences)
        int prev;
        asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;" : "=r"(prev) : "l"(arrive + node) : "memory");
        if (prev == 0) return;
        int c[2] = {left[node], right[node]};
        float4 lo = make_float4(0, 0, 0, 0), hi = lo;
        for (int k = 0; k < 2; ++k) {
            float4 a, b;
            if (c[k] >= n - 1) { a = slo[2 * (c[k] - (n - 1))]; b = shi[2 * (c[k] - (n - 1))]; }
            else { a = __ldcg(nlo + c[k]); b = __ldcg(nhi + c[k]); }
            if (k == 0) { lo = a; hi = b; }
            else {
                lo = make_float4(fminf(lo.x, a.x), fminf(lo.y, a.y), fminf(lo.z, a.z), 0.0f);
                hi = make_float4(fmaxf(hi.x, b.x), fmaxf(hi.y, b.y), fmaxf(hi.z, b.z), 0.0f);
            }
        }
        __stcg(nlo + node, lo);
        __stcg(nhi + node, hi);
        if (node == 0) return;
        node = parent[node];
    }
}

// Agglomerative single pass (Apetrei 2014, "Fast and Simple Agglomerative LBVH Construction"):
// the same binary radix tree as k_karras + k_refit, built bottom-up in one kernel.  A node
// covering sorted leaves [l, r] is the left child of internal node r if keys r, r+1 are closer
// (longer common prefix, ties impossible with index-augmented keys) than keys l-1, l, else the
// right child of internal node l-1; internal node p is the split between leaves p and p+1.
// The first child to arrive at p deposits its outer range bound and leaves; the second
// (acq_rel exchange) merges both boxes and continues.  The root is reported in *root_out.
// split[i] = delta(i, i+1) (common-prefix length of adjacent sorted keys, index-augmented),
// one byte per split: k_agglo reads two bytes per step instead of four 64-bit keys
__device__ __forceinline__ uint32_t range_off(int64_t p, int64_t l, int64_t r) {
    return r - l + 1 <= 7 ? (uint32_t)(p - l) : 7u;
}
__global__ void k_split_delta(const mkey_t *__restrict__ keys, int64_t n, uint8_t *split) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n - 1) split[i] = (uint8_t)delta(keys, n, i, i + 1);
}

// Binary node records (BNode, kernels.h): a = (lo.xyz, left | min(size, 7) << 29), b = (hi.xyz,
// right | off << 29) -- one 32-byte sector per node for the collapse and the sibling reads here.
// Leaf boxes are packed the same way (leaf[2j] = lo, leaf[2j+1] = hi).
// off: a node p of this tree covers the sorted leaves [l, r] with p in [l, r); for nodes of at
// most 7 leaves off = p - l (< 6), so the collapse lists a small subtree's prims as l.. l+size-1
// without walking it; 7 = not recorded (larger nodes; the Karras and PLOC records).
__global__ void k_agglo(const mkey_t *__restrict__ keys, const uint8_t *__restrict__ split, int64_t n,
                        const float4 *__restrict__ leaf, BNode *bn, int *other, int *root_out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t l = i, r = i;
    int cur = (int)(n - 1 + i);
    float4 lo = leaf[2 * i], hi = leaf[2 * i + 1];
    for (;;) {
        bool is_left;
        if (l == 0) is_left = true;
        else if (r == n - 1) is_left = false;
        else if (split) is_left = __ldg(split + r) > __ldg(split + l - 1);
        else is_left = delta(keys, n, r, r + 1) > delta(keys, n, l - 1, l);
        const int64_t p = is_left ? r : l - 1;
        // my id into p's left / right word (the sibling that finishes p reads it)
        if (is_left) __stcg(reinterpret_cast<float *>(&bn[p].a) + 3, __int_as_float(cur));
        else __stcg(reinterpret_cast<float *>(&bn[p].b) + 3, __int_as_float(cur));
        int prev;
        const int val = is_left ? (int)l : (int)r;
        asm volatile("atom.exch.acq_rel.gpu.b32 %0, [%1], %2;" : "=r"(prev) : "l"(other + p), "r"(val) : "memory");
        if (prev < 0) return;  // first arrival: the sibling finishes the node
        const int sib = is_left ? __float_as_int(__ldcg(reinterpret_cast<const float *>(&bn[p].b) + 3))
                                : __float_as_int(__ldcg(reinterpret_cast<const float *>(&bn[p].a) + 3)) & 0x1fffffff;
        float4 a, b;
        if (sib >= n - 1) { a = leaf[2 * (sib - (n - 1))]; b = leaf[2 * (sib - (n - 1)) + 1]; }
        else { a = __ldcg(&bn[sib].a); b = __ldcg(&bn[sib].b); }
        lo = make_float4(fminf(lo.x, a.x), fminf(lo.y, a.y), fminf(lo.z, a.z), 0.0f);
        hi = make_float4(fmaxf(hi.x, b.x), fmaxf(hi.y, b.y), fmaxf(hi.z, b.z), 0.0f);
        if (is_left) r = prev;
        else l = prev;
        const uint32_t cap = (uint32_t)(r - l + 1 < 7 ? r - l + 1 : 7);
        const uint32_t lid = (uint32_t)(is_left ? cur : sib), rid = (uint32_t)(is_left ? sib : cur);
        __stcg(&bn[p].a, make_float4(lo.x, lo.y, lo.z, __uint_as_float(lid | (cap << 29))));
        __stcg(&bn[p].b, make_float4(hi.x, hi.y, hi.z, __uint_as_float(rid | (range_off(p, l, r) << 29))));
        cur = (int)p;
        if (l == 0 && r == n - 1) { *root_out = cur; return; }
    }
}

// The same agglomeration as a persistent kernel with per-lane leaf replacement: a lane whose
// climb ends (first arrival at a node) starts the next leaf of its warp's pool at once, so the
// warp's lanes stay busy (one thread per leaf retires half its warp after the first step and
// ran at 6.4/32 active lanes).  Any order of leaf starts builds the same tree: a node is
// finished by whichever child arrives second.
// The exchange word is 64-bit: (outer range bound << 32) | child id, so the second arrival
// learns its sibling's id from the exchange itself (no separate id store and reload).
__global__ void __launch_bounds__(256) k_agglo_p(const uint8_t *__restrict__ split, int64_t n,
                                                 const float4 *__restrict__ leaf, BNode *bn,
                                                 unsigned long long *other, int *root_out) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    bool alive = false, exhausted = false;
    int64_t l = 0, r = 0, pool = 0, pool_end = 0;
    int64_t chunk = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 64;
    int cur = 0;
    float4 lo = make_float4(0, 0, 0, 0), hi = lo;
    for (;;) {
        const unsigned dead = __ballot_sync(0xffffffffu, !alive);
        if (dead && !exhausted) {
            // refill the dead lanes from the warp's pool (64 leaves per fetch)
            int need = __popc(dead);
            while (need > 0 && !exhausted) {
                if (pool >= pool_end) {
                    // the warp's next chunk of 64 leaves, interleaved over all warps (no shared
                    // counter: one fetch atomic per chunk was a third of the stalls)
                    const int64_t b = chunk;
                    chunk += (int64_t)gridDim.x * (blockDim.x >> 5) * 64;
                    if (b >= n) { exhausted = true; break; }
                    pool = b;
                    pool_end = b + 64 < n ? b + 64 : n;
                }
                const unsigned want = __ballot_sync(0xffffffffu, !alive);
                const int64_t avail = pool_end - pool;
                const int take = (int)(avail < (int64_t)__popc(want) ? avail : (int64_t)__popc(want));
                const int rank = __popc(want & lt);
                if (!alive && rank < take) {
                    const int64_t i = pool + rank;
                    l = r = i;
                    cur = (int)(n - 1 + i);
                    lo = leaf[2 * i];
                    hi = leaf[2 * i + 1];
                    alive = true;
                }
                pool += take;
                need -= take;
            }
        }
        if (!__any_sync(0xffffffffu, alive)) {
            if (exhausted) break;
            continue;
        }
        if (!alive) continue;
        // one climbing step (k_agglo's loop body)
        bool is_left;
        if (l == 0) is_left = true;
        else if (r == n - 1) is_left = false;
        else is_left = __ldg(split + r) > __ldg(split + l - 1);
        const int64_t p = is_left ? r : l - 1;
        const unsigned long long val = ((unsigned long long)(uint32_t)(is_left ? l : r) << 32) | (uint32_t)cur;
        unsigned long long got;
        asm volatile("atom.exch.acq_rel.gpu.b64 %0, [%1], %2;" : "=l"(got) : "l"(other + p), "l"(val) : "memory");
        if (got == ~0ull) { alive = false; continue; }  // first arrival: the sibling finishes the node
        const int prev = (int)(got >> 32), sib = (int)(uint32_t)got;
        float4 a, b;
        if (sib >= n - 1) { a = leaf[2 * (sib - (n - 1))]; b = leaf[2 * (sib - (n - 1)) + 1]; }
        else { a = __ldcg(&bn[sib].a); b = __ldcg(&bn[sib].b); }
        lo = make_float4(fminf(lo.x, a.x), fminf(lo.y, a.y), fminf(lo.z, a.z), 0.0f);
        hi = make_float4(fmaxf(hi.x, b.x), fmaxf(hi.y, b.y), fmaxf(hi.z, b.z), 0.0f);
        if (is_left) r = prev;
        else l = prev;
        const uint32_t cap = (uint32_t)(r - l + 1 < 7 ? r - l + 1 : 7);
        const uint32_t lid = (uint32_t)(is_left ? cur : sib), rid = (uint32_t)(is_left ? sib : cur);
        __stcg(&bn[p].a, make_float4(lo.x, lo.y, lo.z, __uint_as_float(lid | (cap << 29))));
        __stcg(&bn[p].b, make_float4(hi.x, hi.y, hi.z, __uint_as_float(rid | (range_off(p, l, r) << 29))));
        cur = (int)p;
        if (l == 0 && r == n - 1) { *root_out = cur; alive = false; }
    }
}

// Packed records from the separate arrays of the Karras + refit and PLOC builders.
__global__ void k_pack_bnodes(int64_t n, const int *__restrict__ left, const int *__restrict__ right,
                              const int *__restrict__ size, const float4 *__restrict__ nlo,
                              const float4 *__restrict__ nhi, BNode *bn) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n - 1) return;
    const float4 lo = nlo[p], hi = nhi[p];
    const uint32_t cap = (uint32_t)min(size[p], 7);
    bn[p].a = make_float4(lo.x, lo.y, lo.z, __uint_as_float((uint32_t)left[p] | (cap << 29)));
    bn[p].b = make_float4(hi.x, hi.y, hi.z, __uint_as_float((uint32_t)right[p] | (7u << 29)));
}

// Outward padding: |x| + 4 scaled by 2^-18 (>= 1.5e-5 absolute).  Covers the FMA box test
// error and MT hit-point rounding.
__device__ __forceinline__ float pad_lo(float x) { return x - (fabsf(x) + 4.0f) * 0x1p-18f; }
__device__ __forceinline__ float pad_hi(float x) { return x + (fabsf(x) + 4.0f) * 0x1p-18f; }

__global__ void k_gather_prims(const float4 *__restrict__ in, const uint32_t *__restrict__ perm,
                               int64_t n, float4 *out, const float4 *__restrict__ blo,
                               const float4 *__restrict__ bhi, float4 *slo, float4 *shi) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t s = perm[i];
    if (out) {
        out[3 * i + 0] = in[3 * (int64_t)s + 0];
        out[3 * i + 1] = in[3 * (int64_t)s + 1];
        out[3 * i + 2] = in[3 * (int64_t)s + 2];
    }
    slo[2 * i] = blo[2 * (int64_t)s];  // packed leaf record: lo at 2i, hi at 2i + 1 (slo + 1 == shi);
    shi[2 * i] = bhi[2 * (int64_t)s];  // the input boxes are interleaved the same way (one sector)
}

// ---------------------------------------------------------------------------------------
// Collapse of the binary LBVH into compressed 8-wide nodes (WNode, common.cuh), one BFS
// level per launch: each item turns one binary subtree root into one wide node by
// repeatedly opening its largest-area child that is still an internal node with more
// than LEAF_MAX prims, until 8 children or nothing left to open.  Leaf children's prims
// are copied contiguously per wide node (prim_base + offset, offset < 32).
// ---------------------------------------------------------------------------------------

// Binary node ids: internal k in [0, n-1), leaf (sorted prim) j -> n-1+j.  One 32-byte
// record per node (BNode; leaves: a.leaf[2j], a.leaf[2j+1]); sz = min(prim count, 7).
// cl: left id | min(size, 7) << 29 (a leaf: size 1), cr: right id | range offset << 29
__device__ __forceinline__ void bin_child(const CollapseArgs &a, int id, float lo[3], float hi[3], uint32_t &cl,
                                          uint32_t &cr) {
    float4 l, h;
    if (id >= a.n - 1) {
        const int64_t j = id - (a.n - 1);
        l = __ldg(a.leaf + 2 * j); h = __ldg(a.leaf + 2 * j + 1); cl = 1u << 29; cr = 0;
    } else {
        l = __ldg(&a.bn[id].a); h = __ldg(&a.bn[id].b);
        cl = __float_as_uint(l.w); cr = __float_as_uint(h.w);
    }
    lo[0] = pad_lo(l.x); lo[1] = pad_lo(l.y); lo[2] = pad_lo(l.z);
    hi[0] = pad_hi(h.x); hi[1] = pad_hi(h.y); hi[2] = pad_hi(h.z);
}

// One thread per wide node.  (A variant with a group of 8 lanes per node -- one child per
// lane, group reductions -- used 48 instead of 158 registers but executed ~2000 instructions
// per node and ran slower: 7.4 vs 5.7 ms per configs[3] build, r02.)
// Every per-child array is indexed with compile-time indices (unrolled selects), so the child
// boxes, ids, slot costs and quantised planes stay in registers (an earlier version indexed
// them dynamically: a 320-416 B local-memory frame that thrashed L1 at full occupancy).
// Persistent grid-stride loop over the level's items; the item count is read from device
// memory (cnt_in) and the next level's items are appended (cnt_out), so several levels are
// launched back to back without a host round trip.
#ifndef DPR_COLLAPSE_MINB
#define DPR_COLLAPSE_MINB 6
#endif
constexpr int CB = 128;  // collapse block
// Per-thread child state in shared memory, [field][child][thread] (conflict-free: a warp's
// threads read the same child slot of consecutive threads), so a child is inserted with one
// store per field at a dynamic index instead of unrolled selects over 8 register slots (those
// selects were most of the register version's instructions at 164 registers / 18% occupancy).
// Also in shared memory: each child's argmax key (box area; 8 register selects per insert
// before, configs[3] build 11.78 -> 11.66 ms); in registers: the internal / large bit masks;
// the capped sizes ride in the top bits of ccl.
struct CollapseSmem {
    int cid[8][CB];
    uint32_t ccl[8][CB], ccr[8][CB];
    float lo[3][8][CB], hi[3][8][CB];
    uint32_t akey[8][CB];  // argmax keys: box area | 8 | (7 - child)
};

__global__ void __launch_bounds__(CB, DPR_COLLAPSE_MINB) k_collapse_r(const CollapseArgs a, const int2 *__restrict__ items,
                                                    const int *__restrict__ cnt_in, int2 *next, int *cnt_out) {
  extern __shared__ __align__(16) unsigned char collapse_smem[];
  CollapseSmem &S = *reinterpret_cast<CollapseSmem *>(collapse_smem);
  const int tid = threadIdx.x;
  const int nitems = *cnt_in;
  const int lane = threadIdx.x & 31;
  // warp-uniform trip count (the allocation below is one atomic per warp and counter: with one
  // per node the three counters took ~30M same-address atomics per configs[3] build)
  for (int t0 = (int)((blockIdx.x * blockDim.x + threadIdx.x) & ~31u); t0 < nitems; t0 += gridDim.x * blockDim.x) {
    const int t = t0 + lane;
    const bool live = t < nitems;
    const int2 item = live ? items[t] : make_int2(0, 0);
    const int wnode = item.x, b = item.y;
    // argmax keys: box area with the low 4 mantissa bits replaced by 8 | (7 - i) (> 0, ties
    // to the lowest child index); bit masks of internal children and of those with more than
    // LEAF_MAX prims; sizes live in the top bits of ccl
    unsigned inner_m = 0, big_m = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) S.akey[i][tid] = 0;
    auto put = [&](int i, int id) -> void {  // load child id into slot i (smem + registers)
        float lo3[3], hi3[3];
        uint32_t cl, cr;
        bin_child(a, id, lo3, hi3, cl, cr);
        S.cid[i][tid] = id; S.ccl[i][tid] = cl; S.ccr[i][tid] = cr;
#pragma unroll
        for (int c = 0; c < 3; ++c) { S.lo[c][i][tid] = lo3[c]; S.hi[c][i][tid] = hi3[c]; }
        const float ex = hi3[0] - lo3[0], ey = hi3[1] - lo3[1], ez = hi3[2] - lo3[2];
        const float ar = ex * ey + ey * ez + ez * ex;
        const uint32_t key = (__float_as_uint(ar) & ~15u) | 8u | (uint32_t)(7 - i);
        S.akey[i][tid] = key;
        const bool in = id < a.n - 1, big = in && (int)(cl >> 29) > LEAF_MAX;
        inner_m = in ? (inner_m | (1u << i)) : (inner_m & ~(1u << i));
        big_m = big ? (big_m | (1u << i)) : (big_m & ~(1u << i));
    };
    int nc = 0;
    if (!live) {
    } else if (b < 0) {  // single-prim world: the root holds one leaf
        put(0, (int)(a.n - 1));
        nc = 1;
    } else {
        put(0, (int)(__float_as_uint(__ldg(&a.bn[b].a.w)) & 0x1fffffffu));
        put(1, (int)(__float_as_uint(__ldg(&a.bn[b].b.w)) & 0x1fffffffu));
        nc = 2;
    }
    // pass 0: open the largest-area internal child with > LEAF_MAX prims; pass 1
    // (DPR_FILL_LEAVES): then the largest small subtree, while slots are free
    for (int pass = 0; pass < (DPR_FILL_LEAVES ? 2 : 1); ++pass) {
        while (nc < 8) {
            const unsigned elig = (pass == 0 ? (inner_m & big_m) : inner_m) & ((1u << nc) - 1u);
            if (!elig) break;
            uint32_t m = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) m = max(m, (elig >> i & 1) ? S.akey[i][tid] : 0u);
            const int best = 7 - (int)(m & 7u);
            const int l = (int)(S.ccl[best][tid] & 0x1fffffffu), r = (int)(S.ccr[best][tid] & 0x1fffffffu);
            put(best, l);
            put(nc, r);
            nc++;
        }
    }
    // node box
    float nlo_[3], nhi_[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) { nlo_[c] = __int_as_float(0x7f800000); nhi_[c] = -__int_as_float(0x7f800000); }
    for (int i = 0; i < nc; ++i)
#pragma unroll
        for (int c = 0; c < 3; ++c) { nlo_[c] = fminf(nlo_[c], S.lo[c][i][tid]); nhi_[c] = fmaxf(nhi_[c], S.hi[c][i][tid]); }
    // octant slot assignment: greedy on cost(child, slot) = dot(child centre - node centre,
    // octant signs of the slot), highest first; each child's best free slot is cached and
    // recomputed only when another child takes it
    int slot_of[8];
    {
        // candidate keys (in S.akey, free after the opening phase): the cost as an
        // order-preserving integer with its low 6 bits replaced by (slot << 3) | (7 - child), so
        // one integer max picks the child (ties: lowest index) and carries its slot; an assigned
        // child's entry holds its slot (0..7, below every key), an absent child's 0
        auto pack = [](float c, int sl, int i) -> uint32_t {
            const uint32_t u = __float_as_uint(c);
            const uint32_t o = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
            return (o & ~63u) | ((uint32_t)sl << 3) | (uint32_t)(7 - i);
        };
        // (a variant walking a child's slots in falling cost order -- its octant with the sign
        // flips ordered by the flipped |offset| sum -- ran slower: 13.7 vs 12.8 ms per
        // configs[3] build, r02)
        auto best_free = [&](int i, unsigned used, float &bc, int &bs) -> void {
            float dc[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) dc[c] = (S.lo[c][i][tid] + S.hi[c][i][tid]) - (nlo_[c] + nhi_[c]);
            bc = -3.4e38f; bs = 0;
#pragma unroll
            for (int sl = 0; sl < 8; ++sl) {
                const float cst = ((sl & 4) ? dc[0] : -dc[0]) + ((sl & 2) ? dc[1] : -dc[1]) + ((sl & 1) ? dc[2] : -dc[2]);
                if (!(used >> sl & 1) && cst > bc) { bc = cst; bs = sl; }
            }
        };
        // with every slot free, a child's best slot is the octant of its offset and its cost
        // |dx| + |dy| + |dz|
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            uint32_t key = 0;
            if (i < nc) {
                float dc[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) dc[c] = (S.lo[c][i][tid] + S.hi[c][i][tid]) - (nlo_[c] + nhi_[c]);
                key = pack((fabsf(dc[0]) + fabsf(dc[1])) + fabsf(dc[2]),
                           (dc[0] > 0.0f ? 4 : 0) | (dc[1] > 0.0f ? 2 : 0) | (dc[2] > 0.0f ? 1 : 0), i);
            }
            S.akey[i][tid] = key;
        }
        unsigned used_slots = 0;
        // lazy greedy: a child's cached (cost, slot) is an upper bound of its best free slot
        // (costs only fall as slots fill); the largest cached entry is assigned if its slot is
        // still free, else recomputed and the selection repeated -- the same greedy choice,
        // recomputing only the children that come up instead of every child that lost a slot
        // (configs[3] build 12.44 -> 12.03 ms, r02)
        for (int k = 0; k < nc;) {
            uint32_t m = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) m = max(m, S.akey[i][tid]);
            const int bi = 7 - (int)(m & 7u), bs = (int)((m >> 3) & 7u);
            if (used_slots >> bs & 1) {
                float nc_; int ns_;
                best_free(bi, used_slots, nc_, ns_);
                S.akey[bi][tid] = pack(nc_, ns_, bi);
                continue;
            }
            S.akey[bi][tid] = (uint32_t)bs;
            used_slots |= 1u << bs;
            ++k;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) slot_of[i] = i < nc ? (int)S.akey[i][tid] : 0;
    }
    // internal vs leaf children, allocation
    int n_int = 0, n_prims = 0;
    unsigned imask = 0, lmask = 0, leaf_m = 0;
    unsigned long long szslot = 0;  // byte s: prims of the leaf child in slot s
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        if (i >= nc) continue;
        if (!(big_m >> i & 1)) {
            const uint32_t sz = S.ccl[i][tid] >> 29;
            n_prims += (int)sz; lmask |= 1u << slot_of[i]; leaf_m |= 1u << i;
            szslot |= (unsigned long long)sz << (8 * slot_of[i]);
        } else { n_int++; imask |= 1u << slot_of[i]; }
    }
    const unsigned long long szpre = szslot * 0x0101010101010101ull;  // byte s: prims in slots <= s
    int child_base, prim_base, out_base;
    {
        int xi = n_int, xp = n_prims;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int yi = __shfl_up_sync(0xffffffffu, xi, o), yp = __shfl_up_sync(0xffffffffu, xp, o);
            if (lane >= o) { xi += yi; xp += yp; }
        }
        int bi = 0, bp = 0, bo = 0;
        if (lane == 31) {
            bi = xi ? atomicAdd(&a.counters[1], xi) : 0;
            bp = xp ? atomicAdd(&a.counters[2], xp) : 0;
            bo = xi ? atomicAdd(cnt_out, xi) : 0;
        }
        bi = __shfl_sync(0xffffffffu, bi, 31);
        bp = __shfl_sync(0xffffffffu, bp, 31);
        bo = __shfl_sync(0xffffffffu, bo, 31);
        child_base = bi + xi - n_int;
        prim_base = bp + xp - n_prims;
        out_base = bo + xi - n_int;
    }
    if (!live) continue;
    if (child_base + n_int > a.node_cap) { atomicOr(&a.counters[3], 1); continue; }
#ifdef DPR_COLLAPSE_STATS
    atomicAdd(&a.counters[0], nc);
#endif
    // quantisation (outward): smallest e with 255 * 2^e >= extent (frexp, no log2); the
    // per-child planes below multiply by the exact power-of-two reciprocal (no division)
    float p[3];
    int e[3];
    float isc[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        p[c] = nlo_[c];
        const double ext = (double)nhi_[c] - (double)p[c];
        int ee = -126;
        if (ext > 0) {
            int ex;
            frexp(ext / 255.0, &ex);
            ee = ex - 1;
            while (ldexp(255.0, ee) < ext) ee++;
            if (ee < -126) ee = -126;
            if (ee > 127) ee = 127;
        }
        e[c] = ee;
        isc[c] = ldexpf(1.0f, -ee);  // extents of finite boxes keep ee <= 122: a normal float
    }
    uint32_t qw[6][2], mw[2] = {0u, 0u};
#pragma unroll
    for (int k = 0; k < 6; ++k) qw[k][0] = qw[k][1] = 0u;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        if (i >= nc) continue;
        const int sl = slot_of[i];
        const int sh = 8 * (sl & 3);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            // floor / ceil of the exact (child - node) / 2^e: the difference rounded down (up)
            // lands on the same side of every plane k * 2^e (k <= 255: a float), and the
            // power-of-two scaling is exact -- the same planes as the exact computation
            const float ql = floorf(__fsub_rd(S.lo[c][i][tid], p[c]) * isc[c]);
            const float qh = ceilf(__fsub_ru(S.hi[c][i][tid], p[c]) * isc[c]);
            const uint32_t bl = (uint32_t)fminf(fmaxf(ql, 0.0f), 255.0f), bh = (uint32_t)fminf(fmaxf(qh, 0.0f), 255.0f);
            if (sl < 4) { qw[c][0] |= bl << sh; qw[3 + c][0] |= bh << sh; }
            else { qw[c][1] |= bl << sh; qw[3 + c][1] |= bh << sh; }
        }
        const int cidi = S.cid[i][tid];
        if (!(leaf_m >> i & 1)) {
            const int rank = __popc(imask & ((1u << sl) - 1u));
            next[out_base + rank] = make_int2(child_base + rank, cidi);
        } else {
            // prims of the leaf children are laid out in slot order
            const int off = sl ? (int)((szpre >> (8 * (sl - 1))) & 0xffu) : 0;
            const int ci = (int)(S.ccl[i][tid] >> 29);
            const uint32_t m = 0x80u | ((uint32_t)(ci - 1) << 5) | (uint32_t)off;
            if (sl < 4) mw[0] |= m << sh; else mw[1] |= m << sh;
            // the (<= LEAF_MAX) prims of the binary subtree, in sorted order: a contiguous
            // range when the record holds its offset, else a walk of the subtree
            const uint32_t roff = S.ccr[i][tid] >> 29;
            if (cidi >= a.n - 1) {
                a.perm[prim_base + off] = (uint32_t)(cidi - (a.n - 1));
            } else if (roff != 7u) {
                const uint32_t l0 = (uint32_t)cidi - roff;
                for (int k = 0; k < ci; ++k) a.perm[prim_base + off + k] = l0 + (uint32_t)k;
            } else {
                int st[8], sp = 0, k = 0;
                st[sp++] = cidi;
                while (sp) {
                    const int x = st[--sp];
                    if (x >= a.n - 1) a.perm[prim_base + off + k++] = (uint32_t)(x - (a.n - 1));
                    else {
                        st[sp++] = (int)(__float_as_uint(__ldg(&a.bn[x].b.w)) & 0x1fffffffu);
                        st[sp++] = (int)(__float_as_uint(__ldg(&a.bn[x].a.w)) & 0x1fffffffu);
                    }
                }
            }
        }
    }
    WNode nd;
    const uint32_t bits = (uint32_t)(e[0] + 127) | ((uint32_t)(e[1] + 127) << 8) | ((uint32_t)(e[2] + 127) << 16) | (imask << 24);
    nd.w0 = make_float4(p[0], p[1], p[2], __uint_as_float(bits));
    nd.w1 = make_uint4((uint32_t)child_base | ((lmask & 0xfu) << 28), (uint32_t)prim_base | ((lmask >> 4) << 28),
                       mw[0], mw[1]);
    nd.w2 = make_uint4(qw[0][0], qw[0][1], qw[1][0], qw[1][1]);
    nd.w3 = make_uint4(qw[2][0], qw[2][1], qw[3][0], qw[3][1]);
    nd.w4 = make_uint4(qw[4][0], qw[4][1], qw[5][0], qw[5][1]);
    a.nodes[wnode] = nd;
  }
}

#ifndef DPR_COLLAPSE_GRID
#define DPR_COLLAPSE_GRID 8  // resident-grid multiple of the persistent collapse launch (r02 sweep: 1, 4, 8)
#endif
int collapse_grid() {
    static int g = 0;
    if (!g) {
        int dev = 0, nsm = 0, occ = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(k_collapse_r, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(CollapseSmem));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_collapse_r, CB, sizeof(CollapseSmem));
        g = nsm * std::max(1, occ) * DPR_COLLAPSE_GRID;
    }
    return g;
}
void launch_collapse_level(const CollapseArgs &a, const int2 *items, const int *cnt_in, int2 *next, int *cnt_out,
                           int level, cudaStream_t s) {
    // level k holds at most 8^k wide nodes: the first levels get a grid of that size instead
    // of the resident grid (a 7K-block launch that finds one item costs ~20 us)
    int g = collapse_grid();
    if (level < 8) g = std::min<int64_t>(g, std::max<int64_t>(1, (((int64_t)1 << (3 * level)) + CB - 1) / CB));
    k_collapse_r<<<g, CB, sizeof(CollapseSmem), s>>>(a, items, cnt_in, next, cnt_out);
}

// prims_out[i] = prims_in[perm[i]] (3 float4 each).  The two permutations compose: wide-node
// order -> Morton order (perm) -> input order (sortperm).  One thread per prim: its three
// records' loads in flight together (the random gather), 48 contiguous bytes per thread out.
// (An inverse table local id -> prim index was scattered here until r02; the cooperative prim
// tests now record the winning prim index themselves -- the random 4-byte scatter cost a
// 64-byte DRAM read-modify-write per prim.)
__global__ void k_permute_prims(const float4 *__restrict__ in, const uint32_t *__restrict__ perm,
                                const uint32_t *__restrict__ sortperm, int64_t n, float4 *out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t src = __ldg(sortperm + __ldg(perm + i));
    const float4 *q = in + 3 * (int64_t)src;
    const float4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
    out[3 * i] = a;
    out[3 * i + 1] = b;
    out[3 * i + 2] = c;
}

void launch_permute_prims(const float4 *in, const uint32_t *perm, const uint32_t *sortperm, int64_t n,
                          float4 *out, cudaStream_t s) {
    if (n > 0) k_permute_prims<<<nblk(n, 256), 256, 0, s>>>(in, perm, sortperm, n, out);
}

// ---------------------------------------------------------------------------------------
// Macrocells: one block per 16^3 macrocell.  A sample owned by the brick with
// floor(g) in cell c reads voxels c..c+1; a macrocell covers cells [m*16, m*16+16) so it
// reads voxels [m*16, m*16+16] (clamped to the stored range).  Active iff some TF entry in
// the index range that the value range maps to (widened by one entry on each side) has
// alpha > 0 -- exact skipping (u >= 0 is never < 0).
// ---------------------------------------------------------------------------------------
// One block per (macrocell row along x, macrocell y, macrocell z): threads sweep the voxel
// rows of the slab with x fastest (coalesced), each thread keeps min/max of its x columns,
// then per-macrocell reductions in shared memory.
constexpr int MC_BLOCK = 256;
__global__ void __launch_bounds__(MC_BLOCK) k_macrocells(const float *__restrict__ vox, int nx, int ny, int nz,
                                                        int mcx, int mcy, int mcz, const float4 *__restrict__ tf,
                                                        float tf_lo, float tf_hi, float dscale, uint8_t *mc) {
    const int my = blockIdx.x, mz = blockIdx.y;
    const int y0 = my * MC_SIZE, z0 = mz * MC_SIZE;
    const int y1 = min(y0 + MC_SIZE, ny - 1), z1 = min(z0 + MC_SIZE, nz - 1);
    __shared__ float smin[MC_BLOCK], smax[MC_BLOCK];
    // process the x extent in chunks of MC_BLOCK voxels (each chunk covers MC_BLOCK/16
    // macrocells; the +1 overlap voxel is read by the next macrocell's range too)
    for (int xc = 0; xc < mcx * MC_SIZE; xc += MC_BLOCK - MC_BLOCK % MC_SIZE) {
        const int x = xc + threadIdx.x;
        float vmin = __int_as_float(0x7f800000), vmax = -vmin;
        if (x < nx) {
            for (int z = z0; z <= z1; ++z)
                for (int y = y0; y <= y1; ++y) {
                    float v = vox[(int64_t)x + (int64_t)nx * ((int64_t)y + (int64_t)ny * z)];
                    vmin = fminf(vmin, v);
                    vmax = fmaxf(vmax, v);
                }
        }
        smin[threadIdx.x] = vmin;
        smax[threadIdx.x] = vmax;
        __syncthreads();
        const int per = (MC_BLOCK - MC_BLOCK % MC_SIZE) / MC_SIZE;  // macrocells per chunk
        if ((int)threadIdx.x < per) {
            const int mx = xc / MC_SIZE + threadIdx.x;
            if (mx < mcx) {
                const int xa = mx * MC_SIZE - xc, xb = min(mx * MC_SIZE + MC_SIZE, nx - 1) - xc;
                float a = __int_as_float(0x7f800000), b = -a;
                for (int t = xa; t <= xb && t < MC_BLOCK; ++t) { a = fminf(a, smin[t]); b = fmaxf(b, smax[t]); }
                if (xb >= MC_BLOCK) {  // the overlap voxel belongs to the next chunk: read it
                    const int xg = xc + xb;
                    for (int z = z0; z <= z1; ++z)
                        for (int y = y0; y <= y1; ++y) {
                            float v = vox[(int64_t)xg + (int64_t)nx * ((int64_t)y + (int64_t)ny * z)];
                            a = fminf(a, v);
                            b = fmaxf(b, v);
                        }
                }
                float xa_ = fminf(fmaxf((a - tf_lo) / (tf_hi - tf_lo), 0.0f), 1.0f) * 255.0f;
                float xb_ = fminf(fmaxf((b - tf_lo) / (tf_hi - tf_lo), 0.0f), 1.0f) * 255.0f;
                int ja = max((int)floorf(xa_) - 1, 0), jb = min((int)floorf(xb_) + 2, 255);
                bool active = !(a == a) || !(b == b);  // NaN voxels: never skip
                for (int j = ja; j <= jb; ++j) active |= tf[j].w != 0.0f;
                mc[((int64_t)mz * mcy + my) * mcx + mx] = active ? 1 : 0;
            }
        }
        __syncthreads();
    }
}

// Macrocell distance field (empty-space jumps of k_march_*): d = 0 where mc = 1, else the
// Chebyshev distance in macrocells to the nearest mc = 1 cell, capped.  k passes of
// d <- min(d, 1 + min over the 26 neighbours) from d0 = (mc ? 0 : CAP) give min(true, k+1)
// exactly when CAP = k+1 (cells farther than k keep CAP <= their true distance), so a
// distance never overstates the empty box around a cell.  Cells outside the grid hold no
// owned sample and count as empty.
__global__ void k_mc_dist_init(const uint8_t *__restrict__ mc, int64_t n, uint8_t *d) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) d[i] = mc[i] ? 0 : (uint8_t)MC_DIST_CAP;
}
__global__ void k_mc_dist_pass(const uint8_t *__restrict__ din, int mx, int my, int mz, uint8_t *dout) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)mx * my * mz) return;
    const int x = (int)(i % mx), y = (int)((i / mx) % my), z = (int)(i / ((int64_t)mx * my));
    int m = din[i];
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                const int xx = x + dx, yy = y + dy, zz = z + dz;
                if (xx < 0 || yy < 0 || zz < 0 || xx >= mx || yy >= my || zz >= mz) continue;
                m = min(m, 1 + (int)din[((int64_t)zz * my + yy) * mx + xx]);
            }
    dout[i] = (uint8_t)m;
}

// ---------------------------------------------------------------------------------------
// Host-side launchers.
// ---------------------------------------------------------------------------------------

void launch_part_prims(const PrimChunk *chunks, int nchunks, float4 *prims, float4 *blo, float4 *bhi, int *bounds,
                       int *bad_index, cudaStream_t s) {
    if (nchunks > 0) k_part_prims<<<nchunks, 256, 0, s>>>(chunks, prims, blo, bhi, bounds, bad_index);
}
void launch_morton_h(const float4 *blo, const float4 *bhi, int64_t n, const int *bounds, mkey_t *keys, uint32_t *vals,
                     uint32_t *tile_hist0, unsigned long long *hist_all, cudaStream_t s) {
    if (n > 0) {
        const int ntiles = (int)radix_tiles(n);
        k_morton_h<<<ntiles, RS_THREADS, 0, s>>>(blo, bhi, n, bounds, keys, vals, tile_hist0, ntiles, hist_all);
    }
}
int64_t radix_tiles(int64_t n) { return (n + RS_TILE - 1) / RS_TILE; }
__global__ void k_iota(uint32_t *v, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = (uint32_t)i;
}
void launch_iota(uint32_t *v, int64_t n, cudaStream_t s) {
    if (n > 0) k_iota<<<nblk(n, 256), 256, 0, s>>>(v, n);
}
void launch_radix_pass(const mkey_t *kin, const uint32_t *vin, mkey_t *kout, uint32_t *vout,
                       int64_t n, int shift, uint32_t *tile_hist, cudaStream_t s, int *launches, bool hist_ready) {
    int ntiles = (int)radix_tiles(n);
    uint32_t *digit_tot = tile_hist + (int64_t)256 * ntiles;  // 256 extra words
    if (!hist_ready) k_tile_hist<<<ntiles, RS_THREADS, 0, s>>>(kin, n, shift, tile_hist, ntiles);
    else *launches -= 1;
    k_scan_digits<<<256, 1024, 0, s>>>(tile_hist, ntiles, digit_tot);
#ifndef DPR_SCATTER_COALESCED
#define DPR_SCATTER_COALESCED 2  // 2 warp-ranked, 1 ranked per round, 0 direct
#endif
    if (DPR_SCATTER_COALESCED == 2) k_scatter_w<<<ntiles, RS_THREADS, 0, s>>>(kin, vin, kout, vout, n, shift, tile_hist, ntiles, digit_tot);
    else if (DPR_SCATTER_COALESCED) k_scatter_c<<<ntiles, RS_THREADS, 0, s>>>(kin, vin, kout, vout, n, shift, tile_hist, ntiles, digit_tot);
    else k_scatter<<<ntiles, RS_THREADS, 0, s>>>(kin, vin, kout, vout, n, shift, tile_hist, ntiles, digit_tot);
    *launches += 3;
}
void launch_karras(const mkey_t *keys, int64_t n, int *left, int *right, int *parent, int *rlo,
                   int *rhi, int *size, cudaStream_t s) {
    if (n > 1) k_karras<<<nblk(n - 1, 256), 256, 0, s>>>(keys, n, left, right, parent, rlo, rhi, size);
}
void launch_refit(int64_t n, const int *left, const int *right, const int *parent,
                  const float4 *slo, const float4 *shi, float4 *nlo, float4 *nhi, int *arrive,
                  cudaStream_t s) {
    if (n > 1) k_refit<<<nblk(n, 256), 256, 0, s>>>(n, left, right, parent, slo, shi, nlo, nhi, arrive);
}
#ifndef DPR_AGGLO_SPLIT
#define DPR_AGGLO_SPLIT 1
#endif
#ifndef DPR_AGGLO_PERSIST
#define DPR_AGGLO_PERSIST 1
#endif
int launch_agglo(const mkey_t *keys, uint8_t *split_scratch, int64_t n, const float4 *leaf, BNode *bn,
                 void *other, int *root_out, cudaStream_t s) {
    if (n <= 1) return 0;
    uint8_t *split = DPR_AGGLO_SPLIT ? split_scratch : nullptr;
    if (split) k_split_delta<<<nblk(n, 256), 256, 0, s>>>(keys, n, split);
    if (DPR_AGGLO_PERSIST && split) {
        static int grid = 0;
        if (!grid) {
            int dev = 0, nsm = 0, occ = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_agglo_p, 256, 0);
            grid = nsm * std::max(1, occ);
        }
        // a resident grid, or one 64-leaf chunk per warp when the tree is small
        const int64_t need = (n + 8 * 64 - 1) / (8 * 64);
        k_agglo_p<<<(int)std::min<int64_t>(grid, need), 256, 0, s>>>(split, n, leaf, bn,
                                                                       static_cast<unsigned long long *>(other), root_out);
        return 2;
    }
    k_agglo<<<nblk(n, 256), 256, 0, s>>>(keys, split, n, leaf, bn, static_cast<int *>(other), root_out);
    return split ? 2 : 1;
}
void launch_pack_bnodes(int64_t n, const int *left, const int *right, const int *size, const float4 *nlo,
                        const float4 *nhi, BNode *bn, cudaStream_t s) {
    if (n > 1) k_pack_bnodes<<<nblk(n - 1, 256), 256, 0, s>>>(n, left, right, size, nlo, nhi, bn);
}
void launch_gather_prims(const float4 *in, const uint32_t *perm, int64_t n, float4 *out,
                         const float4 *blo, const float4 *bhi, float4 *slo, float4 *shi,
                         cudaStream_t s) {
    if (n > 0) k_gather_prims<<<nblk(n, 256), 256, 0, s>>>(in, perm, n, out, blo, bhi, slo, shi);
}
int launch_macrocells(const float *vox, int nx, int ny, int nz, int mcx, int mcy, int mcz,
                      const float4 *tf, float tf_lo, float tf_hi, float dscale, uint8_t *mc,
                      cudaStream_t s) {
    if (!(mcx > 0 && mcy > 0 && mcz > 0)) return 0;
    k_macrocells<<<dim3(mcy, mcz), MC_BLOCK, 0, s>>>(vox, nx, ny, nz, mcx, mcy, mcz, tf, tf_lo, tf_hi, dscale, mc);
    // distance field at mc + n (ping-pong with mc + 2n; an even number of passes ends in mc + n)
    const int64_t n = (int64_t)mcx * mcy * mcz;
    uint8_t *d0 = mc + n, *d1 = mc + 2 * n;
    k_mc_dist_init<<<nblk(n, 256), 256, 0, s>>>(mc, n, d0);
    static_assert(MC_DIST_PASSES % 2 == 0, "result must end in mc + n");
    for (int k = 0; k < MC_DIST_PASSES; ++k) {
        k_mc_dist_pass<<<nblk(n, 256), 256, 0, s>>>(k % 2 ? d1 : d0, mcx, mcy, mcz, k % 2 ? d0 : d1);
    }
    return 2 + MC_DIST_PASSES;
}

}  // namespace dpr
