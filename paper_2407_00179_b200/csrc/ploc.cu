// ploc.cu -- binary BVH by Parallel Locally-Ordered Clustering (Meister & Bittner 2018,
// "Parallel Locally-Ordered Clustering for Bounding Volume Hierarchy Construction"), built on
// the Morton-sorted prims of lbvh.cu (part of SURVEY 8(a) row a1).
//
// Clusters start as the sorted leaves.  Each iteration:
//   k_ploc_nn     nearest neighbour of every cluster within +-PLOC_R positions, by the surface
//                 area of the merged box, ties broken by the smaller index (a strict total
//                 order, so the globally closest pair is always mutual: progress guaranteed)
//   k_ploc_count  per-block counts of surviving clusters and of merges (i < NN(i) mutual)
//   k_ploc_scan   exclusive scan of the block counts (one block)
//   k_ploc_write  merged clusters become new internal nodes (numbered by the scan:
//                 deterministic), survivors are compacted in order
// until one cluster remains.  Node ids: internal k in [0, n-1), leaf j -> n-1+j (the same
// convention as the Karras builder, so the wide-BVH collapse consumes either).  Boxes and
// subtree sizes are produced bottom-up by construction: no refit pass.
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"

namespace dpr {

constexpr int PLOC_R = 16;
constexpr int PLOC_NN_BLOCK = 256;
constexpr int PLOC_BLOCK = 1024;

static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

__device__ __forceinline__ void node_box(const PlocArgs &a, int id, float4 &lo, float4 &hi) {
    if (id >= a.n - 1) { lo = a.slo[2 * (id - (a.n - 1))]; hi = a.shi[2 * (id - (a.n - 1))]; }  // packed leaf records
    else { lo = a.nlo[id]; hi = a.nhi[id]; }
}

__device__ __forceinline__ float merged_area(float4 al, float4 ah, float4 bl, float4 bh) {
    float dx = fmaxf(ah.x, bh.x) - fminf(al.x, bl.x);
    float dy = fmaxf(ah.y, bh.y) - fminf(al.y, bl.y);
    float dz = fmaxf(ah.z, bh.z) - fminf(al.z, bl.z);
    return dx * dy + dy * dz + dz * dx;
}

__global__ void k_ploc_init(int64_t n, int *clusters) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) clusters[j] = (int)(n - 1 + j);
}

__global__ void __launch_bounds__(PLOC_NN_BLOCK) k_ploc_nn(const PlocArgs a, const int *__restrict__ C, int64_t m,
                                                           int *nn) {
    __shared__ float4 slo[PLOC_NN_BLOCK + 2 * PLOC_R], shi[PLOC_NN_BLOCK + 2 * PLOC_R];
    const int64_t b0 = (int64_t)blockIdx.x * PLOC_NN_BLOCK;
    for (int t = threadIdx.x; t < PLOC_NN_BLOCK + 2 * PLOC_R; t += blockDim.x) {
        int64_t idx = b0 - PLOC_R + t;
        if (idx >= 0 && idx < m) node_box(a, C[idx], slo[t], shi[t]);
    }
    __syncthreads();
    const int64_t i = b0 + threadIdx.x;
    if (i >= m) return;
    const int li = threadIdx.x + PLOC_R;
    const float4 al = slo[li], ah = shi[li];
    float best = __int_as_float(0x7f800000);
    int64_t bj = -1;
    for (int d = -PLOC_R; d <= PLOC_R; ++d) {
        int64_t j = i + d;
        if (d == 0 || j < 0 || j >= m) continue;
        float ar = merged_area(al, ah, slo[li + d], shi[li + d]);
        if (ar < best) { best = ar; bj = j; }  // ascending j: ties keep the smaller index
    }
    nn[i] = (int)bj;
}

// per-block (valid, merge) counts, interleaved: block_counts[2*b], block_counts[2*b+1]
__global__ void __launch_bounds__(PLOC_BLOCK) k_ploc_count(const int *__restrict__ nn, int64_t m, int *block_counts) {
    const int64_t i = (int64_t)blockIdx.x * PLOC_BLOCK + threadIdx.x;
    int valid = 0, merge = 0;
    if (i < m) {
        int j = nn[i];
        bool mutual = nn[j] == (int)i;
        merge = mutual && i < j;
        valid = !(mutual && i > j);
    }
    int v = __syncthreads_count(valid);
    int g = __syncthreads_count(merge);
    if (threadIdx.x == 0) { block_counts[2 * blockIdx.x] = v; block_counts[2 * blockIdx.x + 1] = g; }
}

// exclusive scan of the interleaved block counts in place; totals[0..1] = (valid, merges)
__global__ void __launch_bounds__(1024) k_ploc_scan(int *bc, int64_t nb, int *totals) {
    __shared__ int sv[1024], sg[1024];
    const int64_t chunk = (nb + 1023) / 1024;
    const int64_t b = threadIdx.x * chunk, e = min(nb, b + chunk);
    int v = 0, g = 0;
    for (int64_t k = b; k < e; ++k) { v += bc[2 * k]; g += bc[2 * k + 1]; }
    sv[threadIdx.x] = v;
    sg[threadIdx.x] = g;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        int tv = threadIdx.x >= (unsigned)o ? sv[threadIdx.x - o] : 0;
        int tg = threadIdx.x >= (unsigned)o ? sg[threadIdx.x - o] : 0;
        __syncthreads();
        sv[threadIdx.x] += tv;
        sg[threadIdx.x] += tg;
        __syncthreads();
    }
    int rv = threadIdx.x ? sv[threadIdx.x - 1] : 0, rg = threadIdx.x ? sg[threadIdx.x - 1] : 0;
    for (int64_t k = b; k < e; ++k) {
        int cv = bc[2 * k], cg = bc[2 * k + 1];
        bc[2 * k] = rv;
        bc[2 * k + 1] = rg;
        rv += cv;
        rg += cg;
    }
    if (threadIdx.x == 1023) { totals[0] = sv[1023]; totals[1] = sg[1023]; }
}

__global__ void __launch_bounds__(PLOC_BLOCK) k_ploc_write(const PlocArgs a, const int *__restrict__ C,
                                                           const int *__restrict__ nn, int64_t m,
                                                           const int *__restrict__ bo, int node_base, int *Cn) {
    __shared__ int wv[32], wg[32];
    const int64_t i = (int64_t)blockIdx.x * PLOC_BLOCK + threadIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int valid = 0, merge = 0, j = -1;
    if (i < m) {
        j = nn[i];
        bool mutual = nn[j] == (int)i;
        merge = mutual && i < j;
        valid = !(mutual && i > j);
    }
    const unsigned lt = (1u << lane) - 1u;
    unsigned bv = __ballot_sync(0xffffffffu, valid), bg = __ballot_sync(0xffffffffu, merge);
    if (lane == 0) { wv[warp] = __popc(bv); wg[warp] = __popc(bg); }
    __syncthreads();
    if (warp == 0) {
        int xv = wv[lane], xg = wg[lane];
        for (int o = 1; o < 32; o <<= 1) {
            int yv = __shfl_up_sync(0xffffffffu, xv, o), yg = __shfl_up_sync(0xffffffffu, xg, o);
            if (lane >= o) { xv += yv; xg += yg; }
        }
        wv[lane] = xv - wv[lane];
        wg[lane] = xg - wg[lane];
    }
    __syncthreads();
    if (i >= m || !valid) return;
    const int pos = bo[2 * blockIdx.x] + wv[warp] + __popc(bv & lt);
    const int ci = C[i];
    if (merge) {
        const int k = node_base + bo[2 * blockIdx.x + 1] + wg[warp] + __popc(bg & lt);
        const int cj = C[j];
        float4 al, ah, bl, bh;
        node_box(a, ci, al, ah);
        node_box(a, cj, bl, bh);
        a.nlo[k] = make_float4(fminf(al.x, bl.x), fminf(al.y, bl.y), fminf(al.z, bl.z), 0.0f);
        a.nhi[k] = make_float4(fmaxf(ah.x, bh.x), fmaxf(ah.y, bh.y), fmaxf(ah.z, bh.z), 0.0f);
        a.left[k] = ci;
        a.right[k] = cj;
        a.size[k] = (ci >= a.n - 1 ? 1 : a.size[ci]) + (cj >= a.n - 1 ? 1 : a.size[cj]);
        Cn[pos] = k;
    } else {
        Cn[pos] = ci;
    }
}

int64_t ploc_block_count(int64_t m) { return (m + PLOC_BLOCK - 1) / PLOC_BLOCK; }

void launch_ploc_init(int64_t n, int *clusters, cudaStream_t s) {
    if (n > 0) k_ploc_init<<<nblk(n, 256), 256, 0, s>>>(n, clusters);
}
void launch_ploc_nn(const PlocArgs &a, const int *clusters, int64_t m, int *nn, cudaStream_t s) {
    k_ploc_nn<<<nblk(m, PLOC_NN_BLOCK), PLOC_NN_BLOCK, 0, s>>>(a, clusters, m, nn);
}
void launch_ploc_count(const int *nn, int64_t m, int *block_counts, cudaStream_t s) {
    k_ploc_count<<<nblk(m, PLOC_BLOCK), PLOC_BLOCK, 0, s>>>(nn, m, block_counts);
}
void launch_ploc_scan(int *block_counts, int64_t nblocks, int *totals, cudaStream_t s) {
    k_ploc_scan<<<1, 1024, 0, s>>>(block_counts, nblocks, totals);
}
void launch_ploc_write(const PlocArgs &a, const int *clusters, const int *nn, int64_t m, const int *block_offsets,
                       int node_base, int *next_clusters, cudaStream_t s) {
    k_ploc_write<<<nblk(m, PLOC_BLOCK), PLOC_BLOCK, 0, s>>>(a, clusters, nn, m, block_offsets, node_base,
                                                           next_clusters);
}

}  // namespace dpr
