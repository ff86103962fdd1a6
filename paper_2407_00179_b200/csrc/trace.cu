// trace.cu -- the wavefront kernels of one lock-step step.
//
//   k_gen_primary   (a2) every rank generates the FULL primary wave-front of the batch and
//                   keeps the rays whose first candidate rank is itself -- "generate full
//                   wave-fronts on all ranks ... discard some of the rays ... by testing
//                   them for visibility against their geometry" (S2.2).
//   k_trace_path    (a3) closest hit against the rank's LBVH + bricks; persistent warps
//                   with per-lane ray replacement; result written into the record.
//   k_shade_path    (a4+a6) forward to the next candidate rank (P8) or resolve, shade (P6)
//                   and spawn shadow/AO/bounce rays into per-destination queues.
//   k_trace_occl    (a3) any hit; marks occluded records.
//   k_resolve_occl  (a4) drops occluded rays; forwards or resolves unoccluded ones.
// Queues are appended with warp-aggregated atomics (__match_any_sync per destination).
// All kernels read their input count from device memory, so launch shapes never depend on
// host-known counts.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"

namespace dpr {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// r = a * b + c on two lanes of a packed fp32x2 (sm_100 FFMA2), b and c broadcast
__device__ __forceinline__ void ffma2(float &r0, float &r1, float a0, float a1, float b, float c) {
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %4};\n\tmov.b64 rc, {%5, %5};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(r0), "=f"(r1)
        : "f"(a0), "f"(a1), "f"(b), "f"(c));
}

__device__ __forceinline__ void fb_add(float4 *p, float4 v) {
#if __CUDA_ARCH__ >= 900
    atomicAdd(p, v);
#else
    atomicAdd(&p->x, v.x); atomicAdd(&p->y, v.y); atomicAdd(&p->z, v.z); atomicAdd(&p->w, v.w);
#endif
}

// Framebuffer accumulation with a warp segmented reduction: lanes holding the same pixel in
// consecutive lanes (16 samples of a pixel share a warp) are summed by a shuffle scan and the
// last lane of each run issues ONE float4 atomic (same-address atomics would serialise).
// All 32 lanes must call; inactive lanes pass active = false.
__device__ __forceinline__ void fb_add_seg(float4 *fb, uint32_t p, float4 v, bool active) {
    if (!__any_sync(FULL, active)) return;  // warp-uniform
    const int lane = threadIdx.x & 31;
    const uint32_t key = active ? p : (0x80000000u | (uint32_t)lane);  // unique when inactive
    const uint32_t prev = __shfl_up_sync(FULL, key, 1);
    const unsigned heads = __ballot_sync(FULL, lane == 0 || prev != key);
    const int start = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));
    if (!active) v = make_float4(0, 0, 0, 0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        float x = __shfl_up_sync(FULL, v.x, o), y = __shfl_up_sync(FULL, v.y, o);
        float z = __shfl_up_sync(FULL, v.z, o), w = __shfl_up_sync(FULL, v.w, o);
        if (lane - o >= start) { v.x += x; v.y += y; v.z += z; v.w += w; }
    }
    const bool last = lane == 31 || ((heads >> (lane + 1)) & 1u);
    if (active && last) fb_add(fb + p, v);
}

// Warp-aggregated counter add keyed by an int (all lanes call).
__device__ __forceinline__ void warp_count(bool want, int key, unsigned long long *base) {
    unsigned act = __ballot_sync(FULL, want);
    if (want) {
        unsigned peers = __match_any_sync(act, key);
        if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&base[key], (unsigned long long)__popc(peers));
    }
}

// Block-aggregated queue append: all threads of the block must call it (block-uniform
// control flow).  One global atomicAdd per (block, destination) instead of one per warp:
// at N=1 every append targets the same counter, so per-warp atomics serialise in L2.
// smem: cnt[DPR_MAX_RANKS], base[DPR_MAX_RANKS] provided by the caller.
__device__ __forceinline__ uint32_t block_append(bool want, int dest, uint32_t *const *counts, uint32_t cap,
                                                 unsigned *overflow, unsigned long long *S_row,
                                                 unsigned long long *app_row,
                                                 int self, int nranks, uint32_t *s_cnt, uint32_t *s_base,
                                                 int sys_scope) {
    const int lane = threadIdx.x & 31;
    unsigned act = __ballot_sync(FULL, want);
    uint32_t off = 0;
    unsigned peers = 0;
    int leader = 0;
    if (want) {
        peers = __match_any_sync(act, dest);
        leader = __ffs(peers) - 1;
        if (lane == leader) off = atomicAdd(&s_cnt[dest], (uint32_t)__popc(peers));
        off = __shfl_sync(peers, off, leader) + __popc(peers & lanemask_lt());
    }
    // the first barrier also tells whether any thread of the block appends (block-uniform
    // early exit: nothing was added to s_cnt)
    if (!__syncthreads_or(want)) return 0xffffffffu;
    if ((int)threadIdx.x < nranks) {
        uint32_t c = s_cnt[threadIdx.x];
        uint32_t b = 0;
        if (c) {
            // fused exchange: the counter may live in a peer GPU's memory (NVLink)
            b = sys_scope ? atomicAdd_system(counts[threadIdx.x], c) : atomicAdd(counts[threadIdx.x], c);
            if (S_row && (int)threadIdx.x != self) atomicAdd(&S_row[threadIdx.x], (unsigned long long)c);
            atomicAdd(&app_row[threadIdx.x], (unsigned long long)c);
        }
        s_base[threadIdx.x] = b;
        s_cnt[threadIdx.x] = 0;
    }
    __syncthreads();
    if (!want) return 0xffffffffu;
    uint32_t pos = s_base[dest] + off;
    if (pos >= cap) {
        atomicOr(overflow, 1u);
        return 0xffffffffu;
    }
    return pos;
}

__device__ __forceinline__ void flush(unsigned long long *dst, uint32_t v) {
    v = __reduce_add_sync(FULL, v);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, (unsigned long long)v);
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// The P10 march of a queue of n rays runs in k_march_* (G lanes per ray) rather than inside
// the trace kernels when the rank has bricks, delta tracking is off and the queue is short.
__device__ __forceinline__ bool warp_march_dev(const StepArgs &A, uint32_t n) {
    return A.W.nbricks > 0 && !(A.F.flags & DPR_FLAG_DELTA) && n < A.F.march_inline_min;
}
// lanes per ray for such a queue: forced, or the smallest of 1, 4, 16 (run as 32) that gives
// every lane of the GPU two rays' worth of work; dispatched to the variants 1, 4, 8, 32
__host__ __device__ __forceinline__ int march_variant(int forced, uint32_t n, uint32_t inline_min) {
    int G = forced;
    if (G == 0) {
        G = 1;
        while (G < 32 && (int64_t)n * G < (int64_t)inline_min) G *= 4;
        if (G > 32) G = 32;
    }
    return G <= 1 ? 1 : (G <= 4 ? 4 : (G <= 8 ? 8 : 32));
}
// the occlusion trace resolves its rays itself (host-side conditions, and no k_march_occl)
__device__ __forceinline__ bool fuse_resolve_dev(const StepArgs &A, uint32_t n) {
    return A.F.fuse_resolve && !warp_march_dev(A, n);
}

// trace kernel start / end stamps of the current step (first start via max of ~t)
#ifndef DPR_STAMPS
#define DPR_STAMPS 1
#endif
__device__ __forceinline__ void stamp_kernel(const StepArgs &A, int kind, bool start) {
    if (!DPR_STAMPS || !A.rec || (threadIdx.x & 31) != 0 || (start && threadIdx.x != 0)) return;
    const uint32_t k = min(A.rec->step, (uint32_t)MAX_STEP_REC - 1);
    const unsigned long long t = gtimer();
    if (start) atomicMax(&A.rec->kt[k][kind][0], ~t);
    else atomicMax(&A.rec->kt[k][kind][1], t);
}

// ---------------------------------------------------------------------------------------
// a3: traversal of the rank's LBVH.  Result == brute force over the rank's prims with the P9
// rule (box tests are conservative: padded boxes, FMA slabs; they only decide what to
// skip).  Aila & Laine 2009 "while-while" loop with leaf postponing, run inside a persistent
// loop that REPLACES finished rays per lane (dynamic fetch), so a warp is not held by its
// slowest ray.  Results are written back into the ray record in place; routing / shading
// happen in the coherent resolve kernels that follow.
// ---------------------------------------------------------------------------------------
struct Hit {
    float t;
    uint32_t id;  // global id / VOL_BIT|i / NO_HIT
    int prim;     // local (sorted) prim index of a hit found at THIS rank, or -1
};

struct TraceCounters { uint32_t nodes, tris, sphs, vols; };

#ifndef DPR_REFILL_PATH
#define DPR_REFILL_PATH 24  // r02 re-sweep on configs[1]: 8 20.14, 16 19.85, 20 19.79, 24 19.79 ms frame
#endif
#ifndef DPR_REFILL_OCCL
#define DPR_REFILL_OCCL 4
#endif
// refill a warp's finished lanes once this many are idle (sweeps r01: closest-hit rays prefer
// bigger refill batches, any-hit rays smaller ones)
constexpr int REFILL_PATH = DPR_REFILL_PATH, REFILL_OCCL = DPR_REFILL_OCCL;
constexpr int WSTACK = 32;       // node-group stack entries (wide BVH depth bound)

#ifndef DPR_COOP
#define DPR_COOP 1
#endif
// Warp-cooperative prim tests: per pass every lane hands up to COOP_PER_LANE pending prims to
// a per-warp list that all 32 lanes test (against the owner lane's ray), then the results are
// reduced per owner in shared memory.
#ifndef DPR_COOP_PER_LANE
#define DPR_COOP_PER_LANE 16  // any-hit (r02 re-sweep, configs[1] occlusion trace: 8 13.88, 12 13.68,
                              // 16 13.61, 20 13.74, 24 13.74 ms)
#endif
#ifndef DPR_COOP_PER_LANE_PATH
#define DPR_COOP_PER_LANE_PATH 12  // closest-hit (r01 sweep)
#endif
constexpr int COOP_PER_LANE = DPR_COOP_PER_LANE > DPR_COOP_PER_LANE_PATH ? DPR_COOP_PER_LANE
                                                                         : DPR_COOP_PER_LANE_PATH;  // list size
constexpr int COOP_CAP_ANY = DPR_COOP_PER_LANE, COOP_CAP_PATH = DPR_COOP_PER_LANE_PATH;
#ifndef DPR_FFMA2
#define DPR_FFMA2 1
#endif
#ifndef DPR_ANY_REVERSE
#define DPR_ANY_REVERSE 1
#endif
#ifndef DPR_INLINE_DIST
#define DPR_INLINE_DIST 1
#endif
#ifndef DPR_WARP_MARCH
#define DPR_WARP_MARCH 1
#endif
#ifndef DPR_P1_EXIT_ANY
#define DPR_P1_EXIT_ANY 4
#endif
constexpr int P1_EXIT_ANY = DPR_P1_EXIT_ANY;
struct CoopSmem {
    uint32_t k[32 * COOP_PER_LANE];
    uint8_t ow[32 * COOP_PER_LANE];
    unsigned long long best[32];
};
constexpr int PRIM_BY_ID = 0x7fffffff;  // Hit.prim: a local hit found by id (record W.prims_in[local id])


// Traversal state of one ray over the compressed 8-wide BVH.  A "node group" is the set of
// not-yet-visited internal children of one visited node: (child_base, hit bits in traversal
// order s' = slot ^ octant, parent imask).  A "prim group" is a 32-bit mask of prims at
// prim_base.. of one visited node's hit leaves.
#ifndef DPR_RAY_SMEM
#define DPR_RAY_SMEM 1
#endif
#if DPR_RAY_SMEM
// Ray origin, direction and reciprocal direction live in shared memory (SoA, one slot per
// thread): 9 fewer registers per thread, and the cooperative prim tests read an owner's ray
// directly instead of shuffling it.
__shared__ float s_ray[9][TRACE_BLOCK];
__device__ __forceinline__ f3 ray_o(int t) { return mk(s_ray[0][t], s_ray[1][t], s_ray[2][t]); }
__device__ __forceinline__ f3 ray_d(int t) { return mk(s_ray[3][t], s_ray[4][t], s_ray[5][t]); }
__device__ __forceinline__ f3 ray_id(int t) { return mk(s_ray[6][t], s_ray[7][t], s_ray[8][t]); }
#define RAY_O(S) ray_o(threadIdx.x)
#define RAY_D(S) ray_d(threadIdx.x)
#define RAY_ID(S) ray_id(threadIdx.x)
#else
#define RAY_O(S) (S).o
#define RAY_D(S) (S).d
#define RAY_ID(S) (S).id3
#endif
#ifndef DPR_SM_STACK
#define DPR_SM_STACK 5  // r02 re-sweep with 256-thread CTAs: 3 19.89, 4 19.75, 5 19.64, 6 19.83 ms
#endif
#if DPR_SM_STACK > 0
// the first DPR_SM_STACK node-group stack entries of each thread in shared memory (SoA; sweep
// r01_smstack: 3 best at first, 14.67 -> 14.51 ms occlusion trace on configs[1]; 4 after the
// traversal-order table, r01_v12; 5 with 256-thread CTAs, r02), deeper entries in local memory
__shared__ uint2 s_stack[DPR_SM_STACK][TRACE_BLOCK];
#ifndef DPR_LEAF_BF
#define DPR_LEAF_BF 0
#endif
#ifndef DPR_PERM_LUT
#define DPR_PERM_LUT 1
#endif
#if DPR_PERM_LUT
// hit mask -> traversal order (bit i moves to bit i ^ order), one table of 256 per order
__shared__ uint8_t s_perm[8 * 256];
__device__ __forceinline__ void perm_init() {
    for (uint32_t i = threadIdx.x; i < 8 * 256; i += blockDim.x) {
        const uint32_t o = i >> 8, m = i & 255u;
        uint32_t r = 0;
        for (uint32_t b = 0; b < 8; ++b) r |= ((m >> b) & 1u) << (b ^ o);
        s_perm[i] = (uint8_t)r;
    }
    __syncthreads();
}
#endif
__device__ __forceinline__ void stack_push(uint2 *local, int &sp, uint2 v) {
    if (sp < DPR_SM_STACK) s_stack[sp][threadIdx.x] = v;
    else local[sp - DPR_SM_STACK] = v;
    ++sp;
}
__device__ __forceinline__ uint2 stack_pop(const uint2 *local, int &sp) {
    --sp;
    return sp < DPR_SM_STACK ? s_stack[sp][threadIdx.x] : local[sp - DPR_SM_STACK];
}
#else
__device__ __forceinline__ void stack_push(uint2 *local, int &sp, uint2 v) { local[sp++] = v; }
__device__ __forceinline__ uint2 stack_pop(const uint2 *local, int &sp) { return local[--sp]; }
#endif
struct TravState {
#if !DPR_RAY_SMEM
    f3 o, d, id3;
#endif
    float tmax;
    Hit h;
    uint32_t oct;
    uint2 ng;                  // x = child_base, y = hits (bits 0..7) | imask << 8
    uint32_t tb0, tm0;         // prim group being tested
    uint32_t tb1, tm1;         // speculative prim groups (filled while other lanes of the
    uint32_t tb2, tm2;         //   warp are still descending; sweep r01: 3 slots > 2 >> 1)
    int sp;
};

// rev = 7: children visited back to front (any-hit rays, DPR_ANY_REVERSE)
__device__ __forceinline__ void trav_init(TravState &S, f3 o, f3 d, float tmax, Hit h, int64_t nprims,
                                          uint32_t rev = 0) {
    S.tmax = tmax; S.h = h;
    const float tiny = 1e-20f;  // zero direction components -> finite reciprocal (box tests only)
    const f3 id3 = mk(1.0f / (fabsf(d.x) > tiny ? d.x : copysignf(tiny, d.x)),
                      1.0f / (fabsf(d.y) > tiny ? d.y : copysignf(tiny, d.y)),
                      1.0f / (fabsf(d.z) > tiny ? d.z : copysignf(tiny, d.z)));
#if DPR_RAY_SMEM
    const int t = threadIdx.x;
    s_ray[0][t] = o.x; s_ray[1][t] = o.y; s_ray[2][t] = o.z;
    s_ray[3][t] = d.x; s_ray[4][t] = d.y; s_ray[5][t] = d.z;
    s_ray[6][t] = id3.x; s_ray[7][t] = id3.y; s_ray[8][t] = id3.z;
#else
    S.o = o; S.d = d; S.id3 = id3;
#endif
    S.oct = (d.x < 0.0f ? 4u : 0u) | (d.y < 0.0f ? 2u : 0u) | (d.z < 0.0f ? 1u : 0u);
    S.oct |= (S.oct ^ rev) << 3;  // bits 3..5: traversal order (slot s' = position ^ order)
    // virtual root group: one internal child (slot 0, imask 1) at index 0
    S.ng = make_uint2(0u, nprims > 0 ? ((1u << (S.oct >> 3)) | (1u << 8)) : 0u);
    S.tb0 = S.tb1 = S.tb2 = 0;
    S.tm0 = S.tm1 = S.tm2 = 0;
    S.sp = 0;
}

__device__ __forceinline__ uint32_t pending_prims(const TravState &S) { return S.tm0 | S.tm1 | S.tm2; }

__device__ __forceinline__ void trav_clear(TravState &S) {
    S.ng.y = 0;
    S.sp = 0;
    S.tm0 = S.tm1 = S.tm2 = 0;
}

__device__ __forceinline__ bool trav_done(const TravState &S) {
    return (S.ng.y & 0xffu) == 0 && S.sp == 0 && pending_prims(S) == 0;
}


// One outer iteration, called by ALL 32 lanes (idle lanes have an empty state).  Phase 1
// visits nodes until every lane holds a prim group or has nothing left; phase 2 tests the
// prim groups.  Both loops are warp-uniform.  Returns true when the lane is finished.
template <bool ANY>
__device__ __forceinline__ bool trav_step(const WorldDev &W, TravState &S, uint2 *stack,
                                          TraceCounters &tc, unsigned *overflow, CoopSmem &cs) {
    for (;;) {
        // descend while some lane has no prim group yet; lanes that already hold one keep
        // descending speculatively into the second slot (keeps the phase-1 warp full)
        const bool work = (S.ng.y & 0xffu) != 0 || S.sp > 0;
        // any-hit rays leave phase 1 once at most P1_EXIT_ANY lanes still lack a prim group
        // (the cooperative phase 2 is cheap; sweep r01), closest-hit rays when none does
        const unsigned lacking = __ballot_sync(FULL, work && S.tm0 == 0);
        if (!lacking) break;
        if (ANY && __popc(lacking) <= P1_EXIT_ANY && __any_sync(FULL, pending_prims(S) != 0)) break;
#ifdef DPR_ANYFREE
        if (!(work && (S.tm0 == 0 || S.tm1 == 0 || S.tm2 == 0))) continue;
#else
        if (!(work && S.tm2 == 0)) continue;
#endif
        if ((S.ng.y & 0xffu) == 0) S.ng = stack_pop(stack, S.sp);
        uint32_t hits = S.ng.y & 0xffu, pimask = S.ng.y >> 8;
        int sp_ = __ffs(hits) - 1;
        hits &= hits - 1;
        int slot = sp_ ^ (int)(S.oct >> 3);
        int node = (int)S.ng.x + __popc(pimask & ((1u << slot) - 1u));
        if (hits) {
            if (S.sp < WSTACK) stack_push(stack, S.sp, make_uint2(S.ng.x, hits | (pimask << 8)));
            else atomicOr(overflow, 2u);
        }
        // visit the node: test its (up to) 8 children
#ifdef DPR_CHECKS
        if (node < 0 || node >= W.nnodes) { atomicOr(overflow, 4u); trav_clear(S); S.ng.y = 0; continue; }
#endif
        const WNode *nd = W.wnodes + node;
        float4 w0 = __ldg(&nd->w0);
        uint4 w1 = __ldg(&nd->w1), w2 = __ldg(&nd->w2), w3 = __ldg(&nd->w3), w4 = __ldg(&nd->w4);
        tc.nodes++;
        const uint32_t bits = __float_as_uint(w0.w);
        const uint32_t nimask = bits >> 24;
        // ray-space plane t = q*ps + po.  Bytes are read as f = 2^23 + q (one PRMT, exact), so
        // t = f*ps + (po - 2^23*ps); rounding that offset costs at most |ps|/2, so near planes
        // use offset - |ps| and far planes offset + |ps|: conservative by construction (the
        // remaining relative error is covered by the (|x|+4)*2^-18 box padding).
        const f3 rid = RAY_ID(S), ro = RAY_O(S);
        const float psx = __uint_as_float((bits & 0xffu) << 23) * rid.x;
        const float psy = __uint_as_float(((bits >> 8) & 0xffu) << 23) * rid.y;
        const float psz = __uint_as_float(((bits >> 16) & 0xffu) << 23) * rid.z;
        const float pox = __fmaf_rn(-8388608.0f, psx, (w0.x - ro.x) * rid.x);
        const float poy = __fmaf_rn(-8388608.0f, psy, (w0.y - ro.y) * rid.y);
        const float poz = __fmaf_rn(-8388608.0f, psz, (w0.z - ro.z) * rid.z);
        const float onx = pox - fabsf(psx), ofx = pox + fabsf(psx);
        const float ony = poy - fabsf(psy), ofy = poy + fabsf(psy);
        const float onz = poz - fabsf(psz), ofz = poz + fabsf(psz);
        // near/far planes per axis by ray direction sign
        uint32_t nx0 = w2.x, nx1 = w2.y, fx0 = w3.z, fx1 = w3.w;
        uint32_t ny0 = w2.z, ny1 = w2.w, fy0 = w4.x, fy1 = w4.y;
        uint32_t nz0 = w3.x, nz1 = w3.y, fz0 = w4.z, fz1 = w4.w;
        // sign of the reciprocal == sign of the direction == octant bit
        if (S.oct & 4u) { uint32_t t0 = nx0, t1 = nx1; nx0 = fx0; nx1 = fx1; fx0 = t0; fx1 = t1; }
        if (S.oct & 2u) { uint32_t t0 = ny0, t1 = ny1; ny0 = fy0; ny1 = fy1; fy0 = t0; fy1 = t1; }
        if (S.oct & 1u) { uint32_t t0 = nz0, t1 = nz1; nz0 = fz0; nz1 = fz1; fz0 = t0; fz1 = t1; }
        const float bound = ANY ? S.tmax : S.h.t;
        uint32_t hitm = 0;
#pragma unroll
        const uint32_t k4b = W.prmt_hi;
#if DPR_FFMA2
        // two children per packed fp32x2 FMA (FFMA2: one issue slot, two independently
        // rounded FMAs -- the same values as two __fmaf_rn)
        for (int c = 0; c < 8; c += 2) {
            const uint32_t s0 = (uint32_t)(c & 3) | 0x5440u, s1 = (uint32_t)((c + 1) & 3) | 0x5440u;
            float tnx[2], tfx[2], tny[2], tfy[2], tnz[2], tfz[2];
#define DPR_PLANE2(OUT, W0, W1, PS, PO)                                                                    \
            ffma2(OUT[0], OUT[1], __uint_as_float(__byte_perm(c < 4 ? W0 : W1, k4b, s0)),                 \
                  __uint_as_float(__byte_perm(c < 4 ? W0 : W1, k4b, s1)), PS, PO)
            DPR_PLANE2(tnx, nx0, nx1, psx, onx);
            DPR_PLANE2(tfx, fx0, fx1, psx, ofx);
            DPR_PLANE2(tny, ny0, ny1, psy, ony);
            DPR_PLANE2(tfy, fy0, fy1, psy, ofy);
            DPR_PLANE2(tnz, nz0, nz1, psz, onz);
            DPR_PLANE2(tfz, fz0, fz1, psz, ofz);
#undef DPR_PLANE2
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float tn = fmaxf(fmaxf(tnx[h], tny[h]), fmaxf(tnz[h], 0.0f));
                const float tf = fminf(fminf(tfx[h], tfy[h]), fminf(tfz[h], bound));
                hitm |= (tn <= tf ? 1u : 0u) << (c + h);
            }
        }
#else
        for (int c = 0; c < 8; ++c) {
            const uint32_t sel = (uint32_t)(c & 3) | 0x5440u;
            float tnx = __fmaf_rn(__uint_as_float(__byte_perm(c < 4 ? nx0 : nx1, k4b, sel)), psx, onx);
            float tfx = __fmaf_rn(__uint_as_float(__byte_perm(c < 4 ? fx0 : fx1, k4b, sel)), psx, ofx);
            float tny = __fmaf_rn(__uint_as_float(__byte_perm(c < 4 ? ny0 : ny1, k4b, sel)), psy, ony);
            float tfy = __fmaf_rn(__uint_as_float(__byte_perm(c < 4 ? fy0 : fy1, k4b, sel)), psy, ofy);
            float tnz = __fmaf_rn(__uint_as_float(__byte_perm(c < 4 ? nz0 : nz1, k4b, sel)), psz, onz);
            float tfz = __fmaf_rn(__uint_as_float(__byte_perm(c < 4 ? fz0 : fz1, k4b, sel)), psz, ofz);
            float tn = fmaxf(fmaxf(tnx, tny), fmaxf(tnz, 0.0f));
            float tf = fminf(fminf(tfx, tfy), fminf(tfz, bound));
            hitm |= (tn <= tf ? 1u : 0u) << c;
        }
#endif
        // leaf slots (build time mask in the top nibbles of child_base / prim_base)
        const uint32_t leafm = (w1.x >> 28) | ((w1.y >> 24) & 0xf0u);
        uint32_t ih = hitm & nimask;
        uint32_t lh = hitm & leafm;
        // internal hits into traversal order s' = slot ^ octant (bit permutation)
#if DPR_PERM_LUT
        ih = s_perm[((S.oct >> 3) << 8) | ih];
#else
        const uint32_t ordm = S.oct >> 3;
        if (ordm & 4u) ih = ((ih & 0x0fu) << 4) | ((ih & 0xf0u) >> 4);
        if (ordm & 2u) ih = ((ih & 0x33u) << 2) | ((ih & 0xccu) >> 2);
        if (ordm & 1u) ih = ((ih & 0x55u) << 1) | ((ih & 0xaau) >> 1);
#endif
        uint32_t ihits = ih, tmask = 0;
#if DPR_LEAF_BF
        if (lh) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const uint32_t meta = __byte_perm(c < 4 ? w1.z : w1.w, 0u, (uint32_t)(c & 3));
                const uint32_t m = ((2u << ((meta >> 5) & 3u)) - 1u) << (meta & 31u);
                tmask |= (lh & (1u << c)) ? m : 0u;
            }
            lh = 0;
        }
#endif
        while (lh) {
            const int c = __ffs(lh) - 1;
            lh &= lh - 1;
            // byte c of {w1.z, w1.w} in the low byte (one PRMT); only bits 0..6 are read below
            const uint32_t meta = __byte_perm(w1.z, w1.w, (uint32_t)c);
            tmask |= ((2u << ((meta >> 5) & 3u)) - 1u) << (meta & 31u);
        }
        S.ng = make_uint2(w1.x & 0x0fffffffu, ihits | (nimask << 8));
        if (tmask) {
            const uint32_t pb = w1.y & 0x0fffffffu;
            if (S.tm0 == 0) { S.tb0 = pb; S.tm0 = tmask; }
            else if (S.tm1 == 0) { S.tb1 = pb; S.tm1 = tmask; }
            else { S.tb2 = pb; S.tm2 = tmask; }
        }
    }
#if DPR_COOP
    // phase 2, warp-cooperative: the pending prims of all lanes are tested by all lanes; the
    // P9 rule is a total order on (t, global id), so the per-owner minimum is independent of
    // the order and of which lane tested what (any-hit: an OR).
    const int lane = threadIdx.x & 31;
    while (__any_sync(FULL, pending_prims(S) != 0)) {
        const int c = min(__popc(S.tm0) + __popc(S.tm1) + __popc(S.tm2), ANY ? COOP_CAP_ANY : COOP_CAP_PATH);
        int x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, x, o);
            if (lane >= o) x += y;
        }
        const int T = __shfl_sync(FULL, x, 31);
        int pos = x - c;
        for (int j = 0; j < c; ++j) {
            if (S.tm0 == 0) {
                if (S.tm1 != 0) { S.tb0 = S.tb1; S.tm0 = S.tm1; S.tm1 = 0; }
                else { S.tb0 = S.tb2; S.tm0 = S.tm2; S.tm2 = 0; }
            }
            cs.k[pos] = S.tb0 + (uint32_t)(__ffs(S.tm0) - 1);
            cs.ow[pos] = (uint8_t)lane;
            ++pos;
            S.tm0 &= S.tm0 - 1;
        }
        cs.best[lane] = ANY ? 0ull : ~0ull;
        __syncwarp();
        for (int g0 = 0; g0 < T; g0 += 32) {
            const int g = g0 + lane;
            const bool act = g < T;
            int k = act ? (int)cs.k[g] : 0;
#ifdef DPR_CHECKS
            if (act && (k < 0 || k >= W.nprims)) { atomicOr(overflow, 4u); k = 0; }
#endif
            const int ow = act ? (int)cs.ow[g] : lane;
#if DPR_RAY_SMEM
            const int wb = threadIdx.x & ~31;
            const f3 o = ray_o(wb + ow), d = ray_d(wb + ow);
#else
            const f3 o = mk(__shfl_sync(FULL, S.o.x, ow), __shfl_sync(FULL, S.o.y, ow), __shfl_sync(FULL, S.o.z, ow));
            const f3 d = mk(__shfl_sync(FULL, S.d.x, ow), __shfl_sync(FULL, S.d.y, ow), __shfl_sync(FULL, S.d.z, ow));
#endif
            const float tmax = __shfl_sync(FULL, S.tmax, ow);
            if (!act) continue;
            const float4 *pr = W.prims + 3 * (int64_t)k;
            const float4 a = __ldg(pr);
            const uint32_t idw = __float_as_uint(a.w);
            float t;
            bool ok;
            if (idw & SPHERE_BIT) {
                const float4 b = __ldg(pr + 1);
                tc.sphs++;
                ok = sphere_hit(o, d, tmax, xyz(a), b.x, t);
            } else {
                const float4 b = __ldg(pr + 1), e = __ldg(pr + 2);
                tc.tris++;
                ok = tri_hit(o, d, tmax, xyz(a), xyz(b), xyz(e), t);
            }
            if (!ok) continue;
            if (ANY) cs.best[ow] = 1ull;
            else atomicMin(&cs.best[ow], ((unsigned long long)__float_as_uint(t) << 32) |
                                             (unsigned long long)(W.id_base + (idw & ~SPHERE_BIT)));
        }
        __syncwarp();
        const unsigned long long b = cs.best[lane];
        __syncwarp();  // every lane has read its result before the next pass reuses the list
        if (ANY) {
            if (b) {
                S.h.prim = PRIM_BY_ID;
                trav_clear(S);
            }
        } else if (b != ~0ull) {
            const float t = __uint_as_float((uint32_t)(b >> 32));
            const uint32_t gid = (uint32_t)b;
            if (t < S.h.t || (t == S.h.t && gid < S.h.id)) {
                S.h.t = t;
                S.h.id = gid;
                S.h.prim = PRIM_BY_ID;
            }
        }
    }
#else
    // phase 2: prim groups (one prim per lane per iteration)
    while (__any_sync(FULL, pending_prims(S) != 0)) {
        if (S.tm0 == 0) {  // take the next pending group (any order is exact)
            if (S.tm1 != 0) { S.tb0 = S.tb1; S.tm0 = S.tm1; S.tm1 = 0; }
            else if (S.tm2 != 0) { S.tb0 = S.tb2; S.tm0 = S.tm2; S.tm2 = 0; }
            else continue;
        }
        int k = (int)S.tb0 + __ffs(S.tm0) - 1;
        S.tm0 &= S.tm0 - 1;
        const float4 *pr = W.prims + 3 * (int64_t)k;
        float4 a = __ldg(pr);
        uint32_t idw = __float_as_uint(a.w);
        float t;
        bool ok;
        if (idw & SPHERE_BIT) {
            float4 b = __ldg(pr + 1);
            tc.sphs++;
            ok = sphere_hit(RAY_O(S), RAY_D(S), S.tmax, xyz(a), b.x, t);
        } else {
            float4 b = __ldg(pr + 1), e = __ldg(pr + 2);
            tc.tris++;
            ok = tri_hit(RAY_O(S), RAY_D(S), S.tmax, xyz(a), xyz(b), xyz(e), t);
        }
        if (!ok) continue;
        if (ANY) {
            S.h.prim = k;
            trav_clear(S);
            continue;
        }
        uint32_t gid = W.id_base + (idw & ~SPHERE_BIT);
        if (t < S.h.t || (t == S.h.t && gid < S.h.id)) {
            S.h.t = t;
            S.h.id = gid;
            S.h.prim = k;
        }
    }
#endif
    return trav_done(S);
}

__device__ __forceinline__ f3 prim_normal(const float4 *prims, int64_t k, f3 o, f3 d, float t) {
    const float4 *pr = prims + 3 * k;
    float4 a = __ldg(pr), b = __ldg(pr + 1);
    if (__float_as_uint(a.w) & SPHERE_BIT) return sphere_normal(o, d, t, xyz(a), b.x);
    float4 e = __ldg(pr + 2);
    return tri_normal(xyz(b), xyz(e), d);
}

// ---------------------------------------------------------------------------------------
// P10 brick march (identical sample set and decisions to the oracle's per-rank march).
// ---------------------------------------------------------------------------------------
template <bool ANY>
__device__ __forceinline__ bool march_brick(const BrickDev &B, f3 o, f3 d, float tmax, float bound,
                                            float dt, uint64_t seed, uint32_t p, uint32_t s,
                                            uint32_t depth, uint32_t purpose, uint32_t subhi,
                                            float &t_out, uint32_t &i_out, f3 &rgb_out,
                                            uint32_t &nsamples) {
    float plo[3], phi[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) { plo[c] = B.box_lo[c] - B.h[c]; phi[c] = B.box_hi[c] + B.h[c]; }
    float t0, t1;
    if (!slab(plo, phi, o, d, tmax, t0, t1)) return false;
    float a = floorf(t0 / dt - 0.5f);
    float bb = ceilf(t1 / dt);
    if (bb > 1.0e9f) bb = 1.0e9f;
    // 32-bit sample indices (|i| <= 1e9 + 1 by the clamp above; a < 0 clamps to 0): the same
    // values and the same float conversions as 64-bit ones, without the 64-bit convert
    int i0 = a > 0.0f ? (int)fminf(a, 2.0e9f) - 1 : 0;  // a > 2e9: i0 > i1, no sample (as int64)
    const int i1 = (int)bb + 1;
    const int nx = B.hi[0] - B.lo[0] + 1, ny = B.hi[1] - B.lo[1] + 1;
    const float glx = (float)B.lo[0], ghx = (float)B.hi[0], gly = (float)B.lo[1], ghy = (float)B.hi[1],
                glz = (float)B.lo[2], ghz = (float)B.hi[2];
    uint4 rr = make_uint4(0, 0, 0, 0);
    int rblk = -1;
    for (int i = i0; i <= i1; ++i) {
        float ti = ((float)i + 0.5f) * dt;  // sample_t
        if (!(ti < bound)) return false;
        f3 pt = mk(o.x + ti * d.x, o.y + ti * d.y, o.z + ti * d.z);
        f3 g = grid_coord(B, pt);
        if (!(g.x >= glx && g.x < ghx && g.y >= gly && g.y < ghy && g.z >= glz && g.z < ghz)) continue;
        float fx0 = floorf(g.x), fy0 = floorf(g.y), fz0 = floorf(g.z);
        int ix = (int)fx0 - B.lo[0], iy = (int)fy0 - B.lo[1], iz = (int)fz0 - B.lo[2];
        const int mx = (int)((unsigned)ix / MC_SIZE), my = (int)((unsigned)iy / MC_SIZE), mz = (int)((unsigned)iz / MC_SIZE);  // >= 0 here
#if DPR_INLINE_DIST
        // macrocell distance field: every macrocell within Chebyshev distance dist-1 is empty
        const int dist = __ldg(B.mcd + (mz * B.mc_dims[1] + my) * B.mc_dims[0] + mx);
        if (dist > 0) {
            float mlo[3], mhi[3];
            const int mc3[3] = {mx, my, mz};
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const int c0 = max(B.lo[c] + (mc3[c] - (dist - 1)) * MC_SIZE, B.lo[c]);
                const int c1 = min(B.lo[c] + (mc3[c] + dist) * MC_SIZE, B.hi[c]);
                mlo[c] = B.O[c] + (float)c0 * B.h[c];
                mhi[c] = B.O[c] + (float)c1 * B.h[c];
            }
#else
        if (!__ldg(B.mc + (mz * B.mc_dims[1] + my) * B.mc_dims[0] + mx)) {
            // alpha == 0 for every sample in this macrocell: skipping is exact.  Jump to one
            // sample before the ray leaves the macrocell's box (the margin of >= 1 voxel
            // absorbs the rounding of t -> p -> g); the per-sample tests resume there.
            float mlo[3], mhi[3];
            const int mc3[3] = {mx, my, mz};
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                int c0 = B.lo[c] + mc3[c] * MC_SIZE, c1 = min(c0 + MC_SIZE, B.hi[c]);
                mlo[c] = B.O[c] + (float)c0 * B.h[c];
                mhi[c] = B.O[c] + (float)c1 * B.h[c];
            }
#endif
            float m0, m1;
            slab(mlo, mhi, o, d, tmax, m0, m1);
            // (int64)jf - 2 as before for jf < 2e9 (NaN converts to 0 either way); beyond, past i1
            const float jf = floorf(m1 / dt - 0.5f);
            const int jump = !(jf >= 2.0e9f) ? (int)jf - 2 : i1;
            if (jump > i) i = jump;  // loop ++i resumes at jump + 1
            continue;
        }
        nsamples++;
        float fx = g.x - fx0, fy = g.y - fy0, fz = g.z - fz0;
        const float *v = B.vox + (int64_t)ix + (int64_t)nx * (iy + ny * iz);  // ny * nz < 2^31 (dpr.h brick limits)
        const int64_t sy = nx, sz = (int64_t)nx * ny;
        float v000 = __ldg(v), v100 = __ldg(v + 1), v010 = __ldg(v + sy), v110 = __ldg(v + sy + 1);
        float v001 = __ldg(v + sz), v101 = __ldg(v + sz + 1), v011 = __ldg(v + sz + sy),
              v111 = __ldg(v + sz + sy + 1);
        float c00 = lerpf(v000, v100, fx), c10 = lerpf(v010, v110, fx);
        float c01 = lerpf(v001, v101, fx), c11 = lerpf(v011, v111, fx);
        float c0 = lerpf(c00, c10, fy), c1 = lerpf(c01, c11, fy);
        float sv = lerpf(c0, c1, fz);
        f3 rgb;
        float alpha = tf_alpha_rgb(B, sv, ANY ? nullptr : &rgb);
        if ((i >> 2) != rblk) {
            rblk = i >> 2;
            rr = rng4(seed, p, s, depth, purpose, subhi | (uint32_t)(i >> 2));
        }
        uint32_t x = (i & 3) == 0 ? rr.x : ((i & 3) == 1 ? rr.y : ((i & 3) == 2 ? rr.z : rr.w));
        if (u01(x) < alpha) {
            t_out = ti;
            i_out = (uint32_t)i;
            if (!ANY) rgb_out = rgb;
            return true;
        }
    }
    return false;
}

// ---------------------------------------------------------------------------------------
// The same P10 march in its own kernel (k_march_*, after the surface trace has written
// bestT / the occlusion flag into the record), G lanes per ray.  The per-lane march inside
// the traversal kernels held a warp for its longest ray and paid two dependent memory round
// trips (macrocell byte, then 8 voxels) per sample and one per 16-voxel empty-space jump.
// Here:
//  * a group of G lanes marches one ray in chunks of 4G samples: lane l of the group
//    evaluates samples cb+4l .. cb+4l+3 (one Philox block per lane: P1 counter sub =
//    subhi | i>>2, word i&3); the macrocell loads of a chunk, then its voxel loads, are in
//    flight together, and the first colliding sample of the chunk is the lowest (ballot);
//  * empty space is skipped with a macrocell distance field: d = Chebyshev distance (in
//    macrocells, capped) to the nearest macrocell that may have alpha > 0, so the ray jumps
//    to the exit of the (2d-1)^3-macrocell box of empty cells around it (alpha == 0 for every
//    owned sample in it: exact);
//  * a group whose ray finished fetches the next ray (persistent loop), so no group waits for
//    another group's ray.
// Sample set, arithmetic and decisions are those of march_brick and the oracle's march:
// the range [i0, i1], owned samples only, skipped samples only where alpha is 0, stop at
// t_i >= bound; a path ray's result is the first collision over the rank's bricks.
// ---------------------------------------------------------------------------------------
struct MarchRay {
    f3 o, d;
    float tmax, bound;
    uint32_t p, s, depth, purpose, subhi;
    int bi;               // current brick (nbricks = finished)
    int64_t i, i1;        // next sample, last sample of the current brick's range
    bool hit;
    uint32_t hid;         // VOL_BIT | i of the collision
    f3 rgb;
};

// Advance to the first brick (from r.bi on) whose padded box the ray crosses; set its range.
__device__ __forceinline__ void march_begin_brick(const WorldDev &W, MarchRay &r, float dt) {
    for (; r.bi < W.nbricks; ++r.bi) {
        const BrickDev &B = W.bricks[r.bi];
        float plo[3], phi[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) { plo[c] = B.box_lo[c] - B.h[c]; phi[c] = B.box_hi[c] + B.h[c]; }
        float t0, t1;
        if (!slab(plo, phi, r.o, r.d, r.tmax, t0, t1)) continue;
        float a = floorf(t0 / dt - 0.5f);
        float bb = ceilf(t1 / dt);
        if (bb > 1.0e9f) bb = 1.0e9f;
        const int64_t i0 = (int64_t)a - 1;
        r.i = i0 < 0 ? 0 : i0;
        r.i1 = (int64_t)bb + 1;
        return;
    }
}

template <bool ANY, int G>
__device__ __forceinline__ void march_groups(const StepArgs &A) {
    const FrameDev &F = A.F;
    const WorldDev &W = A.W;
    const float dt = F.dt;
    const int lane = threadIdx.x & 31, gl = lane % G, gbase = lane - gl;
    const uint32_t n_in = A.Q.in_count[ANY ? 1 : 0];
    // this queue is marched here, by this variant (block-uniform exit otherwise)
    if (!warp_march_dev(A, n_in) || march_variant(F.march_g, n_in, F.march_inline_min) != G) return;
    uint32_t *fetch = A.Q.fetch + (ANY ? 3 : 2);
    uint32_t vols = 0;
    MarchRay r;
    r.bi = 0; r.i = 0; r.i1 = -1; r.hit = false; r.hid = 0; r.rgb = mk(0, 0, 0);
    r.o = r.d = mk(0, 0, 0); r.tmax = r.bound = 0.0f; r.p = r.s = r.depth = r.purpose = r.subhi = 0;
    bool alive = false, exhausted = false;
    uint32_t idx = 0;
    for (;;) {
        // refill: the leaders of finished groups fetch one ray each
        const unsigned dl = __ballot_sync(FULL, !alive && gl == 0);
        if (!exhausted && dl) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(fetch, (uint32_t)__popc(dl));
            base = __shfl_sync(FULL, base, 0);
            if (base + (uint32_t)__popc(dl) >= n_in) exhausted = true;
            const uint32_t mine = base + __popc(dl & lanemask_lt());
            const uint32_t gidx = __shfl_sync(FULL, mine, gbase);
            if (!alive && gidx < n_in) {
                idx = gidx;
                alive = true;
                r.bi = 0; r.hit = false; r.hid = 0; r.rgb = mk(0, 0, 0);
                if (ANY) {
                    const OcclRec *q = A.Q.occl_in + idx;
                    const float4 a = __ldcg(&q->a), b = __ldcg(&q->b), c = __ldcg(&q->c);
                    const uint32_t meta = __float_as_uint(c.w), slot = meta >> 24;
                    r.o = xyz(a); r.d = xyz(b); r.tmax = a.w; r.bound = a.w;
                    r.p = __float_as_uint(b.w); r.s = meta & 0xffffu; r.depth = (meta >> 16) & 0xffu;
                    r.purpose = slot == 0 ? PUR_VOL_SHADOW : PUR_VOL_AO;
                    r.subhi = slot == 0 ? 0u : ((slot - 1) << 24);
                    if (!(a.w >= 0.0f)) r.bi = W.nbricks;  // occluded by a surface: nothing to do
                } else {
                    const PathRec *q = A.Q.path_in + idx;
                    const float4 a = __ldcg(&q->a), b = __ldcg(&q->b), c = __ldcg(&q->c), e = __ldcg(&q->e);
                    const uint32_t meta = __float_as_uint(e.w);
                    r.o = xyz(a); r.d = xyz(b); r.tmax = __int_as_float(0x7f800000); r.bound = a.w;
                    r.p = __float_as_uint(c.w); r.s = meta & 0xffffu; r.depth = (meta >> 16) & 0xffu;
                    r.purpose = PUR_VOL_PATH; r.subhi = 0u;
                }
                march_begin_brick(W, r, dt);
            }
        }
        if (!__any_sync(FULL, alive)) {
            if (exhausted) break;
            continue;
        }
        // group-uniform state check (every lane of a group computes the same): 0 idle,
        // 1 chunk, 2 current brick finished
        int mode = 0;
        if (alive) mode = (r.bi >= W.nbricks || r.i > r.i1 || !(sample_t(r.i, dt) < r.bound)) ? 2 : 1;
        // chunk: samples cb .. cb+4G-1 (those in [i, i1] with t < bound, owned, in a macrocell
        // that may have alpha > 0); every lane takes part in the ballot and shuffles below
        const int64_t cb = r.i & ~(int64_t)3;
        const int64_t jl = cb + 4 * gl;
        int hk = 4;                  // first colliding sample of this lane (4: none)
        uint32_t cnt = 0;            // samples this lane evaluated (before / at its collision)
        float th = 0.0f;
        f3 rgbh = mk(0, 0, 0);
        int64_t inext = cb + 4 * G;  // next sample (decided by the group's last lane)
        if (mode == 1) {
            const BrickDev &B = W.bricks[r.bi];
            const int nx = B.hi[0] - B.lo[0] + 1, ny = B.hi[1] - B.lo[1] + 1;
            const int64_t sy = nx, sz = (int64_t)nx * ny;
            bool val[4], own3 = false;
            int dist3 = 0, mc3[3] = {0, 0, 0};
            float tk[4], fx[4], fy[4], fz[4];
            const float *vp[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t j = jl + k;
                tk[k] = sample_t(j, dt);
                const f3 pt = mk(r.o.x + tk[k] * r.d.x, r.o.y + tk[k] * r.d.y, r.o.z + tk[k] * r.d.z);
                const f3 g = grid_coord(B, pt);
                const bool own = g.x >= (float)B.lo[0] && g.x < (float)B.hi[0] && g.y >= (float)B.lo[1] &&
                                 g.y < (float)B.hi[1] && g.z >= (float)B.lo[2] && g.z < (float)B.hi[2];
                const float fx0 = floorf(g.x), fy0 = floorf(g.y), fz0 = floorf(g.z);
                fx[k] = g.x - fx0; fy[k] = g.y - fy0; fz[k] = g.z - fz0;
                const int ix = own ? (int)fx0 - B.lo[0] : 0, iy = own ? (int)fy0 - B.lo[1] : 0,
                          iz = own ? (int)fz0 - B.lo[2] : 0;
                vp[k] = B.vox + (int64_t)ix + sy * iy + sz * iz;
                // distance 0 <=> the macrocell may have alpha > 0 (else the sample is skipped: exact)
                const int dist =
                    own ? (int)__ldg(B.mcd + ((iz / MC_SIZE) * B.mc_dims[1] + iy / MC_SIZE) * B.mc_dims[0] + ix / MC_SIZE)
                        : 0;
                val[k] = own && dist == 0 && j >= r.i && j <= r.i1 && tk[k] < r.bound;
                if (k == 3) {
                    own3 = own; dist3 = dist;
                    mc3[0] = ix / MC_SIZE; mc3[1] = iy / MC_SIZE; mc3[2] = iz / MC_SIZE;
                }
            }
            if (val[0] || val[1] || val[2] || val[3]) {
                const uint4 rr = rng4(F.seed, r.p, r.s, r.depth, r.purpose, r.subhi | (uint32_t)(jl >> 2));
                float v[4][8];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float *q = val[k] ? vp[k] : B.vox;
                    v[k][0] = __ldg(q); v[k][1] = __ldg(q + 1); v[k][2] = __ldg(q + sy); v[k][3] = __ldg(q + sy + 1);
                    v[k][4] = __ldg(q + sz); v[k][5] = __ldg(q + sz + 1); v[k][6] = __ldg(q + sz + sy);
                    v[k][7] = __ldg(q + sz + sy + 1);
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (!val[k] || hk < 4) continue;
                    cnt++;
                    const float c00 = lerpf(v[k][0], v[k][1], fx[k]), c10 = lerpf(v[k][2], v[k][3], fx[k]);
                    const float c01 = lerpf(v[k][4], v[k][5], fx[k]), c11 = lerpf(v[k][6], v[k][7], fx[k]);
                    const float c0 = lerpf(c00, c10, fy[k]), c1 = lerpf(c01, c11, fy[k]);
                    f3 rgb;
                    const float alpha = tf_alpha_rgb(B, lerpf(c0, c1, fz[k]), ANY ? nullptr : &rgb);
                    const uint32_t x = k == 0 ? rr.x : (k == 1 ? rr.y : (k == 2 ? rr.z : rr.w));
                    if (u01(x) < alpha) {
                        hk = k;
                        th = tk[k];
                        if (!ANY) rgbh = rgb;
                    }
                }
            }
            if (gl == G - 1 && own3 && dist3 > 0) {
                // the chunk's last sample lies in empty space: every macrocell within Chebyshev
                // distance dist3-1 of its own is empty, so continue one sample before the ray
                // leaves that box (the margin of march_brick's jump)
                float mlo[3], mhi[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const int c0 = max(B.lo[c] + (mc3[c] - (dist3 - 1)) * MC_SIZE, B.lo[c]);
                    const int c1 = min(B.lo[c] + (mc3[c] + dist3) * MC_SIZE, B.hi[c]);
                    mlo[c] = B.O[c] + (float)c0 * B.h[c];
                    mhi[c] = B.O[c] + (float)c1 * B.h[c];
                }
                float m0, m1;
                slab(mlo, mhi, r.o, r.d, r.tmax, m0, m1);
                const int64_t jump = (int64_t)floorf(m1 / dt - 0.5f) - 2;
                if (jump + 1 > inext) inext = jump + 1;
            }
        }
        // the group's first collision: its lowest lane with a hit
        const unsigned hm_all = __ballot_sync(FULL, hk < 4);
        const unsigned hm = G == 32 ? hm_all : (hm_all >> gbase) & ((1u << G) - 1u);
        const int hl = hm ? __ffs(hm) - 1 : G;
        const int src = gbase + (hm ? hl : 0);
        const float t_hit = __shfl_sync(FULL, th, src);
        const int k_hit = __shfl_sync(FULL, hk, src);
        f3 rgb_hit = mk(0, 0, 0);
        if (!ANY) rgb_hit = mk(__shfl_sync(FULL, rgbh.x, src), __shfl_sync(FULL, rgbh.y, src),
                               __shfl_sync(FULL, rgbh.z, src));
        const int64_t inext_g = G == 1 ? inext : (int64_t)(((uint64_t)__shfl_sync(FULL, (uint32_t)((uint64_t)inext >> 32), gbase + G - 1) << 32) |
                                                           __shfl_sync(FULL, (uint32_t)inext, gbase + G - 1));
        if (mode == 1) {
            if (gl <= hl) vols += cnt;
            if (hm) {
                // collision in this brick: a path ray keeps it as the new bound and goes on with
                // the next brick (only earlier samples can still win); an occlusion ray is done
                r.hit = true;
                r.hid = VOL_BIT | (uint32_t)(cb + 4 * hl + k_hit);
                r.rgb = rgb_hit;
                r.bound = t_hit;
                mode = 2;
                if (ANY) r.bi = W.nbricks;
            } else {
                r.i = inext_g;
            }
        }
        if (mode == 2) {
            if (r.bi < W.nbricks) {
                ++r.bi;
                march_begin_brick(W, r, dt);
            }
            if (r.bi >= W.nbricks) {
                // ray finished: write the result (group leader)
                if (gl == 0 && r.hit) {
                    if (ANY) {
                        A.Q.occl_in[idx].a.w = -1.0f;
                    } else {
                        PathRec *q = A.Q.path_in + idx;
                        q->a.w = r.bound;
                        q->b.w = __uint_as_float(r.hid);
                        q->e.x = r.rgb.x; q->e.y = r.rgb.y; q->e.z = r.rgb.z;
                    }
                }
                alive = false;
            }
        }
    }
    flush(&A.ctr->kc[ANY ? 1 : 0].vols, vols);
}

#ifndef DPR_MARCH_G
#define DPR_MARCH_G 0  // 0: chosen per launch from the ray count
#endif
#ifndef DPR_MARCH_MINB
#define DPR_MARCH_MINB 2
#endif
template <int G>
__global__ void __launch_bounds__(256, DPR_MARCH_MINB) k_march_path(const __grid_constant__ StepArgs A) { march_groups<false, G>(A); }
template <int G>
__global__ void __launch_bounds__(256, DPR_MARCH_MINB) k_march_occl(const __grid_constant__ StepArgs A) { march_groups<true, G>(A); }

// ---------------------------------------------------------------------------------------
// Delta tracking (NEXT f4; readings R-DELTA, R-LOG), the alternative to the P10 march:
// Woodcock tracking with one global majorant amax/dt.  Tentative points are generated from
// the ray's entry into the GLOBAL grid domain, identically on every rank; a rank evaluates
// only the points its own bricks own (half-open), so the first real collision over all
// ranks equals the union's.
// ---------------------------------------------------------------------------------------
// R-LOG: binary32 natural log of x in (0, 1], the same operation sequence as the oracle.
__device__ __forceinline__ float pln(float x) {
    const float Lg1 = 0x1.555554p-1f, Lg2 = 0x1.999c26p-2f, Lg3 = 0x1.23d3dcp-2f, Lg4 = 0x1.f13c4cp-3f;
    const float ln2_hi = 0x1.62e3p-1f, ln2_lo = 0x1.2fefa2p-17f;
    const uint32_t bits = __float_as_uint(x);
    int e = (int)((bits >> 23) & 0xffu) - 127;
    const uint32_t mb = (bits & 0x007fffffu) | 0x3f800000u;
    float m = __uint_as_float(mb);
    if (mb > 0x3fb504f3u) { m = m * 0.5f; e = e + 1; }
    const float f = m - 1.0f;
    const float s = f / (2.0f + f);
    const float z = s * s, w = z * z;
    const float R = z * (Lg1 + w * Lg3) + w * (Lg2 + w * Lg4);
    const float hfsq = (0.5f * f) * f;
    const float fe = (float)e;
    return fe * ln2_hi - ((hfsq - (s * (hfsq + R) + fe * ln2_lo)) - f);
}

template <bool ANY>
__device__ __noinline__ bool delta_track(const WorldDev &W, f3 o, f3 d, float limit, float dt, uint64_t seed,
                                         uint32_t p, uint32_t s, uint32_t depth, uint32_t purpose, uint32_t subhi,
                                         float &t_out, uint32_t &k_out, f3 &rgb_out, uint32_t &nsamples) {
    if (W.nbricks == 0 || !(W.amax > 0.0f)) return false;
    float t, t1;
    if (!slab(W.gdom, W.gdom + 3, o, d, __int_as_float(0x7f800000), t, t1)) return false;
    const float tend = fminf(t1, limit);
    uint4 rr = make_uint4(0, 0, 0, 0);
    for (uint32_t k = 0; k < (1u << 25); ++k) {
        if (!(k & 1)) rr = rng4(seed, p, s, depth, purpose, subhi | (k >> 1));
        const float xi = u01((k & 1) ? rr.z : rr.x), zeta = u01((k & 1) ? rr.w : rr.y);
        const float L = 0.0f - pln(1.0f - xi);
        t = t + (L * dt) / W.amax;
        if (!(t < tend)) return false;
        const f3 pt = mk(o.x + t * d.x, o.y + t * d.y, o.z + t * d.z);
        for (int b = 0; b < W.nbricks; ++b) {
            const BrickDev &B = W.bricks[b];
            const f3 g = grid_coord(B, pt);
            if (!(g.x >= (float)B.lo[0] && g.x < (float)B.hi[0] && g.y >= (float)B.lo[1] && g.y < (float)B.hi[1] &&
                  g.z >= (float)B.lo[2] && g.z < (float)B.hi[2]))
                continue;
            const float fx0 = floorf(g.x), fy0 = floorf(g.y), fz0 = floorf(g.z);
            const int ix = (int)fx0 - B.lo[0], iy = (int)fy0 - B.lo[1], iz = (int)fz0 - B.lo[2];
            // empty macrocell: alpha == 0 for every point in it, no collision (exact)
            if (!__ldg(B.mc + ((iz / MC_SIZE) * B.mc_dims[1] + iy / MC_SIZE) * B.mc_dims[0] + ix / MC_SIZE)) break;
            nsamples++;
            const int nx = B.hi[0] - B.lo[0] + 1, ny = B.hi[1] - B.lo[1] + 1;
            const float fx = g.x - fx0, fy = g.y - fy0, fz = g.z - fz0;
            const float *v = B.vox + (int64_t)ix + (int64_t)nx * (iy + ny * iz);  // ny * nz < 2^31 (dpr.h brick limits)
            const int64_t sy = nx, sz = (int64_t)nx * ny;
            float v000 = __ldg(v), v100 = __ldg(v + 1), v010 = __ldg(v + sy), v110 = __ldg(v + sy + 1);
            float v001 = __ldg(v + sz), v101 = __ldg(v + sz + 1), v011 = __ldg(v + sz + sy),
                  v111 = __ldg(v + sz + sy + 1);
            float c00 = lerpf(v000, v100, fx), c10 = lerpf(v010, v110, fx);
            float c01 = lerpf(v001, v101, fx), c11 = lerpf(v011, v111, fx);
            float c0 = lerpf(c00, c10, fy), c1 = lerpf(c01, c11, fy);
            f3 rgb;
            const float alpha = tf_alpha_rgb(B, lerpf(c0, c1, fz), ANY ? nullptr : &rgb);
            if (zeta * W.amax < alpha) {
                t_out = t;
                k_out = k;
                if (!ANY) rgb_out = rgb;
                return true;
            }
            break;  // one owner per point
        }
    }
    return false;
}

// ---------------------------------------------------------------------------------------
// a2: primary generation + visibility discard.
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_gen_primary(const __grid_constant__ StepArgs A, int s0,
                                                     int nsamp, int spw, int tw, int th) {
    // ray order: a warp holds spw samples of each of (32/spw) pixels of a tw x th tile, so the
    // rays of a warp are nearly identical for spw > 1 (coherent traversal); warps walk tiles,
    // then sample groups.
    const FrameDev &F = A.F;
    // 32-bit index math (the launcher guarantees < 2^32 threads; 64-bit divisions cost ~10x)
    const uint32_t tiles_x = ((uint32_t)F.W + tw - 1) / tw, tiles_y = ((uint32_t)F.H + th - 1) / th;
    const uint32_t per_group = tiles_x * tiles_y * 32u;
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    __shared__ uint32_t s_cnt[DPR_MAX_RANKS], s_base[DPR_MAX_RANKS];
    if (threadIdx.x < DPR_MAX_RANKS) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const bool valid = (uint64_t)t < (uint64_t)per_group * (uint32_t)(nsamp / spw);  // per_group: multiple of 32
    const uint32_t g = t / per_group;
    const uint32_t within = t - g * per_group;
    const uint32_t tile = within >> 5;
    const uint32_t li = within & 31u;
    const uint32_t ty = tile / tiles_x, tx = tile - ty * tiles_x;
    const uint32_t pi = li / (uint32_t)spw;
    uint32_t s = (uint32_t)s0 + g * (uint32_t)spw + (li - pi * (uint32_t)spw);
    const uint32_t py = pi / (uint32_t)tw;
    int x = (int)(tx * (uint32_t)tw + (pi - py * (uint32_t)tw));
    int y = (int)(ty * (uint32_t)th + py);
    bool inimg = valid && x < F.W && y < F.H;
    const int self = A.R.self;
    uint32_t p = (uint32_t)(y * F.W + x);
    if (F.pix_nranks > 1 && inimg)  // replicated mode: pixel ownership split
        inimg = (int)(((int64_t)p * F.pix_nranks) / F.P) == F.pix_rank;
    // rays outside the projection of this rank's box cannot have it as first candidate: only
    // their pixel owner generates them (to resolve misses)
    if (inimg && !(x >= F.gen_rect[0] && x < F.gen_rect[2] && y >= F.gen_rect[1] && y < F.gen_rect[3]))
        inimg = (int)(((int64_t)p * A.R.nranks) / F.P) == self;
    f3 o = mk(F.cE[0], F.cE[1], F.cE[2]), d = mk(0, 0, 0);
    int first = -2;
    if (inimg) {
        float jx = 0.5f, jy = 0.5f;
        if (!(F.flags & DPR_FLAG_JITTER_CENTER)) {
            uint4 r = rng4(F.seed, p, s, 0, PUR_CAMERA, 0);
            jx = u01(r.x);
            jy = u01(r.y);
        }
        float sx = ((float)x + jx) / (float)F.W;
        float sy = ((float)y + jy) / (float)F.H;
        f3 q = mk((F.cL[0] + sx * F.cU[0]) + sy * F.cV[0], (F.cL[1] + sx * F.cU[1]) + sy * F.cV[1],
                  (F.cL[2] + sx * F.cU[2]) + sy * F.cV[2]);
        if (F.lens_radius > 0.0f) {
            // thin lens (reading R-DOF): rejection-sampled disc point, focal point E + fd*q
            float lx = 0.0f, ly = 0.0f;
            for (uint32_t att = 0; att < 16; ++att) {
                uint4 r = rng4(F.seed, p, s, 0, PUR_LENS, att);
                float ax = 2.0f * u01(r.x) - 1.0f, ay = 2.0f * u01(r.y) - 1.0f;
                if (ax * ax + ay * ay <= 1.0f) { lx = ax; ly = ay; break; }
            }
            f3 U = mk(F.cU[0], F.cU[1], F.cU[2]), V = mk(F.cV[0], F.cV[1], F.cV[2]);
            float lu = sqrtf(dot(U, U)), lv = sqrtf(dot(V, V));
            f3 Uh = mk(U.x / lu, U.y / lu, U.z / lu), Vh = mk(V.x / lv, V.y / lv, V.z / lv);
            float a = F.lens_radius * lx, b = F.lens_radius * ly;
            o = mk((F.cE[0] + a * Uh.x) + b * Vh.x, (F.cE[1] + a * Uh.y) + b * Vh.y, (F.cE[2] + a * Uh.z) + b * Vh.z);
            f3 g = mk((F.cE[0] + F.focus_dist * q.x) - o.x, (F.cE[1] + F.focus_dist * q.y) - o.y,
                      (F.cE[2] + F.focus_dist * q.z) - o.z);
            float lg = sqrtf(dot(g, g));
            d = mk(g.x / lg, g.y / lg, g.z / lg);
        } else {
            float len = sqrtf(dot(q, q));
            d = mk(q.x / len, q.y / len, q.z / len);
        }
        if (!(F.flags & DPR_FLAG_RING)) first = first_candidate(A.R, o, d, __int_as_float(0x7f800000));
    }
    bool keep = first == self;
    bool owner_keep = false;
    if (F.flags & DPR_FLAG_RING) {
        // ring schedule (reading R-RING): the home rank generates its pixels, no culling
        keep = inimg && (int)(((int64_t)p * A.R.nranks) / F.P) == self;
    } else if (inimg && first == -1) {
        int owner = (int)(((int64_t)p * A.R.nranks) / F.P);
        owner_keep = owner == self;
    }
    fb_add_seg(A.fb, p, make_float4(F.B[0], F.B[1], F.B[2], 0.0f),
               owner_keep && !(F.flags & DPR_FLAG_NO_BACKGROUND));
    if (owner_keep && A.events) A.events[((int64_t)s * F.max_depth) * F.P + p] = 1u;
    uint32_t gen = __popc(__ballot_sync(FULL, keep || owner_keep));
    if ((threadIdx.x & 31) == 0 && gen) atomicAdd(&A.ctr->gen[K_PATH], (unsigned long long)gen);
    uint32_t pos = block_append(keep, self, A.Q.cnt_path, A.Q.path_cap, &A.ctr->overflow, nullptr, A.ctr->app[0], self,
                                A.R.nranks, s_cnt, s_base, A.Q.fused);
    if (keep && pos != 0xffffffffu) {
        PathRec *r = A.Q.path_out[self] + pos;
        r->a = make_float4(o.x, o.y, o.z, __int_as_float(0x7f800000));
        r->b = make_float4(d.x, d.y, d.z, __uint_as_float(NO_HIT));
        r->c = make_float4(1.0f, 1.0f, 1.0f, __uint_as_float(p));
        r->e = make_float4(0.0f, 0.0f, 0.0f, __uint_as_float(s));
    }
}

// ---------------------------------------------------------------------------------------
// a3: path-ray trace kernel (closest hit + brick march); results in place:
// a.w = bestT, b.w = bestId, e.xyz = normal (surface) or TF rgb (volume).
// ---------------------------------------------------------------------------------------
template <bool ANY>
__device__ __forceinline__ void trace_loop(const StepArgs &A) {
    const FrameDev &F = A.F;
    const int lane = threadIdx.x & 31;
    const uint32_t n_in = A.Q.in_count[ANY ? 1 : 0];
    stamp_kernel(A, ANY ? 1 : 0, true);
    uint32_t *fetch = A.Q.fetch + (ANY ? 1 : 0);
    const float INF = __int_as_float(0x7f800000);
    const bool fuse = ANY && fuse_resolve_dev(A, n_in);
    uint2 stack[WSTACK];
    __shared__ CoopSmem coop[TRACE_BLOCK / 32];
    __shared__ uint32_t s_vis[2];  // fused resolve: shadow / AO rays resolved by this block
    if (fuse) {
        if (threadIdx.x < 2) s_vis[threadIdx.x] = 0;
        __syncthreads();
    }
#if DPR_PERM_LUT
    perm_init();
#endif
    CoopSmem &cs = coop[threadIdx.x >> 5];
    TravState S;
    S.ng = make_uint2(0, 0);
    trav_clear(S);
    uint32_t idx = 0;
    bool alive = false, exhausted = false;
    TraceCounters tc = {0, 0, 0, 0};
    uint32_t rin = 0;
    for (;;) {
        unsigned dead = __ballot_sync(FULL, !alive);
        int ndead = __popc(dead);
        if (!exhausted && ndead >= (ANY ? REFILL_OCCL : REFILL_PATH)) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(fetch, (uint32_t)ndead);
            base = __shfl_sync(FULL, base, 0);
            if (base + (uint32_t)ndead >= n_in) exhausted = true;
            if (!alive) {
                idx = base + __popc(dead & lanemask_lt());
                if (idx < n_in) {
                    alive = true;
                    rin++;
                    if (ANY) {
                        const OcclRec *r = A.Q.occl_in + idx;
                        float4 a = __ldcg(&r->a), b = __ldcg(&r->b);
                        Hit h = {a.w, NO_HIT, -1};
                        // any-hit order (DPR_ANY_REVERSE): 1 back to front for all, 2 for bounded (AO) rays
                        const bool rev = DPR_ANY_REVERSE == 1 || (DPR_ANY_REVERSE == 2 && a.w < INF);
                        trav_init(S, xyz(a), xyz(b), a.w, h, A.W.nprims, rev ? 7u : 0u);
                    } else {
                        const PathRec *r = A.Q.path_in + idx;
                        float4 a = __ldcg(&r->a), b = __ldcg(&r->b);
                        Hit h = {a.w, __float_as_uint(b.w), -1};
                        trav_init(S, xyz(a), xyz(b), INF, h, A.W.nprims);
                    }
                }
            }
        }
        if (!__any_sync(FULL, alive)) {
            if (exhausted) break;
            continue;
        }
        if (!alive) trav_clear(S);
        bool fin = trav_step<ANY>(A.W, S, stack, tc, &A.ctr->overflow, cs);
        if (!(alive && fin)) continue;
        // finished: volume march, then write the result back into the record
        alive = false;
        if (ANY) {
            OcclRec *r = A.Q.occl_in + idx;
            bool occluded = S.h.prim >= 0;
            if (!occluded && A.W.nbricks > 0 && (F.flags & DPR_FLAG_DELTA)) {
                const uint32_t p = __float_as_uint(r->b.w), meta = __float_as_uint(r->c.w);
                const uint32_t s = meta & 0xffffu, depth = (meta >> 16) & 0xffu, slot = meta >> 24;
                float ti; uint32_t ii; f3 rgb;
                occluded = delta_track<true>(A.W, RAY_O(S), RAY_D(S), S.tmax, F.dt, F.seed, p, s, depth,
                                             slot == 0 ? PUR_VOL_SHADOW : PUR_VOL_AO,
                                             slot == 0 ? 0u : ((slot - 1) << 24), ti, ii, rgb, tc.vols);
            } else if (!occluded && A.W.nbricks > 0 && n_in >= F.march_inline_min) {
                const uint32_t p = __float_as_uint(r->b.w), meta = __float_as_uint(r->c.w);
                const uint32_t s = meta & 0xffffu, depth = (meta >> 16) & 0xffu, slot = meta >> 24;
                for (int b = 0; b < A.W.nbricks && !occluded; ++b) {
                    float ti; uint32_t ii; f3 rgb;
                    occluded = march_brick<true>(A.W.bricks[b], RAY_O(S), RAY_D(S), S.tmax, S.tmax, F.dt, F.seed, p, s,
                                                 depth, slot == 0 ? PUR_VOL_SHADOW : PUR_VOL_AO,
                                                 slot == 0 ? 0u : ((slot - 1) << 24), ti, ii, rgb, tc.vols);
                }
            }
            if (occluded && !fuse) r->a.w = -1.0f;  // occluded marker for k_resolve_occl
            if (fuse) {
                // one rank, no ring: no next candidate exists, so the ray resolves here (what
                // k_resolve_occl does): visit count, unoccluded -> framebuffer (+ P13 bit)
                const float4 c = __ldcg(&r->c);
                const uint32_t p = __float_as_uint(__ldcg(&r->b.w)), meta = __float_as_uint(c.w);
                const uint32_t slot = meta >> 24;
                atomicAdd(&s_vis[slot == 0 ? 0 : 1], 1u);
                if (!occluded) {
                    fb_add(A.fb + p, make_float4(c.x, c.y, c.z, 0.0f));
                    if (A.occl)
                        atomicOr(A.occl + ((int64_t)(meta & 0xffffu) * F.max_depth + ((meta >> 16) & 0xffu)) * F.P + p,
                                 1u << slot);
                }
            }
        } else {
            PathRec *r = A.Q.path_in + idx;
            bool changed = S.h.prim >= 0;
            f3 nrm = mk(0, 0, 0);
            if (changed) {
                const bool by_id = S.h.prim == PRIM_BY_ID;
                nrm = prim_normal(by_id ? A.W.prims_in : A.W.prims, by_id ? (int64_t)(S.h.id - A.W.id_base) : S.h.prim,
                                  RAY_O(S), RAY_D(S), S.h.t);
            }
            if (A.W.nbricks > 0 && (F.flags & DPR_FLAG_DELTA)) {
                const uint32_t p = __float_as_uint(r->c.w), meta = __float_as_uint(r->e.w);
                const uint32_t s = meta & 0xffffu, depth = (meta >> 16) & 0xffu;
                float ti; uint32_t kk; f3 rgb;
                if (delta_track<false>(A.W, RAY_O(S), RAY_D(S), S.h.t, F.dt, F.seed, p, s, depth, PUR_VOL_PATH, 0u, ti, kk,
                                       rgb, tc.vols)) {
                    S.h.t = ti; S.h.id = VOL_BIT | kk; nrm = rgb; changed = true;
                }
            } else if (A.W.nbricks > 0 && n_in >= F.march_inline_min) {
                const uint32_t p = __float_as_uint(r->c.w), meta = __float_as_uint(r->e.w);
                const uint32_t s = meta & 0xffffu, depth = (meta >> 16) & 0xffu;
                for (int b = 0; b < A.W.nbricks; ++b) {
                    float ti; uint32_t ii; f3 rgb;
                    if (march_brick<false>(A.W.bricks[b], RAY_O(S), RAY_D(S), INF, S.h.t, F.dt, F.seed, p, s, depth,
                                           PUR_VOL_PATH, 0u, ti, ii, rgb, tc.vols)) {
                        S.h.t = ti; S.h.id = VOL_BIT | ii; nrm = rgb; changed = true;
                    }
                }
            }
            if (changed) {
                r->a.w = S.h.t;
                r->b.w = __uint_as_float(S.h.id);
                r->e.x = nrm.x; r->e.y = nrm.y; r->e.z = nrm.z;
            }
        }
    }
    if (fuse) {
        __syncthreads();
        if (threadIdx.x < 2 && s_vis[threadIdx.x])
            atomicAdd(&A.ctr->V[threadIdx.x == 0 ? K_SHADOW : K_AO], (unsigned long long)s_vis[threadIdx.x]);
    }
    KernelCounters *kc = &A.ctr->kc[ANY ? 1 : 0];
    flush(&kc->nodes, tc.nodes);
    flush(&kc->tris, tc.tris);
    flush(&kc->sphs, tc.sphs);
    flush(&kc->vols, tc.vols);
    flush(&kc->rin, rin);
    stamp_kernel(A, ANY ? 1 : 0, false);  // each warp at its exit: the last one is the kernel's end
}

__global__ void __launch_bounds__(TRACE_BLOCK, TRACE_MINB) k_trace_path(const __grid_constant__ StepArgs A) {
    trace_loop<false>(A);
}
__global__ void __launch_bounds__(TRACE_BLOCK, TRACE_MINB) k_trace_occl(const __grid_constant__ StepArgs A) {
    trace_loop<true>(A);
}

// ---------------------------------------------------------------------------------------
// a4 + a6: path rays after the trace -- forward to the next candidate rank (P8) or resolve
// here: events, background/coverage, shading (P6) and spawning of shadow / AO / bounce rays
// into per-destination queues (warp-aggregated appends; every lane of a warp participates).
// ---------------------------------------------------------------------------------------
#ifndef DPR_SHADE_MINB
#define DPR_SHADE_MINB 8
#endif
#ifndef DPR_SHADE_BLOCK
#define DPR_SHADE_BLOCK 128
#endif
__global__ void __launch_bounds__(DPR_SHADE_BLOCK, DPR_SHADE_MINB) k_shade_path(const __grid_constant__ StepArgs A) {
    const FrameDev &F = A.F;
    const int self = A.R.self, N = A.R.nranks;
    const float INF = __int_as_float(0x7f800000);
    const uint32_t n_in = A.Q.in_count[0];
    uint32_t *const *cnt_path = A.Q.cnt_path;
    uint32_t *const *cnt_occl = A.Q.cnt_occl;
    uint32_t visits = 0, gen_p = 0, gen_s = 0, gen_a = 0, rout_p = 0, rout_o = 0;
    const f3 L = mk(F.l[0], F.l[1], F.l[2]);
    const int K = F.ao_k;
    __shared__ uint32_t s_cnt[DPR_MAX_RANKS], s_base[DPR_MAX_RANKS];
    if (threadIdx.x < DPR_MAX_RANKS) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    for (uint32_t tile = blockIdx.x; tile * blockDim.x < n_in; tile += gridDim.x) {
        uint32_t idx = tile * blockDim.x + threadIdx.x;
        bool active = idx < n_in;
        PathRec r;
        if (active) {
            const PathRec *src = A.Q.path_in + idx;
            r.a = __ldcs(&src->a); r.b = __ldcs(&src->b); r.c = __ldcs(&src->c); r.e = __ldcs(&src->e);
            visits++;
        } else {
            r.a = r.b = r.c = r.e = make_float4(0, 0, 0, 0);
        }
        const f3 o = xyz(r.a), d = xyz(r.b);
        const float bt = r.a.w;
        const uint32_t bid = __float_as_uint(r.b.w);
        const f3 nrm = xyz(r.e);
        const uint32_t p = __float_as_uint(r.c.w);
        const uint32_t meta = __float_as_uint(r.e.w);
        const uint32_t s = meta & 0xffffu, depth = (meta >> 16) & 0xffu;
        const bool ring = F.flags & DPR_FLAG_RING;
        const int home = (int)(((int64_t)p * N) / F.P);
        int next = -1;
        if (ring) next = (active && (self + 1) % N != home) ? (self + 1) % N : -1;  // R-RING
        else if (active) next = next_candidate(A.R, self, o, d, INF, bt);
        bool fwd = active && next >= 0;
        uint32_t pos = 0xffffffffu;
        pos = block_append(fwd, next, cnt_path, A.Q.path_cap, &A.ctr->overflow, A.ctr->S[K_PATH], A.ctr->app[0],
                               self, N, s_cnt, s_base, A.Q.fused);
        if (fwd && pos != 0xffffffffu) {
            PathRec *dst = A.Q.path_out[next] + pos;
            dst->a = r.a; dst->b = r.b; dst->c = r.c; dst->e = r.e;
            rout_p++;
        }
        bool res = active && next < 0;
        bool evt = res && bid != NO_HIT;
        bool vol = evt && (bid & VOL_BIT);
        if (res && A.events) {
            uint32_t code = bid == NO_HIT ? 1u : (vol ? bid : 2u + bid);
            A.events[((int64_t)s * F.max_depth + depth) * F.P + p] = code;
        }
        if (res && depth == 0) {
            if (evt) {
                fb_add(A.fb + p, make_float4(0.0f, 0.0f, 0.0f, 1.0f));
                if (A.depth) atomicMin(A.depth + p, __float_as_uint(bt));  // t > 0: bits order like floats
            } else if (!(F.flags & DPR_FLAG_NO_BACKGROUND)) {
                fb_add(A.fb + p, make_float4(F.B[0], F.B[1], F.B[2], 0.0f));
            }
        }
        if (!__syncthreads_or(evt)) continue;
        f3 hp = mk(o.x + bt * d.x, o.y + bt * d.y, o.z + bt * d.z);  // P5
        f3 org = hp, br = mk(0, 0, 0);
        float c = 0.0f;
        if (evt) {
            f3 beta = xyz(r.c);
            if (!vol) {
                f3 rho = part_albedo(A.T, bid);
                org = mk(hp.x + 1e-4f * nrm.x, hp.y + 1e-4f * nrm.y, hp.z + 1e-4f * nrm.z);
                br = mul(beta, rho);
                c = dot(nrm, L);
            } else {
                br = mul(beta, nrm);  // TF rgb travels in the normal slot
            }
        }
        // children: slot 0 shadow, 1..K AO, K+1 bounce (warp-uniform loop)
        for (int slot = 0; slot < K + 2; ++slot) {
            bool has = false;
            f3 cd = mk(0, 0, 0), w = mk(0, 0, 0);
            float ctmax = INF;
            if (evt) {
                if (slot == 0) {
                    if (!vol) {
                        has = c > 0.0f;
                        w = scale(mul(br, mk(F.E[0], F.E[1], F.E[2])), c);
                    } else {
                        has = true;
                        w = mul(br, mk(F.E[0], F.E[1], F.E[2]));
                    }
                    cd = L;
                } else if (slot <= K) {
                    if (!vol) {
                        has = true;
                        cd = cosine_dir(nrm, F.seed, p, s, depth, PUR_AO, (uint32_t)(slot - 1) << 4);
                        ctmax = F.ao_radius;
                        w = scale(mul(br, mk(F.A[0], F.A[1], F.A[2])), 1.0f / (float)K);
                    }
                } else {
                    has = (int)depth + 1 < F.max_depth;
                    if (has) {
                        cd = vol ? iso_dir(F.seed, p, s, depth)
                                 : cosine_dir(nrm, F.seed, p, s, depth, PUR_BOUNCE, 0u);
                        w = br;
                    }
                }
            }
            int first = has ? (ring ? home : first_candidate(A.R, org, cd, ctmax)) : -1;
            bool app = has && first >= 0;
            bool imm = has && first < 0;  // no candidate: resolves immediately here
            const bool is_path = slot == K + 1;
            if (has) {
                if (is_path) gen_p++;
                else if (slot == 0) gen_s++;
                else gen_a++;
            }
            if (imm) {
                if (is_path) {
                    if (A.events) A.events[((int64_t)s * F.max_depth + depth + 1) * F.P + p] = 1u;
                } else {
                    fb_add(A.fb + p, make_float4(w.x, w.y, w.z, 0.0f));
                    if (A.occl) atomicOr(A.occl + ((int64_t)s * F.max_depth + depth) * F.P + p, 1u << slot);
                }
            }
            if (is_path) {
                uint32_t q = block_append(app, first, cnt_path, A.Q.path_cap, &A.ctr->overflow,
                                          A.ctr->S[K_PATH], A.ctr->app[0], self, N, s_cnt, s_base, A.Q.fused);
                if (app && q != 0xffffffffu) {
                    PathRec *dst = A.Q.path_out[first] + q;
                    dst->a = make_float4(org.x, org.y, org.z, INF);
                    dst->b = make_float4(cd.x, cd.y, cd.z, __uint_as_float(NO_HIT));
                    dst->c = make_float4(w.x, w.y, w.z, __uint_as_float(p));
                    dst->e = make_float4(0.0f, 0.0f, 0.0f, __uint_as_float(s | ((depth + 1) << 16)));
                    rout_p++;
                }
            } else {
                uint32_t q = block_append(app, first, cnt_occl, A.Q.occl_cap, &A.ctr->overflow,
                                          A.ctr->S[slot == 0 ? K_SHADOW : K_AO], A.ctr->app[1], self, N, s_cnt,
                                          s_base, A.Q.fused);
                if (app && q != 0xffffffffu) {
                    OcclRec *dst = A.Q.occl_out[first] + q;
                    dst->a = make_float4(org.x, org.y, org.z, ctmax);
                    dst->b = make_float4(cd.x, cd.y, cd.z, __uint_as_float(p));
                    dst->c = make_float4(w.x, w.y, w.z,
                                         __uint_as_float(s | (depth << 16) | ((uint32_t)slot << 24)));
                    rout_o++;
                }
            }
        }
    }
    if (A.Q.fused) __threadfence_system();  // records written into peer queues are visible
    flush(&A.ctr->V[K_PATH], visits);
    flush(&A.ctr->gen[K_PATH], gen_p);
    flush(&A.ctr->gen[K_SHADOW], gen_s);
    flush(&A.ctr->gen[K_AO], gen_a);
    flush(&A.ctr->kc[0].rout_path, rout_p);
    flush(&A.ctr->kc[0].rout_occl, rout_o);
}

// ---------------------------------------------------------------------------------------
// a4: occlusion rays after the trace -- drop occluded, forward or resolve unoccluded.
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_resolve_occl(const __grid_constant__ StepArgs A) {
    const FrameDev &F = A.F;
    const int self = A.R.self, N = A.R.nranks;
    const uint32_t n_in = A.Q.in_count[1];
    if (fuse_resolve_dev(A, n_in)) return;  // k_trace_occl resolved these rays itself
    uint32_t *const *cnt_occl = A.Q.cnt_occl;
    uint32_t v_s = 0, v_a = 0, rout = 0;
    __shared__ uint32_t s_cnt[DPR_MAX_RANKS], s_base[DPR_MAX_RANKS];
    if (threadIdx.x < DPR_MAX_RANKS) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    for (uint32_t tile = blockIdx.x; tile * blockDim.x < n_in; tile += gridDim.x) {
        uint32_t idx = tile * blockDim.x + threadIdx.x;
        bool active = idx < n_in;
        OcclRec r;
        if (active) {
            const OcclRec *src = A.Q.occl_in + idx;
            r.a = __ldcs(&src->a); r.b = __ldcs(&src->b); r.c = __ldcs(&src->c);
        } else {
            r.a = r.b = r.c = make_float4(0, 0, 0, 0);
        }
        const f3 o = xyz(r.a), d = xyz(r.b);
        const float tmax = r.a.w;
        const uint32_t p = __float_as_uint(r.b.w);
        const uint32_t meta = __float_as_uint(r.c.w);
        const uint32_t s = meta & 0xffffu, depth = (meta >> 16) & 0xffu, slot = meta >> 24;
        const bool occluded = tmax < 0.0f;
        if (active) { if (slot == 0) v_s++; else v_a++; }
        int next = -1;
        if (F.flags & DPR_FLAG_RING) {
            // ring (reading R-RING): occluded or not, the ray completes the ring
            const int home = (int)(((int64_t)p * N) / F.P);
            next = (active && (self + 1) % N != home) ? (self + 1) % N : -1;
        } else if (active && !occluded) {
            next = next_candidate(A.R, self, o, d, tmax, tmax);
        }
        bool fwd = active && next >= 0;
        warp_count(fwd, (slot == 0 ? K_SHADOW : K_AO) * DPR_MAX_RANKS + next, &A.ctr->S[0][0]);
        uint32_t pos = 0xffffffffu;
        pos = block_append(fwd, next, cnt_occl, A.Q.occl_cap, &A.ctr->overflow, nullptr, A.ctr->app[1], self, N,
                               s_cnt, s_base, A.Q.fused);
        if (fwd && pos != 0xffffffffu) {
            OcclRec *dst = A.Q.occl_out[next] + pos;
            dst->a = r.a; dst->b = r.b; dst->c = r.c;
            rout++;
        }
        const bool acc = active && !occluded && next < 0;
        fb_add_seg(A.fb, p, make_float4(r.c.x, r.c.y, r.c.z, 0.0f), acc);
        if (acc && A.occl) atomicOr(A.occl + ((int64_t)s * F.max_depth + depth) * F.P + p, 1u << slot);
    }
    if (A.Q.fused) __threadfence_system();
    flush(&A.ctr->V[K_SHADOW], v_s);
    flush(&A.ctr->V[K_AO], v_a);
    flush(&A.ctr->kc[1].rout_occl, rout);
}

// ---------------------------------------------------------------------------------------
// a7 helpers (the collective itself is ncclReduce, or loopback accumulation).
// ---------------------------------------------------------------------------------------
__global__ void k_fb_accumulate(float4 *dst, const float4 *__restrict__ src, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float4 a = dst[i], b = src[i];
    dst[i] = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__global__ void k_u32_accumulate(uint32_t *dst, const uint32_t *__restrict__ src, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] += src[i];
}
__global__ void k_fb_normalize(float4 *out, const float4 *__restrict__ in, int64_t n, float spp) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float4 a = in[i];
    out[i] = make_float4(a.x / spp, a.y / spp, a.z / spp, a.w / spp);
}

// ---------------------------------------------------------------------------------------
// Compositing contrast device: per owned pixel, sort the N ranks' RGBA-z
// fragments by depth (ties: lower rank) and composite front to back, background last.
// ---------------------------------------------------------------------------------------
__global__ void k_depth_init(uint32_t *depth, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) depth[i] = 0x7f800000u;  // +inf
}

__global__ void k_composite(const float4 *__restrict__ frag_rgba, const float *__restrict__ frag_z, int nranks,
                            int64_t span, int64_t count, float br, float bg, float bb, float4 *out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    int ord[DPR_MAX_RANKS];
    float z[DPR_MAX_RANKS];
    for (int q = 0; q < nranks; ++q) {
        z[q] = frag_z[(int64_t)q * span + i];
        int k = q;  // insertion sort by (z, rank); ranks arrive in ascending order
        while (k > 0 && z[ord[k - 1]] > z[q]) { ord[k] = ord[k - 1]; --k; }
        ord[k] = q;
    }
    float cr = 0.0f, cg = 0.0f, cb = 0.0f, a = 0.0f;
    for (int k = 0; k < nranks; ++k) {
        float4 f = frag_rgba[(int64_t)ord[k] * span + i];
        float t = 1.0f - a;
        cr += t * f.x; cg += t * f.y; cb += t * f.z;
        a += t * f.w;
    }
    float t = 1.0f - a;
    out[i] = make_float4(cr + t * br, cg + t * bg, cb + t * bb, a);
}

// ---------------------------------------------------------------------------------------
// Step boundary (P8b lock-step: "wave-fronts are synchronized ... until all wave-fronts contain
// zero rays").  One block.  Phase 1 (end of a step): snapshot every local rank's
// cumulative routing row S[k][self][*] and visits V[k] into its StepRec (the per-step matrices),
// reset the consumed queue tails (fused exchange) and the persistent kernels' fetch heads, count
// the step.  Both phases: total of the next queues -- local ranks directly, the other ranks
// through the mailbox barrier: each rank stores {seq, path, occl, err} into slot [seq&1][self]
// of EVERY rank's mailbox (NVLink peer mappings; release order after a system fence, so the
// step's appends into peer queues and the tail resets are visible first) and spins until all
// N slots of its own mailbox carry seq (acquire).  Double-buffered by seq parity: a rank can be
// at most one boundary ahead of any other.  A barrier that does not complete within timeout_ns
// (a dead peer) sets err 0x100 and ends the loop.  Output: more[slot] = "another step", and the
// IF handle of the device-driven loop.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// The mailbox barrier of one rank (one thread): publish {seq, path, occl, err} into slot
// [seq&1][self] of every rank's mailbox, then wait until every slot [seq&1][*] of its own
// mailbox carries seq; returns the sums over ranks (err: OR, | 0x100 on timeout).
__device__ __forceinline__ void mailbox_barrier(uint32_t *mbox_self, uint32_t *const *mbox_peer, uint32_t *seq_ctr,
                                                int self, int nranks, uint32_t mine_p, uint32_t mine_o,
                                                uint32_t mine_err, unsigned long long timeout_ns,
                                                unsigned long long &tot, uint32_t &err) {
    const unsigned long long t0 = gtimer();
    const uint32_t seq = *seq_ctr + 1u;
    *seq_ctr = seq;
    const int b = seq & 1u;
    __threadfence_system();  // this rank's appends / tail resets before the mailbox stores
    for (int r = 0; r < nranks; ++r) {
        uint32_t *slot = mbox_peer[r] + ((size_t)b * DPR_MAX_RANKS + self) * 4;
        slot[1] = mine_p; slot[2] = mine_o; slot[3] = mine_err;
        st_release_sys(slot, seq);
    }
    tot = 0;
    err = mine_err;
    for (int r = 0; r < nranks; ++r) {
        const uint32_t *slot = mbox_self + ((size_t)b * DPR_MAX_RANKS + r) * 4;
        while (ld_acquire_sys(slot) != seq) {
            if (gtimer() - t0 > timeout_ns) { err |= 0x100u; break; }
        }
        if (err & 0x100u) break;
        tot += (unsigned long long)ld_acquire_sys(slot + 1) + ld_acquire_sys(slot + 2);
        err |= ld_acquire_sys(slot + 3);
    }
    __threadfence_system();
}

__global__ void __launch_bounds__(256) k_step_end(const __grid_constant__ StepEndArgs A) {
    __shared__ unsigned long long s_tot;
    __shared__ uint32_t s_err;
    const int tid = threadIdx.x;
    if (A.phase == 1) {
        // snapshots: nlocal x (3 x N S entries + 3 V entries)
        const int per = 3 * A.nranks + 5;
        for (int j = tid; j < A.nlocal * per; j += blockDim.x) {
            const int i = j / per, q = j - i * per;
            StepRec *R = A.rec[i];
            const uint32_t k = min(R->step, (uint32_t)MAX_STEP_REC - 1);
            if (q < 3 * A.nranks) R->S[k][q / A.nranks][q % A.nranks] = A.ctr[i]->S[q / A.nranks][q % A.nranks];
            else if (q < 3 * A.nranks + 3) R->V[k][q - 3 * A.nranks] = A.ctr[i]->V[q - 3 * A.nranks];
            else R->rin[k][q - 3 * A.nranks - 3] = A.ctr[i]->kc[q - 3 * A.nranks - 3].rin;
        }
    }
    if (tid == 0) {
        unsigned long long tot = 0;
        uint32_t err = 0;
        for (int i = 0; i < A.nlocal; ++i) {
            if (A.fused) tot += (unsigned long long)A.next_tails[i][0] + A.next_tails[i][1];
            err |= A.ctr[i]->overflow;
        }
        s_tot = tot;
        s_err = err;
    }
    if (tid < A.nlocal) {
        if (A.fused && A.phase == 1) { A.cons_tails[tid][0] = 0u; A.cons_tails[tid][1] = 0u; }
        for (int w = 0; w < 4; ++w) A.fetch[tid][w] = 0u;
    }
    __syncthreads();
    if (tid == 0) {
        unsigned long long t_sync = 0;
        if (A.barrier) {
            const unsigned long long t0 = gtimer();
            // what this rank appended in this step, all destinations (its own tail is not
            // final until every sender is done; the appends of this rank are): the global
            // total of the next step's queues is the sum over ranks
            unsigned long long app[2] = {0, 0};
            for (int k = 0; k < 2; ++k)
                for (int r = 0; r < A.nranks; ++r) app[k] += A.ctr[0]->app[k][r];
            StepRec *R0 = A.rec[0];
            const uint32_t mine_p = (uint32_t)(app[0] - R0->app_prev[0]), mine_o = (uint32_t)(app[1] - R0->app_prev[1]);
            R0->app_prev[0] = app[0];
            R0->app_prev[1] = app[1];
            unsigned long long tot = 0;
            uint32_t err = 0;
            mailbox_barrier(A.mbox_self, A.mbox_peer, A.seq, A.self, A.nranks, mine_p, mine_o, s_err, A.timeout_ns,
                            tot, err);
            s_tot = tot;
            s_err = err;
            t_sync = gtimer() - t0;
        }
        const unsigned long long now = gtimer();
        const uint32_t more = s_tot > 0 && s_err == 0;
        for (int i = 0; i < A.nlocal; ++i) {
            StepRec *R = A.rec[i];
            R->err |= s_err;
            if (A.phase == 1) {
                const uint32_t k = min(R->step, (uint32_t)MAX_STEP_REC - 1);
                R->t_end[k] = now;
                R->t_sync[k] += t_sync;
                R->step = R->step + 1;
            }
            R->t_begin[min(R->step, (uint32_t)MAX_STEP_REC)] = now;
        }
        if (A.more_slot >= 0) A.more[A.more_slot] = more;
        if (A.set_if) cudaGraphSetConditional(A.h_if, more);
    }
}

// Test of the mailbox barrier protocol on ONE GPU (B200_PROFILING.md: ranks that wait on one
// another must be one kernel): block r plays rank r with its own mailbox and sequence counter;
// every iteration each rank publishes counts f(it, r) after a pseudo-random delay and checks
// the sums.  mbox: [nranks][2][DPR_MAX_RANKS][4], seq: [nranks], bad: mismatches.
__global__ void k_barrier_emulate(uint32_t *mbox, uint32_t *seq, int nranks, int iters, uint32_t *bad) {
    const int r = blockIdx.x;
    if (threadIdx.x != 0) return;
    uint32_t *peers[DPR_MAX_RANKS];
    for (int q = 0; q < nranks; ++q) peers[q] = mbox + (size_t)q * 2 * DPR_MAX_RANKS * 4;
    for (int it = 0; it < iters; ++it) {
        uint32_t h = (uint32_t)(it * 2654435761u) ^ (uint32_t)(r * 2246822519u);
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        const unsigned long long until = gtimer() + (h & 1023u);  // skew the ranks
        while (gtimer() < until) {}
        unsigned long long tot = 0, want = 0;
        uint32_t err = 0;
        mailbox_barrier(peers[r], peers, seq + r, r, nranks, (uint32_t)(it + 3 * r), (uint32_t)(7 * it + r),
                        (uint32_t)((it % 5 == 4 && r == nranks - 1) ? 1 : 0), 2000000000ull, tot, err);
        for (int q = 0; q < nranks; ++q) want += (unsigned long long)(it + 3 * q) + (7ull * it + q);
        const uint32_t want_err = it % 5 == 4 ? 1u : 0u;
        if (tot != want || err != want_err) atomicAdd(bad, 1u);
    }
}

__global__ void k_set_ifs(const __grid_constant__ IfArgs A) {
    const int t = threadIdx.x;
    if (t < 2 * A.n) {
        const bool run = A.tails[t >> 1][t & 1] > 0u;
        cudaGraphSetConditional(A.h[t >> 1][t & 1], run);
        if (run) atomicAdd(A.count, A.kernels[t >> 1][t & 1]);
    }
}
void launch_set_ifs(const IfArgs &a, cudaStream_t s) { k_set_ifs<<<1, 32, 0, s>>>(a); }

__global__ void k_loop_cond(uint32_t *more, cudaGraphConditionalHandle h, int init) {
    cudaGraphSetConditional(h, init ? more[0] : (more[0] && more[1]));
    if (!init) more[2]++;  // WHILE iterations (launch accounting)
}

void launch_step_end(const StepEndArgs &a, cudaStream_t s) { k_step_end<<<1, 256, 0, s>>>(a); }
int test_step_barrier(int nranks, int iters, uint32_t *mbox, uint32_t *seq, uint32_t *bad, cudaStream_t s) {
    void *args[] = {&mbox, &seq, &nranks, &iters, &bad};
    return (int)cudaLaunchCooperativeKernel((const void *)k_barrier_emulate, dim3(nranks), dim3(32), args, 0, s);
}
void launch_loop_cond(uint32_t *more, cudaGraphConditionalHandle h, int init, cudaStream_t s) {
    k_loop_cond<<<1, 1, 0, s>>>(more, h, init);
}

static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }


void launch_depth_init(uint32_t *depth, int64_t n, cudaStream_t s) {
    if (n > 0) k_depth_init<<<nblk(n, 256), 256, 0, s>>>(depth, n);
}
void launch_composite(const float4 *frag_rgba, const float *frag_z, int nranks, int64_t span, int64_t count,
                      float br, float bg, float bb, float4 *out, cudaStream_t s) {
    if (count > 0) k_composite<<<nblk(count, 256), 256, 0, s>>>(frag_rgba, frag_z, nranks, span, count, br, bg, bb, out);
}

void launch_gen_primary(const StepArgs &a, int s0, int nsamp, int spw_max, cudaStream_t s) {
    int spw = 1;  // largest power of two <= spw_max dividing nsamp
    while (spw * 2 <= spw_max && spw * 2 <= 32 && nsamp % (spw * 2) == 0) spw *= 2;
    static const int TW[6] = {8, 4, 4, 2, 2, 1};  // tile width for spw = 1,2,4,8,16,32
    int lg = __builtin_ctz(spw);
    int tw = TW[lg], th = (32 / spw) / tw;
    int64_t per = (int64_t)((a.F.W + tw - 1) / tw) * ((a.F.H + th - 1) / th) * 32;
    int64_t total = per * (nsamp / spw);
    if (total > 0) k_gen_primary<<<nblk(total, 256), 256, 0, s>>>(a, s0, nsamp, spw, tw, th);
}
// The P10 march: with enough rays to give every lane of the GPU two, per lane inside the
// trace kernels (all lanes of a warp march together, right after the traversal); with fewer
// (long marches of few rays would serialise), in k_march_* with G lanes per ray.  Delta
// tracking always runs inside the trace kernels.  The choice is made on the device from the
// queue length (warp_march_dev / march_variant); the host launches the variant(s) that can
// apply.  Test override DPR_MARCH="<inline_min>[:G]" (e.g. "0": always inline;
// "1000000000:4": always k_march_* with 4 lanes per ray).
int march_g_env() {
    const char *e = getenv("DPR_MARCH");
    const char *c = e ? strchr(e, ':') : nullptr;
    return c ? atoi(c + 1) : DPR_MARCH_G;
}
uint32_t march_inline_min(int nsm) {
    if (const char *e = getenv("DPR_MARCH")) return (uint32_t)strtoul(e, nullptr, 10);
    return DPR_WARP_MARCH ? (uint32_t)nsm * 1024u * 2u : 0u;
}
static bool use_warp_march(const StepArgs &a, uint32_t n) {
    return a.W.nbricks > 0 && !(a.F.flags & DPR_FLAG_DELTA) && n < a.F.march_inline_min;
}
#ifndef DPR_FUSE_RESOLVE
#define DPR_FUSE_RESOLVE 1
#endif
bool fuse_resolve_ok(const StepArgs &a) {
    // read per call (a few times per frame) so a process can switch it (tests)
    return DPR_FUSE_RESOLVE && getenv("DPR_NO_FUSE_RESOLVE") == nullptr && a.R.nranks == 1 && !(a.F.flags & DPR_FLAG_RING);
}
template <int G>
static int march_grid(bool any) {
    static int grid[2] = {0, 0};
    if (!grid[any]) {
        int dev = 0, nsm = 0, occ = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (any) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_march_occl<G>, 256, 0);
        else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_march_path<G>, 256, 0);
        grid[any] = nsm * std::max(1, occ);
    }
    return grid[any];
}
// n: known queue length (no more groups than rays), or 0xffffffff (unknown: full grid)
template <int G>
static void launch_march(const StepArgs &a, bool any, uint32_t n, cudaStream_t s) {
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>(march_grid<G>(any), ((int64_t)n * G + 255) / 256));
    if (any) k_march_occl<G><<<g, 256, 0, s>>>(a);
    else k_march_path<G><<<g, 256, 0, s>>>(a);
}
static void launch_march_g(const StepArgs &a, bool any, int G, uint32_t n, cudaStream_t s) {
    if (G == 1) launch_march<1>(a, any, n, s);
    else if (G == 4) launch_march<4>(a, any, n, s);
    else if (G == 8) launch_march<8>(a, any, n, s);
    else launch_march<32>(a, any, n, s);
}
int launch_trace_path(const StepArgs &a, int grid, uint32_t n, cudaStream_t s) {
    k_trace_path<<<grid, TRACE_BLOCK, 0, s>>>(a);
    if (!use_warp_march(a, n)) return 1;
    launch_march_g(a, false, march_variant(a.F.march_g, n, a.F.march_inline_min), n, s);
    return 2;
}
int launch_trace_occl(const StepArgs &a, int grid, uint32_t n, cudaStream_t s) {
    k_trace_occl<<<grid, TRACE_BLOCK, 0, s>>>(a);
    if (!use_warp_march(a, n)) return 1;
    launch_march_g(a, true, march_variant(a.F.march_g, n, a.F.march_inline_min), n, s);
    return 2;
}
bool march_needed(const StepArgs &a, uint32_t n) { return use_warp_march(a, n); }
void k_launch_trace_path(const StepArgs &a, int grid, cudaStream_t s) { k_trace_path<<<grid, TRACE_BLOCK, 0, s>>>(a); }
void k_launch_trace_occl(const StepArgs &a, int grid, cudaStream_t s) { k_trace_occl<<<grid, TRACE_BLOCK, 0, s>>>(a); }
void march_grids_init() {
    for (int any = 0; any < 2; ++any) {
        march_grid<1>(any); march_grid<4>(any); march_grid<8>(any); march_grid<32>(any);
    }
}
int march_variants_count(const StepArgs &a) {
    if (a.W.nbricks == 0 || (a.F.flags & DPR_FLAG_DELTA) || a.F.march_inline_min == 0) return 0;
    return a.F.march_g ? 1 : 3;
}
int launch_march_variants(const StepArgs &a, bool any, cudaStream_t s) {
    if (a.W.nbricks == 0 || (a.F.flags & DPR_FLAG_DELTA) || a.F.march_inline_min == 0) return 0;
    if (a.F.march_g) {
        launch_march_g(a, any, march_variant(a.F.march_g, 0, 0), 0xffffffffu, s);
        return 1;
    }
    for (int G : {1, 4, 32}) launch_march_g(a, any, G, 0xffffffffu, s);
    return 3;
}
void launch_shade_path(const StepArgs &a, int grid, cudaStream_t s) {
    k_shade_path<<<grid * (256 / DPR_SHADE_BLOCK), DPR_SHADE_BLOCK, 0, s>>>(a);
}
void launch_resolve_occl(const StepArgs &a, int grid, cudaStream_t s) {
    k_resolve_occl<<<grid, 256, 0, s>>>(a);
}
int trace_path_occupancy(int block) {
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_trace_path, block, 0);
    return n;
}
int trace_occl_occupancy(int block) {
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_trace_occl, block, 0);
    return n;
}
void launch_fb_accumulate(float4 *dst, const float4 *src, int64_t n, cudaStream_t s) {
    if (n > 0) k_fb_accumulate<<<nblk(n, 256), 256, 0, s>>>(dst, src, n);
}
void launch_u32_accumulate(uint32_t *dst, const uint32_t *src, int64_t n, cudaStream_t s) {
    if (n > 0) k_u32_accumulate<<<nblk(n, 256), 256, 0, s>>>(dst, src, n);
}
void launch_fb_normalize(float4 *out, const float4 *in, int64_t n, float spp, cudaStream_t s) {
    if (n > 0) k_fb_normalize<<<nblk(n, 256), 256, 0, s>>>(out, in, n, spp);
}

}  // namespace dpr
