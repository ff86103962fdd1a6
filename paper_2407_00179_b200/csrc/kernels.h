// kernels.h -- launch wrappers shared between the kernels and the host orchestration.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace dpr {

// Morton key of a prim's centroid: 10 bits per axis, 30 bits (LSD radix sort, 4 digit passes)
typedef uint32_t mkey_t;
constexpr int MKEY_DIGITS = 4;

// ---- lbvh.cu ---------------------------------------------------------------------------
// one block of k_part_prims: prims [start, start+count) of one part (global ids g0...)
struct PrimChunk {
    const void *src;       // float verts[3*nv] (triangles) or float4 spheres[]
    const int32_t *idx;    // triangles: int32 idx[3*nt]
    int64_t nv;            // triangles: vertex count (index validation)
    int64_t start;         // first prim of the chunk within its part
    uint32_t g0;           // global (rank-local) id of that prim
    int count, kind, slot; // prims in the chunk, DPR_PART_*, bounds slot (part k -> k+1)
};
constexpr int PRIM_CHUNK = 4096;
void launch_part_prims(const PrimChunk *chunks, int nchunks, float4 *prims, float4 *blo, float4 *bhi, int *bounds,
                       int *bad_index, cudaStream_t s);
int64_t radix_tiles(int64_t n);
void launch_iota(uint32_t *v, int64_t n, cudaStream_t s);  // v[i] = i (the sort test's values)
void launch_radix_pass(const mkey_t *kin, const uint32_t *vin, mkey_t *kout, uint32_t *vout,
                       int64_t n, int shift, uint32_t *tile_hist, cudaStream_t s, int *launches,
                       bool hist_ready = false);  // hist_ready: tile_hist already holds this pass's tile counts
// Morton codes fused with the first pass's tile histogram and all digits' totals (hist_all,
// zeroed by the caller)
void launch_morton_h(const float4 *blo, const float4 *bhi, int64_t n, const int *bounds, mkey_t *keys, uint32_t *vals,
                     uint32_t *tile_hist0, unsigned long long *hist_all, cudaStream_t s);
void launch_karras(const mkey_t *keys, int64_t n, int *left, int *right, int *parent, int *rlo,
                   int *rhi, int *size, cudaStream_t s);
void launch_refit(int64_t n, const int *left, const int *right, const int *parent,
                  const float4 *slo, const float4 *shi, float4 *nlo, float4 *nhi, int *arrive,
                  cudaStream_t s);
// Binary node record (32 B, one sector): a = (lo.xyz, left id | min(size, 7) << 29),
// b = (hi.xyz, right id | off << 29), off = p - (first sorted leaf) for nodes of <= 7 leaves
// of the agglomerative tree, else 7; ids: internal k in [0, n-1), leaf j -> n-1+j.
struct BNode { float4 a, b; };
// split_scratch: >= n-1 bytes (the unused radix-sort key buffer); leaf: packed leaf boxes
// (leaf[2j] = lo, leaf[2j+1] = hi); returns kernels launched
int launch_agglo(const mkey_t *keys, uint8_t *split_scratch, int64_t n, const float4 *leaf, BNode *bn,
                 void *other, int *root_out, cudaStream_t s);
// BNode records from the separate arrays of the Karras + refit / PLOC builders
void launch_pack_bnodes(int64_t n, const int *left, const int *right, const int *size, const float4 *nlo,
                        const float4 *nhi, BNode *bn, cudaStream_t s);
// slo / shi: the packed leaf records (slo = leaf, shi = leaf + 1; written at stride 2)
void launch_gather_prims(const float4 *in, const uint32_t *perm, int64_t n, float4 *out,
                         const float4 *blo, const float4 *bhi, float4 *slo, float4 *shi,
                         cudaStream_t s);
struct CollapseArgs {
    int64_t n;
    const BNode *bn;     // binary internal nodes
    const float4 *leaf;  // packed leaf boxes (leaf[2j] = lo, leaf[2j+1] = hi)
    uint32_t *perm;  // per-wide-node contiguous prim order: perm[dst] = sorted prim index
    WNode *nodes;
    int *counters;  // [1] wide nodes allocated, [2] prims placed, [3] capacity overflow
    int node_cap;
};
// one BFS level of the collapse: *cnt_in items (device memory) -> next, appending to *cnt_out
void launch_collapse_level(const CollapseArgs &a, const int2 *items, const int *cnt_in, int2 *next, int *cnt_out,
                           int level, cudaStream_t s);
void launch_permute_prims(const float4 *in, const uint32_t *perm, const uint32_t *sortperm, int64_t n,
                          float4 *out, cudaStream_t s);
// ---- ploc.cu: PLOC binary builder (Meister & Bittner 2018) ------------------------------
struct PlocArgs {
    int64_t n;
    const float4 *slo, *shi;  // leaf boxes (Morton order), packed records: index 2j
    float4 *nlo, *nhi;        // internal node boxes
    int *left, *right, *size; // internal nodes [0, n-1)
};
int64_t ploc_block_count(int64_t m);
void launch_ploc_init(int64_t n, int *clusters, cudaStream_t s);
void launch_ploc_nn(const PlocArgs &a, const int *clusters, int64_t m, int *nn, cudaStream_t s);
void launch_ploc_count(const int *nn, int64_t m, int *block_counts, cudaStream_t s);
void launch_ploc_scan(int *block_counts, int64_t nblocks, int *totals, cudaStream_t s);
void launch_ploc_write(const PlocArgs &a, const int *clusters, const int *nn, int64_t m, const int *block_offsets,
                       int node_base, int *next_clusters, cudaStream_t s);

// mc: 3 x (mcx*mcy*mcz) bytes: flags, distance field, scratch; returns kernels launched
int launch_macrocells(const float *vox, int nx, int ny, int nz, int mcx, int mcy, int mcz,
                      const float4 *tf, float tf_lo, float tf_hi, float dscale, uint8_t *mc,
                      cudaStream_t s);

// ---- trace.cu --------------------------------------------------------------------------
struct FrameDev {
    int W, H, P, spp, max_depth, ao_k;
    float ao_radius;
    float l[3], E[3], A[3], B[3];
    float dt;
    uint64_t seed;
    uint32_t flags;
    float cE[3], cL[3], cU[3], cV[3];  // camera basis (P2)
    float lens_radius, focus_dist;     // thin lens (reading R-DOF); 0 = pinhole
    int pix_rank, pix_nranks;          // replicated mode: generate only pixels owned by pix_rank
    int gen_rect[4];                   // pixels [x0,x1) x [y0,y1) whose rays can meet this rank's
                                       // padded box (conservative screen projection); others are
                                       // generated only by their pixel owner
    int fuse_resolve;                  // k_trace_occl may resolve its rays itself (one rank, no ring);
                                       // it does unless the queue goes to k_march_occl (decided on
                                       // the device from the queue length: fuse_resolve_dev)
    uint32_t march_inline_min;         // P10 march inside the trace kernels when the queue holds
                                       // at least this many rays, else in k_march_* (G lanes/ray)
    int march_g;                       // forced lanes per ray of k_march_* (0: from the ray count)
};

struct QueuesDev {
    PathRec *path_in;
    OcclRec *occl_in;
    const uint32_t *in_count;   // [2]: path, occl
    PathRec *path_out[DPR_MAX_RANKS];
    OcclRec *occl_out[DPR_MAX_RANKS];
    uint32_t *cnt_path[DPR_MAX_RANKS];  // append counter of each destination's path queue
    uint32_t *cnt_occl[DPR_MAX_RANKS];  //   (send-recv mode: local counts; fused mode: the
                                        //    destination's next-queue tail, possibly a peer's)
    int fused;                          // 1: appends go straight into the destination's queue
    uint32_t path_cap, occl_cap;
    uint32_t *fetch;            // [2] persistent-kernel fetch heads
};

// Per-step record of one rank (device memory, zeroed per frame): the step counter, per-step
// cumulative routing rows / visits (the per-step matrices of P8b) and globaltimer stamps.
// Steps beyond MAX_STEP_REC accumulate into the last slot.
constexpr int MAX_STEP_REC = 256;
struct StepRec {
    uint32_t step;                                      // steps completed this frame (all batches)
    uint32_t err;                                       // overflow bits | 0x100 barrier timeout
    unsigned long long app_prev[2];                     // appended totals (path, occl) at the last boundary
    unsigned long long t_begin[MAX_STEP_REC + 1];       // globaltimer when step k could start
    unsigned long long t_end[MAX_STEP_REC];             // ... when its step boundary completed
    unsigned long long t_sync[MAX_STEP_REC];            // ns inside the step barrier (fused, N>1)
    unsigned long long kt[MAX_STEP_REC][2][2];          // trace kernel (path, occl): ~first start, last end
    unsigned long long S[MAX_STEP_REC][3][DPR_MAX_RANKS];  // cumulative S row of this rank after step k
    unsigned long long V[MAX_STEP_REC][3];                 // cumulative visits of this rank after step k
    unsigned long long rin[MAX_STEP_REC][2];               // cumulative rays traced (path, occl) after step k
};

struct StepArgs {
    FrameDev F;
    Routing R;
    WorldDev W;
    PartTable T;
    QueuesDev Q;
    float4 *fb;
    uint32_t *events;  // debug dumps or nullptr
    uint32_t *occl;
    uint32_t *depth;   // per-pixel min primary hit t (float bits; +inf init) or nullptr
    Counters *ctr;
    StepRec *rec;      // trace kernels stamp their start / end into rec->kt[rec->step]
};

// Step boundary (one block): per-step snapshot of the routing rows and visits, reset of the
// consumed queue tails and fetch heads, the global next-queue total (local ranks, plus the
// peers' through a mailbox barrier over NVLink peer memory when barrier = 1), and the
// conditional handles of the device-driven step loop.
struct StepEndArgs {
    int nlocal;                               // ranks handled here (loopback: all; else 1)
    int nranks, self;                         // world size; this rank (barrier mode)
    int phase;                                // 0: before a batch's first step, 1: end of a step
    int fused;                                // next counts are the fused tails (local ranks; with
                                              // the barrier, each rank publishes what IT appended)
    const uint32_t *next_tails[DPR_MAX_RANKS];  // fused: {path, occl} of the next parity
    uint32_t *cons_tails[DPR_MAX_RANKS];      // fused: consumed parity tails -> 0 (phase 1)
    uint32_t *fetch[DPR_MAX_RANKS];           // 4 fetch heads per local rank -> 0
    const Counters *ctr[DPR_MAX_RANKS];
    StepRec *rec[DPR_MAX_RANKS];
    int barrier;                              // 1: exchange counts with the peers (mailboxes)
    uint32_t *mbox_self;                      // [2][DPR_MAX_RANKS][4] {seq, path, occl, err}
    uint32_t *mbox_peer[DPR_MAX_RANKS];       // every rank's mailbox (peer mappings; self too)
    uint32_t *seq;                            // barrier sequence number (persistent)
    unsigned long long timeout_ns;
    uint32_t *more;                           // [2]: "another step" flags for the loop graph
    int more_slot;                            // which flag this boundary writes (-1: none)
    int set_if;                               // set h_if to "another step"
    cudaGraphConditionalHandle h_if;
};
void launch_step_end(const StepEndArgs &a, cudaStream_t s);
// the device loop's per-rank kernel-group conditions: h[i][0] = path queue of local rank i
// non-empty, h[i][1] = occlusion queue non-empty (tails[i] = {path, occl} input counts)
struct IfArgs {
    int n;
    const uint32_t *tails[DPR_MAX_RANKS];
    cudaGraphConditionalHandle h[DPR_MAX_RANKS][2];
    uint32_t kernels[DPR_MAX_RANKS][2];  // kernels in each group (launch accounting)
    uint32_t *count;                     // += kernels of the groups that run
};
int march_variants_count(const StepArgs &a);  // k_march_* launches launch_march_variants makes
void launch_set_ifs(const IfArgs &a, cudaStream_t s);
// the mailbox barrier of nranks ranks emulated as one cooperative launch (test); returns a
// cudaError_t; *bad counts iterations whose sums were wrong
int test_step_barrier(int nranks, int iters, uint32_t *mbox, uint32_t *seq, uint32_t *bad, cudaStream_t s);
// WHILE handle of the loop graph := more[0] && more[1] (end of the unrolled double step)
void launch_loop_cond(uint32_t *more, cudaGraphConditionalHandle h, int init, cudaStream_t s);

void launch_gen_primary(const StepArgs &a, int s0, int nsamp, int spw_max, cudaStream_t s);
// n: input rays (sizes the march launch); returns the number of kernels launched
uint32_t march_inline_min(int nsm);
int march_g_env();  // DPR_MARCH "<min>:G" override of the k_march_* lanes per ray (0: auto)
// the host-side part of the occlusion trace's own resolve (one rank, no ring, env); the
// kernel also requires that the queue is not marched by k_march_occl
bool fuse_resolve_ok(const StepArgs &a);
// launch every k_march_* variant that a queue of unknown length could need (device loop):
// each exits unless the device-side choice for the actual length is its own
int launch_march_variants(const StepArgs &a, bool any, cudaStream_t s);
bool march_needed(const StepArgs &a, uint32_t n);  // a queue of n rays goes to k_march_*
void march_grids_init();                            // occupancy-derived grids (before a capture)
// the trace kernels alone (device loop: the march variants are launched separately)
void k_launch_trace_path(const StepArgs &a, int grid, cudaStream_t s);
void k_launch_trace_occl(const StepArgs &a, int grid, cudaStream_t s);
int launch_trace_path(const StepArgs &a, int grid, uint32_t n, cudaStream_t s);
int launch_trace_occl(const StepArgs &a, int grid, uint32_t n, cudaStream_t s);
void launch_shade_path(const StepArgs &a, int grid, cudaStream_t s);
void launch_resolve_occl(const StepArgs &a, int grid, cudaStream_t s);
int trace_path_occupancy(int block);
int trace_occl_occupancy(int block);
#ifndef DPR_TRACE_BLOCK
#define DPR_TRACE_BLOCK 256  // r02 re-sweep (configs[1] frame): 64 19.96, 128 19.75, 256 19.66 ms
#endif
constexpr int TRACE_BLOCK = DPR_TRACE_BLOCK;
#ifndef DPR_TRACE_MINB
#define DPR_TRACE_MINB (1024 / DPR_TRACE_BLOCK)
#endif
constexpr int TRACE_MINB = DPR_TRACE_MINB;  // 1024 threads per SM -> <= 64 registers (sweep r01)

void launch_fb_accumulate(float4 *dst, const float4 *src, int64_t n, cudaStream_t s);
void launch_u32_accumulate(uint32_t *dst, const uint32_t *src, int64_t n, cudaStream_t s);
void launch_fb_normalize(float4 *out, const float4 *in, int64_t n, float spp, cudaStream_t s);
void launch_depth_init(uint32_t *depth, int64_t n, cudaStream_t s);
void launch_composite(const float4 *frag_rgba, const float *frag_z, int nranks, int64_t span, int64_t count,
                      float br, float bg, float bb, float4 *out, cudaStream_t s);

}  // namespace dpr
