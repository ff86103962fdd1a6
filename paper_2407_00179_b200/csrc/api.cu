// api.cu -- the C ABI of include/dpr.h and the host orchestration of the wavefront loop.
//
// One process per GPU; every rank owns a dpr_device.  A frame (S3.2) is:
//   1. consistency: allgather of a 64-bit digest of camera+frame
//   2. allgather of {rank box, prim count, part table} -> routing table (P8), global id
//      bases (P12), global part->albedo table (shading at the resolving rank, reading A3)
//   3. per spp batch: k_gen_primary, then lock-step steps {k_trace_path, k_trace_occl ->
//      allgather of the per-destination counts -> grouped ncclSend/ncclRecv of the ray
//      records} until every queue on every rank is empty (S2.2)
//   4. ncclReduce(sum) of the float4 framebuffers (and debug dumps) to rank 0
//   5. allgather of per-rank counters -> global routing matrices / visits / timings
// The loopback group runs the same loop over N virtual ranks on one GPU with device copies
// in place of NCCL (test fixture).
#include <cuda.h>  // CUdeviceptr / CUresult only (the driver entry point is looked up at run time)
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dpr.h"
#include "common.cuh"
#include "kernels.h"

using namespace dpr;

namespace {

// 1/h when h is a normal power of two whose reciprocal is normal (then x/h == x*(1/h) exactly
// in binary32), else 0 (the kernels then divide)
float exact_recip_pow2(float h) {
    uint32_t b;
    std::memcpy(&b, &h, 4);
    const uint32_t e = (b >> 23) & 0xffu, m = b & 0x7fffffu;
    if (m != 0 || e < 1 || e > 253) return 0.0f;
    return 1.0f / h;
}

thread_local std::string g_err;

// NVTX ranges (frame, phases, wavefront steps, kernel groups) for nsys timelines; no-ops
// unless a tool is attached
struct Nvtx {
    explicit Nvtx(const char *name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
};

struct Dev;

struct Buf {
    void *p = nullptr;
    size_t bytes = 0;
    bool raw = false;  // cudaMalloc'd (IPC-exportable), not from the allocator
};

struct PartStore {
    int kind = 0;
    float albedo[3] = {0, 0, 0};
    Buf verts, idx, spheres, vox, tf, mc;
    int64_t nv = 0, nt = 0, ns = 0;
    int gdims[3] = {0, 0, 0}, lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0}, mc_dims[3] = {0, 0, 0};
    float origin[3] = {0, 0, 0}, spacing[3] = {1, 1, 1};
    float tf_lo = 0, tf_hi = 1, dscale = 1;
    float amax = 0;  // bricks: max over TF entries of min(1, a * dscale)
    int has_hint = 0;
    float hint[6] = {0, 0, 0, 0, 0, 0};
    int64_t nprims() const { return kind == DPR_PART_TRIANGLES ? nt : (kind == DPR_PART_SPHERES ? ns : 0); }
};

struct LoopGroup {
    std::vector<Dev *> devs;
};

constexpr int MAXP = 1024;  // parts per rank in the frame allgather

struct PartInfo {
    uint32_t first, count;
    float albedo[3];
    float pad;
};

struct RankInfo {
    uint64_t digest;
    float box[6];
    int32_t nonempty;
    uint32_t nprims;
    int32_t nparts;
    float amax;  // max TF alpha over this rank's bricks (delta-tracking majorant, R-DELTA)
    PartInfo parts[MAXP];
};

struct StatsMsg {
    int64_t V[3];
    int64_t S[3][DPR_MAX_RANKS];
    int64_t gen[3];
    double ms_frame;
    int64_t nsteps;
    int64_t stepS[MAX_STEP_REC][3][DPR_MAX_RANKS];  // cumulative after each step (this rank's row)
    int64_t stepV[MAX_STEP_REC][3];
    double step_ms[MAX_STEP_REC], step_sync_ms[MAX_STEP_REC];
};

struct Dev {
    int rank = 0, nranks = 1, cuda_dev = 0, nsm = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t cstream = nullptr;          // side copy stream for geometry uploads
    cudaEvent_t copy_ev = nullptr, order_ev = nullptr;
    bool copy_pending = false;
    std::vector<Buf> part_pool;              // recycled geometry buffers
    // the committed world's volume state (renders use it while the parts of the next world
    // are being committed): bricks, their majorant, and brick buffers of cleared parts that
    // the committed world still references (freed by the next build)
    std::vector<BrickDev> wbricks;
    float amax_local = 0.0f;
    std::vector<Buf> retired;
    ncclComm_t comm = nullptr;
    LoopGroup *group = nullptr;
    dpr_allocator alloc{};
    bool has_alloc = false;
    std::vector<PartStore> parts;
    // world
    bool world_ready = false;
    int64_t nprims = 0;
    float box[6];
    bool nonempty = false;
    Buf b_prims_u, b_blo, b_bhi, b_keys[2], b_vals[2], b_tile, b_left, b_right, b_parent, b_rlo,
        b_rhi, b_nlo, b_nhi, b_arrive, b_prims, b_slo, b_shi, b_bounds, b_hist, b_wnodes, b_chunks,
        b_prims_w, b_items[2], b_wcnt, b_wperm, b_witems[2], b_size, b_bn;
    int builder = 1;  // 0 PLOC, 1 agglomerative LBVH (default), 2 Karras + refit (env DPR_BUILDER=ploc|karras)
    int build_iters = 0;
    int64_t wnodes_count = 0;
    int bvh_levels = 0;
    std::vector<PartInfo> local_parts;
    // frame
    dpr_camera_basis cam{};
    dpr_frame_desc fr{};
    bool cam_set = false, fr_set = false;
    Buf b_fb, b_fb_out, b_events, b_occl, b_ctr, b_counts, b_in_count, b_fetch, b_part_lo,
        b_part_alb, b_scratch;
    Buf b_path[2], b_occlq[2], b_send_path[DPR_MAX_RANKS], b_send_occl[DPR_MAX_RANKS];
    uint32_t path_cap = 0, occl_cap = 0;
    uint32_t *h_counts = nullptr;  // pinned: [N][2N+1]
    uint32_t *h_in = nullptr;      // pinned: [2]
    uint64_t *h_app = nullptr;     // pinned: Counters.app ([2][DPR_MAX_RANKS])
    uint64_t app_prev[2][DPR_MAX_RANKS] = {};  // host loop: Counters.app at the last boundary
    int frame_done = 0;
    int mapped_w = 0, mapped_h = 0;
    int spw = 16;  // max samples per warp in primary generation (env DPR_SPW; sweep r01)
    // exchange: 0 = per-step counts allgather + grouped ncclSend/ncclRecv (send-recv);
    //           1 = fused: kernels append straight into the destination rank's next queue
    //               (peer pointers, remote tail atomics); env DPR_EXCHANGE=fused|sendrecv
    int exch = 1;
    // step loop of the fused exchange: 1 = device-driven (one CUDA graph per spp batch: a
    // conditional WHILE node over the step kernels + k_step_end, no host round trip per
    // step), 0 = host loop (per-step counts to the host); env DPR_STEP_LOOP=host|device.
    // The send-recv exchange always needs the host (NCCL message sizes are host arguments).
    int step_loop = 1;
    Buf b_rec;                                    // StepRec of the current frame
    Buf b_more;                                   // [2] loop flags of the step graph
    Buf b_mbox, b_seq;                            // step-barrier mailbox (IPC-exported), sequence
    uint32_t *peer_mbox[DPR_MAX_RANKS] = {};
    float4 *peer_fb[DPR_MAX_RANKS] = {};          // host-collective mode: peers' framebuffers / dumps
    uint32_t *peer_events[DPR_MAX_RANKS] = {}, *peer_occl_dump[DPR_MAX_RANKS] = {};
    cudaStream_t gstream = nullptr, gstream2 = nullptr;  // capture streams of the step graph
    cudaGraph_t graph = nullptr;                  // device-driven step loop (cached per signature)
    cudaGraphExec_t gexec = nullptr;
    uint64_t gkey = 0;
    int64_t graph_kernels = 0;                    // kernel nodes per graph launch (counted at capture)
    int64_t graph_builds = 0;
    dpr_host_collectives hc{};                    // host-collective transport (no NCCL)
    bool has_hc = false;
    bool broken = false;                          // the communicator was aborted
    double timeout_s = 600.0;                     // collective / step-barrier timeout
    // per-step records of the last frame (global: every rank's rows)
    int64_t nsteps_rec = 0;
    std::vector<int64_t> step_S, step_V;          // [step][3][N][N], [step][3][N] (per-step deltas)
    std::vector<double> step_ms, step_sync_ms;    // [step] max over ranks
    Buf b_tails;                                  // [parity][kind] next-queue tails (fused)
    PathRec *peer_path[2][DPR_MAX_RANKS] = {};    // fused: every rank's queues, both parities
    OcclRec *peer_occl[2][DPR_MAX_RANKS] = {};
    uint32_t *peer_tails[DPR_MAX_RANKS] = {};
    std::vector<void *> ipc_opened;               // peer mappings to close
    uint64_t ipc_sig = 0;                         // signature of the exported buffers
    // compositing contrast device
    bool want_depth = false;
    Buf b_depth, b_frag_rgba, b_frag_z, b_comp, b_comp_out;
    Dev *lv = nullptr;                            // local-only view of this rank's world
    const float *frame_out = nullptr;             // what dpr_map_frame returns
    bool replicated_frame = false;                // last frame: dumps live in the local view
    int pix_rank = 0, pix_nranks = 1;             // replicated mode pixel split (local view)
    int64_t build_launches = 0, frame_exch_bytes = 0, tpl = 0, tol = 0;
    double ms_build = 0;
    bool dumps_valid = false;
    dpr_stats stats{};
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
};

// ---------------------------------------------------------------------------------------
int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess)                                                                  \
            return fail(e_ == cudaErrorMemoryAllocation ? DPR_ERR_OOM : DPR_ERR_CUDA,           \
                        std::string(#x) + ": " + cudaGetErrorString(e_));                       \
    } while (0)

#define NK(x)                                                                                   \
    do {                                                                                        \
        ncclResult_t r_ = (x);                                                                  \
        if (r_ != ncclSuccess) return fail(DPR_ERR_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_)); \
    } while (0)

#define RET(x)                    \
    do {                          \
        int rc_ = (x);            \
        if (rc_ != DPR_OK) return rc_; \
    } while (0)

void *dmalloc(Dev *d, size_t bytes) {
    if (bytes == 0) return nullptr;
    if (d->has_alloc) return d->alloc.alloc(d->alloc.ctx, bytes, d->stream);
    void *p = nullptr;
    if (cudaMallocAsync(&p, bytes, d->stream) != cudaSuccess) return nullptr;
    return p;
}

void dfree(Dev *d, Buf &b) {
    if (!b.p) return;
    if (b.raw) {
        cudaStreamSynchronize(d->stream);
        cudaFree(b.p);
        b.p = nullptr;
        b.bytes = 0;
        b.raw = false;
        return;
    }
    if (d->has_alloc) d->alloc.free(d->alloc.ctx, b.p, b.bytes, d->stream);
    else cudaFreeAsync(b.p, d->stream);
    b.p = nullptr;
    b.bytes = 0;
}

int ensure(Dev *d, Buf &b, size_t bytes) {
    if (b.bytes >= bytes && (b.p || bytes == 0)) return DPR_OK;
    dfree(d, b);
    if (bytes == 0) return DPR_OK;
    b.p = dmalloc(d, bytes);
    if (!b.p) return fail(DPR_ERR_OOM, "device allocation of " + std::to_string(bytes) + " bytes failed");
    b.bytes = bytes;
    return DPR_OK;
}

// cudaMalloc'd buffer (exportable with cudaIpcGetMemHandle for the fused NCCL exchange)
int ensure_raw(Dev *d, Buf &b, size_t bytes, bool *changed) {
    if (b.bytes >= bytes && b.p && b.raw) return DPR_OK;
    dfree(d, b);
    if (bytes == 0) return DPR_OK;
    if (cudaMalloc(&b.p, bytes) != cudaSuccess) {
        b.p = nullptr;
        return fail(DPR_ERR_OOM, "cudaMalloc of " + std::to_string(bytes) + " bytes failed");
    }
    b.bytes = bytes;
    b.raw = true;
    if (changed) *changed = true;
    return DPR_OK;
}

template <class T> T *P(Buf &b) { return reinterpret_cast<T *>(b.p); }

cudaEvent_t next_event(Dev *d) {
    if (d->ev_used == d->ev_pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        d->ev_pool.push_back(e);
    }
    return d->ev_pool[d->ev_used++];
}

uint64_t fnv1a(const void *p, size_t n, uint64_t h = 1469598103934665603ull) {
    const unsigned char *c = (const unsigned char *)p;
    for (size_t i = 0; i < n; ++i) { h ^= c[i]; h *= 1099511628211ull; }
    return h;
}

// Digest of the camera + frame parameters (P:349-353 consistency check), field by field: the
// structs' padding (dpr_frame_desc has 4 tail bytes after flags) never enters it.
uint64_t frame_digest(const Dev *d) {
    const dpr_camera_basis &c = d->cam;
    uint64_t h = fnv1a(c.E, sizeof(c.E));
    h = fnv1a(c.L, sizeof(c.L), h);
    h = fnv1a(c.U, sizeof(c.U), h);
    h = fnv1a(c.V, sizeof(c.V), h);
    h = fnv1a(&c.lens_radius, sizeof(float), h);
    h = fnv1a(&c.focus_dist, sizeof(float), h);
    const dpr_frame_desc &f = d->fr;
    const int32_t ints[6] = {f.W, f.H, f.spp, f.spp_batch, f.max_depth, f.ao_k};
    h = fnv1a(ints, sizeof(ints), h);
    h = fnv1a(&f.ao_radius, sizeof(float), h);
    h = fnv1a(f.light_dir, sizeof(f.light_dir), h);
    h = fnv1a(f.E, sizeof(f.E), h);
    h = fnv1a(f.A, sizeof(f.A), h);
    h = fnv1a(f.B, sizeof(f.B), h);
    h = fnv1a(&f.dt, sizeof(float), h);
    h = fnv1a(&f.seed, sizeof(f.seed), h);
    return fnv1a(&f.flags, sizeof(f.flags), h);
}

bool valid_dev(dpr_device h) { return h != nullptr; }

// ---------------------------------------------------------------------------------------
// Collectives (NCCL or loopback).  `L` is the list of local ranks (1 for NCCL mode).
// ---------------------------------------------------------------------------------------
// Abort the communicator after an NCCL (async) error or a collective timeout: every later
// collective call on this device returns DPR_ERR_NCCL (dpr.h: release the device).
int abort_comm(Dev *d, const std::string &why) {
    if (d->comm) ncclCommAbort(d->comm);
    d->comm = nullptr;
    d->broken = true;
    return fail(DPR_ERR_NCCL, why + " (communicator aborted)");
}

// Wait for the device's stream.  With NCCL, poll the stream and ncclCommGetAsyncError, and give
// up after timeout_s (a dead peer would otherwise hang the collective forever): abort.
// Test hook DPR_TEST_NCCL_FAULT=1 reports an asynchronous NCCL error at the first poll.
int wait_stream(Dev *d) {
    if (!d->comm) {
        CK(cudaStreamSynchronize(d->stream));
        return DPR_OK;
    }
    const bool fault = getenv("DPR_TEST_NCCL_FAULT") && atoi(getenv("DPR_TEST_NCCL_FAULT")) == 1;
    const auto t0 = std::chrono::steady_clock::now();
    for (int it = 0;; ++it) {
        const cudaError_t e = cudaStreamQuery(d->stream);
        if (e == cudaSuccess) return DPR_OK;
        if (e != cudaErrorNotReady)
            return fail(DPR_ERR_CUDA, std::string("stream: ") + cudaGetErrorString(e));
        ncclResult_t ar = ncclSuccess;
        if (ncclCommGetAsyncError(d->comm, &ar) != ncclSuccess || fault)
            ar = ncclSystemError;
        if (ar != ncclSuccess && ar != ncclInProgress)
            return abort_comm(d, std::string("NCCL asynchronous error: ") + ncclGetErrorString(ar));
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (el > d->timeout_s) return abort_comm(d, "collective timed out");
        if (it > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}

// ---------------------------------------------------------------------------------------
// Collectives (NCCL, host collectives, or loopback).  `L` is the list of local ranks (1 for
// NCCL / host-collective mode).
// ---------------------------------------------------------------------------------------
int allgather_host(std::vector<Dev *> &L, const std::vector<const void *> &send, size_t bytes,
                   std::vector<std::vector<char>> &out) {
    Dev *d0 = L[0];
    int N = d0->nranks;
    if (d0->broken) return fail(DPR_ERR_NCCL, "communicator was aborted; release the device");
    if (d0->has_hc) {  // host-collective transport (blocking, every rank calls it)
        out.assign(1, std::vector<char>((size_t)N * bytes));
        if (d0->hc.allgather(d0->hc.ctx, send[0], out[0].data(), bytes) != 0)
            return fail(DPR_ERR_NCCL, "host-collective allgather failed");
        return DPR_OK;
    }
    if (!d0->comm) {  // loopback group or single rank without NCCL
        std::vector<char> all((size_t)N * bytes);
        for (size_t i = 0; i < L.size(); ++i) memcpy(all.data() + (size_t)L[i]->rank * bytes, send[i], bytes);
        out.assign(L.size(), all);
        return DPR_OK;
    }
    RET(ensure(d0, d0->b_scratch, bytes * (N + 1)));
    char *sbuf = P<char>(d0->b_scratch), *rbuf = sbuf + bytes;
    CK(cudaMemcpyAsync(sbuf, send[0], bytes, cudaMemcpyHostToDevice, d0->stream));
    NK(ncclAllGather(sbuf, rbuf, bytes, ncclUint8, d0->comm, d0->stream));
    out.assign(1, std::vector<char>((size_t)N * bytes));
    CK(cudaMemcpyAsync(out[0].data(), rbuf, bytes * N, cudaMemcpyDeviceToHost, d0->stream));
    RET(wait_stream(d0));
    return DPR_OK;
}

// A barrier of the host-collective transport (after the local stream is idle).
int hc_barrier(Dev *d) {
    CK(cudaStreamSynchronize(d->stream));
    std::vector<Dev *> L = {d};
    const uint32_t one = 1;
    std::vector<const void *> snd = {&one};
    std::vector<std::vector<char>> o;
    return allgather_host(L, snd, sizeof(one), o);
}

// ---------------------------------------------------------------------------------------
// World build (a1).
// ---------------------------------------------------------------------------------------
int build_world(Dev *d) {
    cudaStream_t s = d->stream;
    d->world_ready = false;  // until this build succeeds (dpr.h: a failed commit leaves no world)
    if (d->copy_pending) {  // geometry copied on the side stream (DPR_MEMORY_HOST_ASYNC)
        CK(cudaStreamWaitEvent(s, d->copy_ev, 0));
        d->copy_pending = false;
    }
    int64_t n = 0;
    for (auto &p : d->parts) n += p.nprims();
    if (n >= (int64_t)0x0fffffff) return fail(DPR_ERR_INVALID_ARG, "too many primitives on one rank (max 2^28-2)");
    d->nprims = n;
    int np = (int)d->parts.size();
    // per-part bounds + overall centroid box
    RET(ensure(d, d->b_bounds, sizeof(int) * (12 * (np + 1) + 1)));
    std::vector<int> binit(12 * (np + 1) + 1, 0);  // last word: bad triangle index flag
    for (int k = 0; k <= np; ++k)
        for (int c = 0; c < 12; ++c) binit[12 * k + c] = (c % 6) < 3 ? 0x7fffffff : (int)0x80000000;
    CK(cudaMemcpyAsync(d->b_bounds.p, binit.data(), binit.size() * sizeof(int), cudaMemcpyHostToDevice, s));
    if (n > 0) {
        RET(ensure(d, d->b_prims_u, sizeof(float4) * 3 * n));
        RET(ensure(d, d->b_blo, sizeof(float4) * 2 * n));  // prim boxes, lo / hi interleaved (32 B each)
    }
    int64_t off = 0;
    int launches = 0;
    // all parts' prim records, boxes and bounds in one launch (one block per chunk)
    std::vector<PrimChunk> chunks;
    for (int k = 0; k < np; ++k) {
        PartStore &p = d->parts[k];
        const int64_t cnt = p.nprims();
        for (int64_t st = 0; st < cnt; st += PRIM_CHUNK) {
            PrimChunk c;
            c.src = p.kind == DPR_PART_TRIANGLES ? (const void *)P<float>(p.verts) : (const void *)P<float4>(p.spheres);
            c.idx = p.kind == DPR_PART_TRIANGLES ? P<int32_t>(p.idx) : nullptr;
            c.nv = p.nv;
            c.start = st;
            c.g0 = (uint32_t)(off + st);
            c.count = (int)std::min<int64_t>(PRIM_CHUNK, cnt - st);
            c.kind = p.kind;
            c.slot = k + 1;
            chunks.push_back(c);
        }
        off += cnt;
    }
    if (!chunks.empty()) {
        RET(ensure(d, d->b_chunks, sizeof(PrimChunk) * chunks.size()));
        CK(cudaMemcpyAsync(d->b_chunks.p, chunks.data(), sizeof(PrimChunk) * chunks.size(), cudaMemcpyHostToDevice, s));
        launch_part_prims(P<PrimChunk>(d->b_chunks), (int)chunks.size(), P<float4>(d->b_prims_u), P<float4>(d->b_blo),
                          P<float4>(d->b_blo) + 1, P<int>(d->b_bounds), P<int>(d->b_bounds) + 12 * (np + 1), s);
        launches++;
    }
    // Morton keys (+ the first radix pass's tile histogram)
    if (n > 0) {
        for (int i = 0; i < 2; ++i) {
            RET(ensure(d, d->b_keys[i], sizeof(mkey_t) * n + 64));  // + the agglomeration fetch counter
            RET(ensure(d, d->b_vals[i], sizeof(uint32_t) * n));
        }
        RET(ensure(d, d->b_tile, sizeof(uint32_t) * 256 * (radix_tiles(n) + 1)));
        launch_morton_h(P<float4>(d->b_blo), P<float4>(d->b_blo) + 1, n, P<int>(d->b_bounds), P<mkey_t>(d->b_keys[0]),
                        P<uint32_t>(d->b_vals[0]), P<uint32_t>(d->b_tile), nullptr, s);
        launches += 1;
    }
    // part bounds + validation flags: read back without a wait here; checked after the build's
    // first host synchronisation (the collapse level counts), so the GPU runs the whole build
    // without draining in between (a failed check then leaves no world, as before)
    std::vector<int> bnd(12 * (np + 1) + 1);
    CK(cudaMemcpyAsync(bnd.data(), d->b_bounds.p, bnd.size() * sizeof(int), cudaMemcpyDeviceToHost, s));
    auto finish_bounds = [&]() -> int {
    if (bnd[12 * (np + 1)] & 1) return fail(DPR_ERR_INVALID_ARG, "triangle index out of range (checked on the GPU)");
    if (bnd[12 * (np + 1)] & 2)
        return fail(DPR_ERR_INVALID_ARG, "non-finite vertex / sphere, or sphere radius <= 0 (checked on the GPU)");
    auto ord2f = [](int i) { int j = i >= 0 ? i : i ^ 0x7fffffff; float f; memcpy(&f, &j, 4); return f; };
    // rank box = exact union of prim boxes and brick cell-domain boxes (P8)
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    d->local_parts.clear();
    off = 0;
    for (int k = 0; k < np; ++k) {
        PartStore &p = d->parts[k];
        float plo[3], phi[3];
        bool have = false;
        if (p.kind == DPR_PART_BRICK) {
            for (int c = 0; c < 3; ++c) {
                plo[c] = p.origin[c] + (float)p.lo[c] * p.spacing[c];
                phi[c] = p.origin[c] + (float)p.hi[c] * p.spacing[c];
            }
            have = true;
        } else if (p.nprims() > 0) {
            for (int c = 0; c < 3; ++c) { plo[c] = ord2f(bnd[12 * (k + 1) + c]); phi[c] = ord2f(bnd[12 * (k + 1) + 3 + c]); }
            have = true;
            PartInfo pi{};
            pi.first = (uint32_t)off;
            pi.count = (uint32_t)p.nprims();
            for (int c = 0; c < 3; ++c) pi.albedo[c] = p.albedo[c];
            d->local_parts.push_back(pi);
        }
        if (have) {
            if (p.has_hint)
                for (int c = 0; c < 3; ++c)
                    if (!(p.hint[c] <= plo[c] && p.hint[3 + c] >= phi[c]))
                        return fail(DPR_ERR_INVALID_ARG, "part " + std::to_string(k) + ": bounds_hint does not contain the part");
            for (int c = 0; c < 3; ++c) { lo[c] = fminf(lo[c], plo[c]); hi[c] = fmaxf(hi[c], phi[c]); }
        }
        off += p.nprims();
    }
    if ((int)d->local_parts.size() > MAXP) return fail(DPR_ERR_INVALID_ARG, "too many parts on one rank");
    d->nonempty = lo[0] <= hi[0];
    for (int c = 0; c < 3; ++c) { d->box[c] = lo[c]; d->box[3 + c] = hi[c]; }
    return DPR_OK;
    };
    if (n > 0) {
        // LSD radix sort, all four passes (a constant digit is an identity pass: stable)
        int cur = 0;
        for (int pass = 0; pass < MKEY_DIGITS; ++pass) {
            // pass 0's tile histogram came with the Morton codes (keys still in input order)
            launch_radix_pass(P<mkey_t>(d->b_keys[cur]), P<uint32_t>(d->b_vals[cur]),
                              P<mkey_t>(d->b_keys[cur ^ 1]), P<uint32_t>(d->b_vals[cur ^ 1]), n,
                              8 * pass, P<uint32_t>(d->b_tile), s, &launches, pass == 0);
            cur ^= 1;
        }
        mkey_t *keys = P<mkey_t>(d->b_keys[cur]);
        uint32_t *perm = P<uint32_t>(d->b_vals[cur]);
        // packed leaf records in Morton order: leaf[2j] = lo, leaf[2j+1] = hi
        RET(ensure(d, d->b_slo, sizeof(float4) * 2 * n));
        float4 *leaf = P<float4>(d->b_slo);
        launch_gather_prims(P<float4>(d->b_prims_u), perm, n, nullptr, P<float4>(d->b_blo),
                            P<float4>(d->b_blo) + 1, leaf, leaf + 1, s);
        launches++;
        int root_id = 0;
        const int *root_dev = nullptr;  // device copy of the root id (agglomerative builder)
        if (n > 1) RET(ensure(d, d->b_bn, sizeof(BNode) * (n - 1)));
        if (n > 1 && d->builder != 1) {  // separate arrays of the Karras / PLOC builders
            RET(ensure(d, d->b_left, sizeof(int) * (n - 1)));
            RET(ensure(d, d->b_right, sizeof(int) * (n - 1)));
            RET(ensure(d, d->b_size, sizeof(int) * (n - 1)));
            RET(ensure(d, d->b_nlo, sizeof(float4) * (n - 1)));
            RET(ensure(d, d->b_nhi, sizeof(float4) * (n - 1)));
        }
        if (n > 1) {
            if (d->builder == 0) {
                // PLOC (DPR_BUILDER=ploc): locally-ordered agglomerative clustering on the Morton order
                RET(ensure(d, d->b_items[0], sizeof(int) * n));  // reused as cluster lists
                RET(ensure(d, d->b_items[1], sizeof(int) * n));
                RET(ensure(d, d->b_parent, sizeof(int) * n));     // reused as nearest neighbours
                int64_t nbmax = ploc_block_count(n);
                RET(ensure(d, d->b_rlo, sizeof(int) * 2 * nbmax + 16));  // block counts + totals
                PlocArgs pa;
                pa.n = n; pa.slo = leaf; pa.shi = leaf + 1;
                pa.nlo = P<float4>(d->b_nlo); pa.nhi = P<float4>(d->b_nhi);
                pa.left = P<int>(d->b_left); pa.right = P<int>(d->b_right); pa.size = P<int>(d->b_size);
                int *cl[2] = {P<int>(d->b_items[0]), P<int>(d->b_items[1])};
                int *nn = P<int>(d->b_parent);
                int *bc = P<int>(d->b_rlo);
                int *tot = bc + 2 * nbmax + 8;
                launch_ploc_init(n, cl[0], s);
                int64_t m = n;
                int node_base = 0, c = 0, iters = 0;
                int h_tot[2];
                while (m > 1) {
                    int64_t nb = ploc_block_count(m);
                    launch_ploc_nn(pa, cl[c], m, nn, s);
                    launch_ploc_count(nn, m, bc, s);
                    launch_ploc_scan(bc, nb, tot, s);
                    launch_ploc_write(pa, cl[c], nn, m, bc, node_base, cl[c ^ 1], s);
                    launches += 4;
                    CK(cudaMemcpyAsync(h_tot, tot, sizeof(h_tot), cudaMemcpyDeviceToHost, s));
                    CK(cudaStreamSynchronize(s));
                    if (h_tot[1] <= 0) return fail(DPR_ERR_STATE, "PLOC made no progress");
                    m = h_tot[0];
                    node_base += h_tot[1];
                    c ^= 1;
                    iters++;
                }
                if (node_base != n - 1) return fail(DPR_ERR_STATE, "PLOC produced a wrong node count");
                CK(cudaMemcpyAsync(&root_id, cl[c], sizeof(int), cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                d->build_iters = iters;
                launch_pack_bnodes(n, P<int>(d->b_left), P<int>(d->b_right), P<int>(d->b_size), P<float4>(d->b_nlo),
                                   P<float4>(d->b_nhi), P<BNode>(d->b_bn), s);
                launches++;
            } else if (d->builder == 1) {
                // agglomerative LBVH (default): topology + boxes in one bottom-up pass
                // exchange words: 8 bytes per internal node (all ones = no arrival yet), then the root id
                RET(ensure(d, d->b_arrive, sizeof(unsigned long long) * (n - 1) + sizeof(int)));
                unsigned long long *other = P<unsigned long long>(d->b_arrive);
                CK(cudaMemsetAsync(other, 0xff, sizeof(unsigned long long) * (n - 1), s));
                // the other radix-sort key buffer is free now: per-split prefix lengths
                uint8_t *split = P<uint8_t>(d->b_keys[keys == P<mkey_t>(d->b_keys[0]) ? 1 : 0]);
                int *root = reinterpret_cast<int *>(other + (n - 1));
                launches += launch_agglo(keys, split, n, leaf, P<BNode>(d->b_bn), other, root, s);
                root_dev = root;  // read by the first collapse level on the device
            } else {
                // Karras 2012 LBVH + bottom-up refit
                RET(ensure(d, d->b_rlo, sizeof(int) * (n - 1)));
                RET(ensure(d, d->b_rhi, sizeof(int) * (n - 1)));
                RET(ensure(d, d->b_parent, sizeof(int) * (2 * n - 1)));
                RET(ensure(d, d->b_arrive, sizeof(int) * (n - 1)));
                CK(cudaMemsetAsync(d->b_arrive.p, 0, sizeof(int) * (n - 1), s));
                launch_karras(keys, n, P<int>(d->b_left), P<int>(d->b_right), P<int>(d->b_parent),
                              P<int>(d->b_rlo), P<int>(d->b_rhi), P<int>(d->b_size), s);
                launch_refit(n, P<int>(d->b_left), P<int>(d->b_right), P<int>(d->b_parent), leaf, leaf + 1,
                             P<float4>(d->b_nlo), P<float4>(d->b_nhi), P<int>(d->b_arrive), s);
                launch_pack_bnodes(n, P<int>(d->b_left), P<int>(d->b_right), P<int>(d->b_size), P<float4>(d->b_nlo),
                                   P<float4>(d->b_nhi), P<BNode>(d->b_bn), s);
                launches += 3;
            }
        }
        // collapse into compressed 8-wide nodes, one BFS level per launch
        const int node_cap = (int)std::max<int64_t>(n, 2);
        RET(ensure(d, d->b_wnodes, sizeof(WNode) * node_cap));
        RET(ensure(d, d->b_prims_w, sizeof(float4) * 3 * n));
        RET(ensure(d, d->b_wperm, sizeof(uint32_t) * n));
        RET(ensure(d, d->b_witems[0], sizeof(int2) * node_cap));
        RET(ensure(d, d->b_witems[1], sizeof(int2) * node_cap));
        RET(ensure(d, d->b_wcnt, sizeof(int) * 4));
        // levels are launched in batches without a host round trip: each level kernel reads its
        // item count from device memory (lvl[L]) and appends the next level's (lvl[L+1])
        // the first batch covers the expected depth (log8 n + 3 levels: 9 of 10M prims, 11 of 55M),
        // so the usual build makes one host round trip here; then batches of 4
        constexpr int MAXL = 120, BATCH = 4, MAXB = 32;
        int first_batch = 3;
        for (int64_t m = 1; m < n && first_batch < MAXB; m *= 8) first_batch++;
        RET(ensure(d, d->b_wcnt, sizeof(int) * (4 + MAXL + MAXB + 1)));
        int *cnt = P<int>(d->b_wcnt), *lvl = cnt + 4;
        CK(cudaMemsetAsync(cnt, 0, sizeof(int) * (4 + MAXL + MAXB + 1), s));
        int h_init[5] = {0, 1, 0, 0, 1};  // counters {-, nodes = 1 (root), prims, overflow}, lvl[0] = 1
        CK(cudaMemcpyAsync(cnt, h_init, sizeof(h_init), cudaMemcpyHostToDevice, s));
        int2 root = make_int2(0, n > 1 ? root_id : -1);
        CK(cudaMemcpyAsync(d->b_witems[0].p, &root, sizeof(root), cudaMemcpyHostToDevice, s));
        if (n > 1 && root_dev)  // agglomerative builder: the root id stays on the device
            CK(cudaMemcpyAsync(&P<int2>(d->b_witems[0])->y, root_dev, sizeof(int), cudaMemcpyDeviceToDevice, s));
        CollapseArgs ca;
        ca.n = n; ca.bn = P<BNode>(d->b_bn); ca.leaf = leaf;
        ca.perm = P<uint32_t>(d->b_wperm); ca.nodes = P<WNode>(d->b_wnodes); ca.counters = cnt;
        ca.node_cap = node_cap;
        int h_cnt[4 + MAXL + MAXB + 1];
        int levels = -1;
        for (int L = 0, B = first_batch; levels < 0; L += B, B = BATCH) {
            if (L >= MAXL) return fail(DPR_ERR_STATE, "wide BVH deeper than the collapse level limit");
            for (int k = L; k < L + B; ++k) {
                launch_collapse_level(ca, P<int2>(d->b_witems[k & 1]), lvl + k, P<int2>(d->b_witems[(k + 1) & 1]),
                                      lvl + k + 1, k, s);
                launches++;
            }
            CK(cudaMemcpyAsync(h_cnt, cnt, sizeof(int) * (4 + L + B + 1), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (h_cnt[3]) return fail(DPR_ERR_STATE, "wide BVH node capacity exceeded");
            for (int k = L; k <= L + B; ++k)
                if (h_cnt[4 + k] == 0) { levels = k; break; }
        }
        RET(finish_bounds());
        if (h_cnt[2] != n) return fail(DPR_ERR_STATE, "wide BVH collapse lost primitives");
        launch_permute_prims(P<float4>(d->b_prims_u), P<uint32_t>(d->b_wperm), perm, n, P<float4>(d->b_prims_w), s);
        launches++;
        d->wnodes_count = h_cnt[1];
#ifdef DPR_COLLAPSE_STATS
        fprintf(stderr, "collapse: %d wide nodes, %.3f children per node, %.3f prims per leaf child\n", h_cnt[1],
                (double)h_cnt[0] / h_cnt[1], (double)n / (h_cnt[0] - (h_cnt[1] - 1)));
#endif
        d->bvh_levels = levels;
    } else {
        CK(cudaStreamSynchronize(s));
        RET(finish_bounds());
    }
    // bricks: macrocells
    for (auto &p : d->parts) {
        if (p.kind != DPR_PART_BRICK) continue;
        int nx = p.hi[0] - p.lo[0] + 1, ny = p.hi[1] - p.lo[1] + 1, nz = p.hi[2] - p.lo[2] + 1;
        for (int c = 0; c < 3; ++c) p.mc_dims[c] = (p.hi[c] - p.lo[c] + MC_SIZE - 1) / MC_SIZE;
        size_t nm = (size_t)p.mc_dims[0] * p.mc_dims[1] * p.mc_dims[2];
        RET(ensure(d, p.mc, std::max<size_t>(3 * nm, 1)));  // flags | distance field | scratch
        launches += launch_macrocells(P<float>(p.vox), nx, ny, nz, p.mc_dims[0], p.mc_dims[1], p.mc_dims[2],
                                      P<float4>(p.tf), p.tf_lo, p.tf_hi, p.dscale, P<uint8_t>(p.mc), s);
    }
    CK(cudaGetLastError());
    // snapshot of the volume state of this world
    d->wbricks.clear();
    d->amax_local = 0.0f;
    for (auto &p : d->parts) {
        if (p.kind != DPR_PART_BRICK || (int)d->wbricks.size() >= MAX_BRICKS) continue;
        BrickDev B;
        for (int c = 0; c < 3; ++c) {
            B.lo[c] = p.lo[c]; B.hi[c] = p.hi[c]; B.mc_dims[c] = p.mc_dims[c];
            B.O[c] = p.origin[c]; B.h[c] = p.spacing[c];
            B.box_lo[c] = p.origin[c] + (float)p.lo[c] * p.spacing[c];
            B.box_hi[c] = p.origin[c] + (float)p.hi[c] * p.spacing[c];
            B.gd[c] = p.gdims[c];
        }
        B.vox = P<float>(p.vox); B.mc = P<uint8_t>(p.mc);
        B.mcd = P<uint8_t>(p.mc) + (size_t)p.mc_dims[0] * p.mc_dims[1] * p.mc_dims[2];
        B.tf = P<float4>(p.tf);
        B.tf_lo = p.tf_lo; B.tf_hi = p.tf_hi; B.dscale = p.dscale;
        B.tf_rd = exact_recip_pow2(B.tf_hi - B.tf_lo);  // the same binary32 difference as the kernels

        d->wbricks.push_back(B);
        d->amax_local = std::max(d->amax_local, p.amax);
    }
    for (auto &b : d->retired) dfree(d, b);  // stream-ordered after the renders that used them
    d->retired.clear();
    d->build_launches = launches;
    d->world_ready = true;
    return DPR_OK;
}

// ---------------------------------------------------------------------------------------
// Frame.
// ---------------------------------------------------------------------------------------
struct FrameCtx {
    Routing R;
    float amax = 0.0f;  // global delta-tracking majorant
    std::vector<uint32_t> id_base;
    std::vector<uint32_t> part_lo;
    std::vector<float4> part_alb;
};

int frame_setup(std::vector<Dev *> &L, FrameCtx &fc) {
    Dev *d0 = L[0];
    const int N = d0->nranks;
    std::vector<RankInfo> infos(L.size());
    std::vector<const void *> sends;
    for (size_t i = 0; i < L.size(); ++i) {
        Dev *d = L[i];
        RankInfo &ri = infos[i];
        memset(&ri, 0, sizeof(ri));
        ri.digest = frame_digest(d);
        for (int c = 0; c < 6; ++c) ri.box[c] = d->box[c];
        ri.nonempty = d->nonempty;
        ri.nprims = (uint32_t)d->nprims;
        ri.nparts = (int)d->local_parts.size();
        for (int k = 0; k < ri.nparts; ++k) ri.parts[k] = d->local_parts[k];
        ri.amax = d->amax_local;
        sends.push_back(&ri);
    }
    std::vector<std::vector<char>> out;
    RET(allgather_host(L, sends, sizeof(RankInfo), out));
    const RankInfo *all = reinterpret_cast<const RankInfo *>(out[0].data());
    for (int r = 1; r < N; ++r)
        if (all[r].digest != all[0].digest)
            return fail(DPR_ERR_CONSISTENCY, "camera/frame parameters differ between ranks (rank " +
                                                 std::to_string(r) + " vs rank 0)");
    fc.R.nranks = N;
    fc.id_base.assign(N, 0);
    uint64_t base = 0;
    for (int r = 0; r < N; ++r) {
        fc.id_base[r] = (uint32_t)base;
        base += all[r].nprims;
        fc.R.nonempty[r] = all[r].nonempty;
        if (all[r].amax > fc.amax) fc.amax = all[r].amax;
        for (int c = 0; c < 3; ++c) {  // P8 padding, f32 host arithmetic
            fc.R.box[r][c] = all[r].box[c] - 1e-4f;
            fc.R.box[r][3 + c] = all[r].box[3 + c] + 1e-4f;
        }
        for (int k = 0; k < all[r].nparts; ++k) {
            const PartInfo &pi = all[r].parts[k];
            fc.part_lo.push_back(fc.id_base[r] + pi.first);
            fc.part_alb.push_back(make_float4(pi.albedo[0], pi.albedo[1], pi.albedo[2], 0.0f));
        }
    }
    if (base >= 0x7fffffffull) return fail(DPR_ERR_INVALID_ARG, "more than 2^31-1 primitives in the world");
    if (fc.part_lo.empty()) { fc.part_lo.push_back(0); fc.part_alb.push_back(make_float4(0, 0, 0, 0)); }
    return DPR_OK;
}

int frame_buffers(Dev *d, const FrameCtx &fc) {
    const dpr_frame_desc &f = d->fr;
    const int N = d->nranks;
    int64_t P_ = (int64_t)f.W * f.H;
    int64_t rays = P_ * f.spp_batch;
    if (rays > 0xe0000000ll) return fail(DPR_ERR_INVALID_ARG, "W*H*spp_batch too large for 32-bit queues");
    uint32_t pcap = (uint32_t)rays;
    int64_t ocap64 = rays * (1 + f.ao_k) * f.max_depth;
    if (ocap64 > 0xfffffff0ll) ocap64 = 0xfffffff0ll;
    uint32_t ocap = (uint32_t)ocap64;
    // IPC-exported (cudaMalloc'd) buffers: fused queues with NCCL or host collectives; in
    // host-collective mode also the framebuffer and dumps (rank 0 reduces through mappings)
    const bool ipc = d->exch && (d->comm || d->has_hc);
    if (d->has_hc) {
        RET(ensure_raw(d, d->b_fb, sizeof(float4) * P_, nullptr));
    } else {
        RET(ensure(d, d->b_fb, sizeof(float4) * P_));
    }
    RET(ensure(d, d->b_fb_out, sizeof(float4) * P_));
    if (f.flags & DPR_FLAG_DEBUG_DUMPS) {
        size_t nd = (size_t)f.spp * f.max_depth * P_;
        if (d->has_hc) {
            RET(ensure_raw(d, d->b_events, sizeof(uint32_t) * nd, nullptr));
            RET(ensure_raw(d, d->b_occl, sizeof(uint32_t) * nd, nullptr));
        } else {
            RET(ensure(d, d->b_events, sizeof(uint32_t) * nd));
            RET(ensure(d, d->b_occl, sizeof(uint32_t) * nd));
        }
    }
    for (int i = 0; i < 2; ++i) {
        if (ipc) {
            RET(ensure_raw(d, d->b_path[i], sizeof(PathRec) * (size_t)pcap, nullptr));
            RET(ensure_raw(d, d->b_occlq[i], sizeof(OcclRec) * (size_t)ocap, nullptr));
        } else {
            RET(ensure(d, d->b_path[i], sizeof(PathRec) * (size_t)pcap));
            RET(ensure(d, d->b_occlq[i], sizeof(OcclRec) * (size_t)ocap));
        }
    }
    if (d->exch) {
        if (ipc) RET(ensure_raw(d, d->b_tails, sizeof(uint32_t) * 4, nullptr));
        else RET(ensure(d, d->b_tails, sizeof(uint32_t) * 4));
        CK(cudaMemsetAsync(d->b_tails.p, 0, sizeof(uint32_t) * 4, d->stream));
    } else {
        for (int r = 0; r < N; ++r) {
            if (r == d->rank) continue;
            RET(ensure(d, d->b_send_path[r], sizeof(PathRec) * (size_t)pcap));
            RET(ensure(d, d->b_send_occl[r], sizeof(OcclRec) * (size_t)ocap));
        }
    }
    d->path_cap = pcap;
    d->occl_cap = ocap;
    RET(ensure(d, d->b_ctr, sizeof(Counters)));
    RET(ensure(d, d->b_rec, sizeof(StepRec)));
    RET(ensure(d, d->b_more, sizeof(uint32_t) * 4));
    RET(ensure(d, d->b_counts, sizeof(uint32_t) * (2 * N + 1)));
    RET(ensure(d, d->b_in_count, sizeof(uint32_t) * 2));
    RET(ensure(d, d->b_fetch, sizeof(uint32_t) * 4));  // trace path/occl, march path/occl
    RET(ensure(d, d->b_part_lo, sizeof(uint32_t) * fc.part_lo.size()));
    RET(ensure(d, d->b_part_alb, sizeof(float4) * fc.part_alb.size()));
    if (!d->h_counts) {
        CK(cudaMallocHost(&d->h_counts, sizeof(uint32_t) * DPR_MAX_RANKS * (2 * DPR_MAX_RANKS + 1)));
        CK(cudaMallocHost(&d->h_in, sizeof(uint32_t) * 2));
        CK(cudaMallocHost(&d->h_app, sizeof(uint64_t) * 2 * DPR_MAX_RANKS));
    }
    cudaStream_t s = d->stream;
    CK(cudaMemcpyAsync(d->b_part_lo.p, fc.part_lo.data(), sizeof(uint32_t) * fc.part_lo.size(), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d->b_part_alb.p, fc.part_alb.data(), sizeof(float4) * fc.part_alb.size(), cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(d->b_fb.p, 0, sizeof(float4) * P_, s));
    if (f.flags & DPR_FLAG_DEBUG_DUMPS) {
        size_t nd = (size_t)f.spp * f.max_depth * P_;
        CK(cudaMemsetAsync(d->b_events.p, 0, sizeof(uint32_t) * nd, s));
        CK(cudaMemsetAsync(d->b_occl.p, 0, sizeof(uint32_t) * nd, s));
    }
    CK(cudaMemsetAsync(d->b_ctr.p, 0, sizeof(Counters), s));
    memset(d->app_prev, 0, sizeof(d->app_prev));
    CK(cudaMemsetAsync(d->b_rec.p, 0, sizeof(StepRec), s));
    CK(cudaMemsetAsync(d->b_more.p, 0, sizeof(uint32_t) * 4, s));
    CK(cudaMemsetAsync(d->b_fetch.p, 0, sizeof(uint32_t) * 4, s));
    if (d->want_depth) {
        RET(ensure(d, d->b_depth, sizeof(uint32_t) * P_));
        launch_depth_init(P<uint32_t>(d->b_depth), P_, s);
    }
    return DPR_OK;
}

// Conservative pixel rectangle of the projection of this rank's padded routing box (P8): a
// primary ray whose first candidate is this rank passes through the box, so its pixel lies in
// the projection.  A point X is seen through screen position (sx, sy) iff
// X - E = lam * (L + sx*U + sy*V) with lam > 0 (P2), i.e. (lam, lam*sx, lam*sy) solves the 3x3
// system [L U V] * y = X - E -- for ANY basis (sheared / off-axis / cropped image regions
// included).  With every corner in front (lam > 0; lam is linear, so the whole box is), the
// box projects into the convex hull of its corners' projections.  Solved in double with a
// 2-pixel margin; the whole frame when the basis is (nearly) singular, a corner is not in
// front of the eye, for thin-lens cameras, at N=1; an empty rect for an empty rank (then
// only the pixel owner's misses matter).
void gen_rect(const Dev *d, const FrameCtx &fc, int rect[4]) {
    const int W = d->fr.W, H = d->fr.H;
    rect[0] = 0; rect[1] = 0; rect[2] = W; rect[3] = H;
    static const bool off = getenv("DPR_GEN_CULL") && atoi(getenv("DPR_GEN_CULL")) == 0;
    if (off || fc.R.nranks <= 1 || d->cam.lens_radius > 0.0f) return;
    if (!fc.R.nonempty[d->rank]) { rect[2] = 0; rect[3] = 0; return; }
    const dpr_camera_basis &c = d->cam;
    // columns L, U, V; inverse by the adjugate (cofactors in double)
    const double M[3][3] = {{c.L[0], c.U[0], c.V[0]}, {c.L[1], c.U[1], c.V[1]}, {c.L[2], c.U[2], c.V[2]}};
    double A[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
            A[j][i] = M[i1][j1] * M[i2][j2] - M[i1][j2] * M[i2][j1];  // adj = cofactor^T
        }
    const double det = M[0][0] * A[0][0] + M[0][1] * A[1][0] + M[0][2] * A[2][0];
    double scale = 0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) scale = std::max(scale, std::fabs(M[i][j]));
    if (!(std::fabs(det) > 1e-9 * scale * scale * scale)) return;  // degenerate basis: whole frame
    double x0 = 1e300, x1 = -1e300, y0 = 1e300, y1 = -1e300;
    const float *b = fc.R.box[d->rank];
    for (int m = 0; m < 8; ++m) {
        double X[3] = {b[(m & 1) ? 3 : 0], b[(m & 2) ? 4 : 1], b[(m & 4) ? 5 : 2]};
        double rel[3] = {X[0] - c.E[0], X[1] - c.E[1], X[2] - c.E[2]};
        double y[3];
        for (int i = 0; i < 3; ++i) y[i] = (A[i][0] * rel[0] + A[i][1] * rel[1] + A[i][2] * rel[2]) / det;
        const double lam = y[0];
        if (!(lam > 1e-9 * std::sqrt(rel[0] * rel[0] + rel[1] * rel[1] + rel[2] * rel[2]) / std::max(scale, 1e-30)))
            return;  // a corner at or behind the eye plane: whole frame
        const double su = y[1] / lam, sv = y[2] / lam;
        x0 = std::min(x0, su * W); x1 = std::max(x1, su * W);
        y0 = std::min(y0, sv * H); y1 = std::max(y1, sv * H);
    }
    if (!(x0 > -1e9 && x1 < 1e9 && y0 > -1e9 && y1 < 1e9)) return;
    rect[0] = (int)std::max(0.0, std::floor(x0) - 2.0);
    rect[1] = (int)std::max(0.0, std::floor(y0) - 2.0);
    rect[2] = (int)std::min((double)W, std::ceil(x1) + 2.0);
    rect[3] = (int)std::min((double)H, std::ceil(y1) + 2.0);
    if (rect[2] < rect[0]) rect[2] = rect[0];
    if (rect[3] < rect[1]) rect[3] = rect[1];
}

StepArgs make_args(Dev *d, const FrameCtx &fc, int cur) {
    StepArgs a;
    memset(&a, 0, sizeof(a));
    const dpr_frame_desc &f = d->fr;
    a.F.W = f.W; a.F.H = f.H; a.F.P = f.W * f.H; a.F.spp = f.spp; a.F.max_depth = f.max_depth;
    a.F.ao_k = f.ao_k; a.F.ao_radius = f.ao_radius; a.F.dt = f.dt; a.F.seed = f.seed; a.F.flags = f.flags;
    a.F.pix_rank = d->pix_rank; a.F.pix_nranks = d->pix_nranks;
    for (int c = 0; c < 3; ++c) {
        a.F.l[c] = f.light_dir[c]; a.F.E[c] = f.E[c]; a.F.A[c] = f.A[c]; a.F.B[c] = f.B[c];
        a.F.cE[c] = d->cam.E[c]; a.F.cL[c] = d->cam.L[c]; a.F.cU[c] = d->cam.U[c]; a.F.cV[c] = d->cam.V[c];
    }
    a.F.lens_radius = d->cam.lens_radius;
    a.F.focus_dist = d->cam.focus_dist;
    gen_rect(d, fc, a.F.gen_rect);
    a.F.march_inline_min = march_inline_min(d->nsm);
    a.F.march_g = march_g_env();
    a.R = fc.R;
    a.R.self = d->rank;
    a.W.wnodes = P<WNode>(d->b_wnodes);
    a.W.prmt_hi = 0x4b00u;
    a.W.prims = P<float4>(d->b_prims_w);
    a.W.prims_in = P<float4>(d->b_prims_u);
    a.W.nnodes = d->wnodes_count;
    a.W.nprims = d->nprims;
    a.W.id_base = fc.id_base[d->rank];
    a.W.nbricks = 0;
    a.W.amax = fc.amax;
    for (const BrickDev &B : d->wbricks) {
        if (a.W.nbricks == 0)
            for (int c = 0; c < 3; ++c) {  // global grid domain (all bricks share gdims/origin/spacing)
                a.W.gdom[c] = B.O[c];
                a.W.gdom[3 + c] = B.O[c] + (float)(B.gd[c] - 1) * B.h[c];
            }
        a.W.bricks[a.W.nbricks++] = B;
    }
    a.T.n = (int)fc.part_lo.size();
    a.T.id_lo = P<uint32_t>(d->b_part_lo);
    a.T.albedo = P<float4>(d->b_part_alb);
    int nxt = cur ^ 1;
    a.Q.path_in = P<PathRec>(d->b_path[cur]);
    a.Q.occl_in = P<OcclRec>(d->b_occlq[cur]);
    a.Q.in_count = P<uint32_t>(d->b_in_count);
    a.Q.fused = d->exch;
    for (int r = 0; r < d->nranks; ++r) {
        if (d->exch) {
            a.Q.path_out[r] = d->peer_path[nxt][r];
            a.Q.occl_out[r] = d->peer_occl[nxt][r];
            a.Q.cnt_path[r] = d->peer_tails[r] + 2 * nxt;
            a.Q.cnt_occl[r] = d->peer_tails[r] + 2 * nxt + 1;
        } else {
            a.Q.path_out[r] = r == d->rank ? P<PathRec>(d->b_path[nxt]) : P<PathRec>(d->b_send_path[r]);
            a.Q.occl_out[r] = r == d->rank ? P<OcclRec>(d->b_occlq[nxt]) : P<OcclRec>(d->b_send_occl[r]);
            a.Q.cnt_path[r] = P<uint32_t>(d->b_counts) + r;
            a.Q.cnt_occl[r] = P<uint32_t>(d->b_counts) + d->nranks + r;
        }
    }
    if (d->exch) a.Q.in_count = P<uint32_t>(d->b_tails) + 2 * cur;
    a.Q.path_cap = d->path_cap;
    a.Q.occl_cap = d->occl_cap;
    a.Q.fetch = P<uint32_t>(d->b_fetch);
    a.fb = P<float4>(d->b_fb);
    a.events = (f.flags & DPR_FLAG_DEBUG_DUMPS) ? P<uint32_t>(d->b_events) : nullptr;
    a.occl = (f.flags & DPR_FLAG_DEBUG_DUMPS) ? P<uint32_t>(d->b_occl) : nullptr;
    a.depth = d->want_depth ? P<uint32_t>(d->b_depth) : nullptr;
    a.ctr = P<Counters>(d->b_ctr);
    a.rec = P<StepRec>(d->b_rec);
    a.F.fuse_resolve = fuse_resolve_ok(a);
    return a;
}

// counts[k][src][dst] for the step just finished; also returns the overflow flags.
int gather_counts(std::vector<Dev *> &L, std::vector<int64_t> &C, unsigned &overflow) {
    Dev *d0 = L[0];
    const int N = d0->nranks;
    const size_t W = 2 * N + 1;
    C.assign((size_t)2 * N * N, 0);
    overflow = 0;
    std::vector<const uint32_t *> rows(N, nullptr);
    if (!d0->comm) {
        for (Dev *d : L) {
            // the overflow word lives in the Counters block; mirror it into the counts tail
            CK(cudaMemcpyAsync(P<uint32_t>(d->b_counts) + 2 * N, &P<Counters>(d->b_ctr)->overflow,
                               sizeof(uint32_t), cudaMemcpyDeviceToDevice, d->stream));
            CK(cudaMemcpyAsync(d->h_counts, d->b_counts.p, sizeof(uint32_t) * W, cudaMemcpyDeviceToHost,
                               d->stream));
        }
        for (Dev *d : L) CK(cudaStreamSynchronize(d->stream));
        for (Dev *d : L) rows[d->rank] = d->h_counts;
    } else {
        RET(ensure(d0, d0->b_scratch, sizeof(uint32_t) * W * (N + 1)));
        uint32_t *recv = P<uint32_t>(d0->b_scratch);
        CK(cudaMemcpyAsync(P<uint32_t>(d0->b_counts) + 2 * N, &P<Counters>(d0->b_ctr)->overflow,
                           sizeof(uint32_t), cudaMemcpyDeviceToDevice, d0->stream));
        NK(ncclAllGather(d0->b_counts.p, recv, W, ncclUint32, d0->comm, d0->stream));
        CK(cudaMemcpyAsync(d0->h_counts, recv, sizeof(uint32_t) * W * N, cudaMemcpyDeviceToHost, d0->stream));
        RET(wait_stream(d0));
        for (int r = 0; r < N; ++r) rows[r] = d0->h_counts + (size_t)r * W;
    }
    for (int src = 0; src < N; ++src)
        for (int k = 0; k < 2; ++k)
            for (int dst = 0; dst < N; ++dst) C[((size_t)k * N + src) * N + dst] = rows[src][k * N + dst];
    for (int src = 0; src < N; ++src) overflow |= rows[src][2 * N];
    return DPR_OK;
}

// Fused exchange: every rank learns every rank's next-queue pointers and tails (and, for the
// device-driven loop with peers, their step-barrier mailboxes; in host-collective mode their
// framebuffer / dumps for the a7 reduction).  Loopback: the virtual ranks' buffers directly.
// One rank without a transport: its own buffers.  NCCL / host collectives: cudaIpc handles of
// the cudaMalloc'd buffers are allgathered and opened (NVLink peer mappings, or the same
// device for processes sharing a GPU), re-done when a buffer changes.
constexpr int IPC_NBUF = 8;  // path[0], path[1], occl[0], occl[1], tails, mbox, fb, events|occl
struct IpcMsg {
    cudaIpcMemHandle_t h[IPC_NBUF + 1];
    uint64_t off[IPC_NBUF + 1];  // buffer offset inside the exported allocation
    uint32_t have;               // bit k: buffer k exported
    uint64_t sig;
};

// The driver may place a small cudaMalloc inside a larger allocation; an IPC handle names the
// whole allocation and opens at its base, so the buffer's offset travels with the handle
// (cuMemGetAddressRange, looked up through the runtime: no link-time libcuda dependency).
int alloc_base(void *p, char **base) {
    typedef CUresult (*Fn)(CUdeviceptr *, size_t *, CUdeviceptr);
    static Fn fn = nullptr;
    if (!fn) {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q));
        if (!f || q != cudaDriverEntryPointSuccess) return fail(DPR_ERR_CUDA, "cuMemGetAddressRange not found");
        fn = (Fn)f;
    }
    CUdeviceptr b = 0;
    size_t sz = 0;
    if (fn(&b, &sz, (CUdeviceptr)p) != CUDA_SUCCESS) return fail(DPR_ERR_CUDA, "cuMemGetAddressRange failed");
    *base = (char *)b;
    return DPR_OK;
}

int ensure_mbox(Dev *d) {
    if (d->b_mbox.p) return DPR_OK;
    const size_t mb = sizeof(uint32_t) * 2 * DPR_MAX_RANKS * 4;
    if (d->comm || d->has_hc) RET(ensure_raw(d, d->b_mbox, mb, nullptr));
    else RET(ensure(d, d->b_mbox, mb));
    RET(ensure(d, d->b_seq, sizeof(uint32_t)));
    CK(cudaMemsetAsync(d->b_mbox.p, 0, mb, d->stream));
    CK(cudaMemsetAsync(d->b_seq.p, 0, sizeof(uint32_t), d->stream));
    CK(cudaStreamSynchronize(d->stream));  // zeroed before any peer can store into it
    return DPR_OK;
}

constexpr int FUSED_UNAVAILABLE = 1;  // fused_peers: no peer mappings on some rank (all ranks agree)
int fused_peers(std::vector<Dev *> &L) {
    Dev *d0 = L[0];
    const int N = d0->nranks;
    for (Dev *d : L) RET(ensure_mbox(d));
    if (d0->group || (N == 1 && !d0->comm && !d0->has_hc)) {
        for (Dev *d : L)
            for (int r = 0; r < N; ++r) {
                Dev *q = L[r];
                for (int k = 0; k < 2; ++k) {
                    d->peer_path[k][r] = P<PathRec>(q->b_path[k]);
                    d->peer_occl[k][r] = P<OcclRec>(q->b_occlq[k]);
                }
                d->peer_tails[r] = P<uint32_t>(q->b_tails);
                d->peer_mbox[r] = P<uint32_t>(q->b_mbox);
            }
        return DPR_OK;
    }
    Dev *d = d0;
    void *mine[IPC_NBUF + 1] = {d->b_path[0].p, d->b_path[1].p, d->b_occlq[0].p, d->b_occlq[1].p, d->b_tails.p,
                                d->b_mbox.p, d->has_hc ? d->b_fb.p : nullptr,
                                d->has_hc ? d->b_events.p : nullptr, d->has_hc ? d->b_occl.p : nullptr};
    uint64_t sig = 1469598103934665603ull;
    for (void *p : mine) sig = fnv1a(&p, sizeof(p), sig);
    IpcMsg msg;
    memset(&msg, 0, sizeof(msg));
    for (int k = 0; k <= IPC_NBUF; ++k)
        if (mine[k]) {
            char *base = nullptr;
            RET(alloc_base(mine[k], &base));
            CK(cudaIpcGetMemHandle(&msg.h[k], base));
            msg.off[k] = (uint64_t)((char *)mine[k] - base);
            msg.have |= 1u << k;
        }
    msg.sig = sig;
    // every rank reallocates at the same frames (same frame descriptor); the combined signature
    // keeps the (collective) decision identical on all ranks anyway
    uint64_t all_sig = 0;
    {
        std::vector<const void *> sg = {&sig};
        std::vector<std::vector<char>> so;
        RET(allgather_host(L, sg, sizeof(sig), so));
        for (int r = 0; r < N; ++r) all_sig = fnv1a(so[0].data() + 8 * r, 8, all_sig);
    }
    if (all_sig == d->ipc_sig && d->peer_tails[d->rank]) return DPR_OK;
    std::vector<const void *> sends = {&msg};
    std::vector<std::vector<char>> out;
    RET(allgather_host(L, sends, sizeof(IpcMsg), out));
    for (void *p : d->ipc_opened) cudaIpcCloseMemHandle(p);
    d->ipc_opened.clear();
    const IpcMsg *all = reinterpret_cast<const IpcMsg *>(out[0].data());
    cudaError_t open_err = cudaSuccess;
    for (int r = 0; r < N && open_err == cudaSuccess; ++r) {
        void *ptr[IPC_NBUF + 1];
        void *opened[IPC_NBUF + 1];  // one mapping per distinct allocation of the peer
        for (int k = 0; k <= IPC_NBUF; ++k) {
            ptr[k] = opened[k] = nullptr;
            if (r == d->rank) { ptr[k] = mine[k]; continue; }
            if (!(all[r].have & (1u << k))) continue;
            for (int j = 0; j < k; ++j)
                if (opened[j] && memcmp(&all[r].h[j], &all[r].h[k], sizeof(cudaIpcMemHandle_t)) == 0)
                    opened[k] = opened[j];
            if (!opened[k]) {
                open_err = cudaIpcOpenMemHandle(&opened[k], all[r].h[k], cudaIpcMemLazyEnablePeerAccess);
                if (open_err != cudaSuccess) break;
                d->ipc_opened.push_back(opened[k]);
            }
            ptr[k] = (char *)opened[k] + all[r].off[k];
        }
        if (open_err != cudaSuccess) break;
        d->peer_path[0][r] = (PathRec *)ptr[0];
        d->peer_path[1][r] = (PathRec *)ptr[1];
        d->peer_occl[0][r] = (OcclRec *)ptr[2];
        d->peer_occl[1][r] = (OcclRec *)ptr[3];
        d->peer_tails[r] = (uint32_t *)ptr[4];
        d->peer_mbox[r] = (uint32_t *)ptr[5];
        d->peer_fb[r] = (float4 *)ptr[6];
        d->peer_events[r] = (uint32_t *)ptr[7];
        d->peer_occl_dump[r] = (uint32_t *)ptr[8];
    }
    // every rank learns whether every rank mapped every peer: if one could not (no peer access
    // between some pair of GPUs), all ranks switch to the send/recv exchange together
    {
        (void)cudaGetLastError();
        // test hook: DPR_TEST_FUSED_FAIL=<rank> makes that rank report a failed mapping
        if (const char *e = getenv("DPR_TEST_FUSED_FAIL"))
            if (atoi(e) == d->rank) open_err = cudaErrorPeerAccessUnsupported;
        const int ok = open_err == cudaSuccess ? 1 : 0;
        std::vector<const void *> sg = {&ok};
        std::vector<std::vector<char>> so;
        RET(allgather_host(L, sg, sizeof(int), so));
        bool all_ok = true;
        for (int r = 0; r < N; ++r) all_ok = all_ok && reinterpret_cast<const int *>(so[0].data())[r] != 0;
        if (!all_ok) {
            for (void *p : d->ipc_opened) cudaIpcCloseMemHandle(p);
            d->ipc_opened.clear();
            d->ipc_sig = 0;
            if (d->has_hc)  // the host-collective transport has no other data plane
                return fail(DPR_ERR_CUDA, std::string("fused exchange: peer mapping failed: ") +
                                              cudaGetErrorString(open_err == cudaSuccess ? cudaErrorPeerAccessUnsupported : open_err));
            return FUSED_UNAVAILABLE;
        }
    }
    d->ipc_sig = all_sig;
    return DPR_OK;
}

// Fused step boundary of the HOST loop.  A queue is complete only when every rank that
// appends into it has finished its step, so the boundary exchanges what each rank APPENDED
// in the step, per destination and kind (Counters.app deltas), never a peer's tail: after the
// exchange (the barrier) every rank knows every queue's length.  Loopback: the local ranks'
// counters; NCCL / host collectives: an allgather of {appended[2][N], overflow} per rank.
// in[r] = {path, occl} appended into rank r's next queue; returns the global total.
struct AppMsg {
    int64_t app[2][DPR_MAX_RANKS];
    int64_t ovf;
};

int fused_sync(std::vector<Dev *> &L, std::vector<uint32_t> &in, int64_t &total, unsigned &ovf, double &ms_coll) {
    Dev *d0 = L[0];
    const int N = d0->nranks;
    std::vector<AppMsg> mine(L.size());
    for (size_t i = 0; i < L.size(); ++i) {
        Dev *d = L[i];
        Counters *c = P<Counters>(d->b_ctr);
        CK(cudaMemcpyAsync(d->h_app, c->app, sizeof(c->app), cudaMemcpyDeviceToHost, d->stream));
        CK(cudaMemcpyAsync(d->h_counts, &c->overflow, sizeof(uint32_t), cudaMemcpyDeviceToHost, d->stream));
    }
    for (Dev *d : L) CK(cudaStreamSynchronize(d->stream));  // this rank's appends are final
    for (size_t i = 0; i < L.size(); ++i) {
        Dev *d = L[i];
        memset(&mine[i], 0, sizeof(AppMsg));
        for (int k = 0; k < 2; ++k)
            for (int r = 0; r < N; ++r) {
                const uint64_t now = d->h_app[k * DPR_MAX_RANKS + r];
                mine[i].app[k][r] = (int64_t)(now - d->app_prev[k][r]);
                d->app_prev[k][r] = now;
            }
        mine[i].ovf = d->h_counts[0];
    }
    std::vector<const void *> snd;
    for (auto &m : mine) snd.push_back(&m);
    std::vector<std::vector<char>> o;
    const auto c0 = std::chrono::steady_clock::now();  // the exchange proper: after the local sync
    RET(allgather_host(L, snd, sizeof(AppMsg), o));  // loopback: a copy; else the barrier
    ms_coll += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - c0).count();
    const AppMsg *all = reinterpret_cast<const AppMsg *>(o[0].data());
    in.assign((size_t)2 * N, 0);
    total = 0;
    ovf = 0;
    for (int src = 0; src < N; ++src) {
        ovf |= (unsigned)all[src].ovf;
        for (int k = 0; k < 2; ++k)
            for (int r = 0; r < N; ++r) {
                in[2 * r + k] += (uint32_t)all[src].app[k][r];
                total += all[src].app[k][r];
            }
    }
    return DPR_OK;
}

// The step boundary kernel's arguments for the local ranks L; cur[i] = the parity rank i
// consumed in this step (phase 1) or 1 (phase 0: the batch's primaries are in parity 0).
StepEndArgs make_step_end(std::vector<Dev *> &L, const std::vector<int> &cur, int phase, bool barrier) {
    StepEndArgs e;
    memset(&e, 0, sizeof(e));
    Dev *d0 = L[0];
    e.nlocal = (int)L.size();
    e.nranks = d0->nranks;
    e.self = d0->rank;
    e.phase = phase;
    e.fused = d0->exch;
    for (size_t i = 0; i < L.size(); ++i) {
        Dev *d = L[i];
        if (d->exch) {
            e.next_tails[i] = P<uint32_t>(d->b_tails) + 2 * (cur[i] ^ 1);
            e.cons_tails[i] = P<uint32_t>(d->b_tails) + 2 * cur[i];
        }
        e.fetch[i] = P<uint32_t>(d->b_fetch);
        e.ctr[i] = P<Counters>(d->b_ctr);
        e.rec[i] = P<StepRec>(d->b_rec);
    }
    e.barrier = barrier ? 1 : 0;
    if (barrier) {
        e.mbox_self = P<uint32_t>(d0->b_mbox);
        for (int r = 0; r < d0->nranks; ++r) e.mbox_peer[r] = d0->peer_mbox[r];
        e.seq = P<uint32_t>(d0->b_seq);
        e.timeout_ns = (unsigned long long)(std::min(d0->timeout_s, 60.0) * 1e9);  // one step boundary
    }
    e.more = P<uint32_t>(d0->b_more);
    e.more_slot = -1;
    return e;
}

// One step's kernels of local rank d, input parity cur.  n_path / n_occl: host-known queue
// lengths (host loops: empty kinds are skipped, the march variant chosen on the host), or
// UNKNOWN (device-driven loop: every kernel is launched and decides from the device count).
constexpr uint32_t UNKNOWN = 0xffffffffu;
struct StepTimers {
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> path, occl;
};
int launch_step(Dev *d, const FrameCtx &fc, int cur, uint32_t n_path, uint32_t n_occl, int grid_p, int grid_o,
                StepTimers *tm, int64_t &launches) {
    StepArgs a = make_args(d, fc, cur);
    const int grid_r = d->nsm * 8;
    const bool dev = n_path == UNKNOWN || n_occl == UNKNOWN;
    if (n_path) {
        Nvtx r("trace_path+shade");
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (tm) { e0 = next_event(d); e1 = next_event(d); CK(cudaEventRecord(e0, d->stream)); }
        int nk = 1;
        if (dev) {
            k_launch_trace_path(a, grid_p, d->stream);
            nk += launch_march_variants(a, false, d->stream);
        } else {
            nk = launch_trace_path(a, grid_p, n_path, d->stream);
        }
        if (tm) { CK(cudaEventRecord(e1, d->stream)); tm->path.push_back({e0, e1}); }
        launch_shade_path(a, grid_r, d->stream);
        launches += 1 + nk;
        d->tpl++;
    }
    if (n_occl) {
        Nvtx r("trace_occl+resolve");
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (tm) { e0 = next_event(d); e1 = next_event(d); CK(cudaEventRecord(e0, d->stream)); }
        int nk = 1;
        bool resolve = true;
        if (dev) {
            k_launch_trace_occl(a, grid_o, d->stream);
            nk += launch_march_variants(a, true, d->stream);
        } else {
            nk = launch_trace_occl(a, grid_o, n_occl, d->stream);
            // the host knows the length: skip the resolve launch when the trace resolves itself
            resolve = !(a.F.fuse_resolve && !march_needed(a, n_occl));
        }
        if (tm) { CK(cudaEventRecord(e1, d->stream)); tm->occl.push_back({e0, e1}); }
        if (resolve) launch_resolve_occl(a, grid_r, d->stream);
        launches += (resolve ? 1 : 0) + nk;
        d->tol++;
    }
    CK(cudaGetLastError());
    return DPR_OK;
}

// Signature of everything the step graph bakes in (kernel arguments of both parities, grids,
// the step-boundary arguments): the graph is re-captured when it changes.
uint64_t graph_key(std::vector<Dev *> &L, const FrameCtx &fc, const std::vector<int> &grid_p,
                   const std::vector<int> &grid_o, bool barrier) {
    uint64_t h = 1469598103934665603ull;
    for (size_t i = 0; i < L.size(); ++i)
        for (int c = 0; c < 2; ++c) {
            StepArgs a = make_args(L[i], fc, c);
            h = fnv1a(&a, sizeof(a), h);
        }
    for (int c = 0; c < 2; ++c) {
        std::vector<int> cur(L.size(), c);
        StepEndArgs e = make_step_end(L, cur, 1, barrier);
        h = fnv1a(&e, sizeof(e), h);
    }
    h = fnv1a(grid_p.data(), sizeof(int) * grid_p.size(), h);
    h = fnv1a(grid_o.data(), sizeof(int) * grid_o.size(), h);
    const int b = barrier;
    return fnv1a(&b, sizeof(b), h);
}

// Build the device-driven step loop of one spp batch (the batch's primaries are in parity 0):
//   k_step_end(phase 0) -> k_loop_cond(init) -> WHILE(h_loop) {
//       step(parity 0) -> k_step_end -> IF(h_if) { step(parity 1) -> k_step_end } -> k_loop_cond }
//   step(c) = k_set_ifs (from every local rank's input tails) -> per local rank
//             IF(path queue non-empty) { k_trace_path, k_march_path variants, k_shade_path }
//             IF(occl queue non-empty) { k_trace_occl, k_march_occl variants, k_resolve_occl }
// The loop body is unrolled twice so that every kernel node has fixed arguments (queue
// parities alternate).  Every decision is taken on the device: "another step" by k_step_end
// (local tails; the peers' appended counts through the mailbox barrier), which kernel groups
// run by k_set_ifs (the input tails are final once the boundary is passed), march variants
// and the occlusion trace's own resolve by the kernels from the queue length.
int capture_step(std::vector<Dev *> &L, const FrameCtx &fc, int cur, const std::vector<int> &grid_p,
                 const std::vector<int> &grid_o, cudaGraph_t g, cudaStream_t s, cudaStream_t s2, int64_t &kernels) {
    // IF handles of this step (created on the graph that holds the IF nodes)
    IfArgs ia;
    memset(&ia, 0, sizeof(ia));
    ia.n = (int)L.size();
    ia.count = P<uint32_t>(L[0]->b_more) + 3;
    for (size_t i = 0; i < L.size(); ++i) {
        ia.tails[i] = P<uint32_t>(L[i]->b_tails) + 2 * cur;
        for (int k = 0; k < 2; ++k) CK(cudaGraphConditionalHandleCreate(&ia.h[i][k], g, 0, cudaGraphCondAssignDefault));
        const int mv = march_variants_count(make_args(L[i], fc, cur));
        ia.kernels[i][0] = ia.kernels[i][1] = 2 + mv;  // trace, march variants, shade / resolve
    }
    launch_set_ifs(ia, s);
    kernels++;
    for (size_t i = 0; i < L.size(); ++i)
        for (int k = 0; k < 2; ++k) {
            cudaStreamCaptureStatus st;
            const cudaGraphNode_t *deps = nullptr;
            size_t ndeps = 0;
            cudaGraph_t cg = nullptr;
            CK(cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, &deps, &ndeps));
            cudaGraphNodeParams ip = {};
            ip.type = cudaGraphNodeTypeConditional;
            ip.conditional.handle = ia.h[i][k];
            ip.conditional.type = cudaGraphCondTypeIf;
            ip.conditional.size = 1;
            cudaGraphNode_t node;
            CK(cudaGraphAddNode(&node, cg, deps, ndeps, &ip));
            CK(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
            // the group's kernels, captured into the IF body on the second stream
            cudaGraph_t out = nullptr;
            CK(cudaStreamBeginCaptureToGraph(s2, ip.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                             cudaStreamCaptureModeThreadLocal));
            Dev *d = L[i];
            const cudaStream_t keep = d->stream;
            d->stream = s2;
            int64_t l = 0;
            const int rc = launch_step(d, fc, cur, k == 0 ? UNKNOWN : 0, k == 1 ? UNKNOWN : 0, grid_p[i], grid_o[i],
                                       nullptr, l);
            d->stream = keep;
            CK(cudaStreamEndCapture(s2, &out));
            RET(rc);
            kernels += l;
        }
    return DPR_OK;
}

int build_step_graph(std::vector<Dev *> &L, const FrameCtx &fc, const std::vector<int> &grid_p,
                     const std::vector<int> &grid_o, bool barrier) {
    Dev *d0 = L[0];
    // capture on the library's own non-blocking streams (the caller's may be the legacy default
    // stream, which cannot be captured); the graph is launched on the caller's stream
    if (!d0->gstream) CK(cudaStreamCreateWithFlags(&d0->gstream, cudaStreamNonBlocking));
    if (!d0->gstream2) CK(cudaStreamCreateWithFlags(&d0->gstream2, cudaStreamNonBlocking));
    cudaStream_t s = d0->gstream, s2 = d0->gstream2;
    if (d0->gexec) { cudaGraphExecDestroy(d0->gexec); d0->gexec = nullptr; }
    if (d0->graph) { cudaGraphDestroy(d0->graph); d0->graph = nullptr; }
    int64_t kernels = 0;
    march_grids_init();  // occupancy queries before the capture
    cudaGraph_t g = nullptr;
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h_loop;
    CK(cudaGraphConditionalHandleCreate(&h_loop, g, 0, cudaGraphCondAssignDefault));
    // top level: initial total, then the WHILE node
    CK(cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    {
        StepEndArgs e0 = make_step_end(L, std::vector<int>(L.size(), 1), 0, barrier);
        e0.more_slot = 0;
        launch_step_end(e0, s);
        launch_loop_cond(P<uint32_t>(d0->b_more), h_loop, 1, s);
        kernels += 2;
    }
    cudaStreamCaptureStatus st;
    const cudaGraphNode_t *deps = nullptr;
    size_t ndeps = 0;
    cudaGraph_t cg = nullptr;
    CK(cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, &deps, &ndeps));
    cudaGraphNodeParams wp = {};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = h_loop;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t wnode;
    CK(cudaGraphAddNode(&wnode, cg, deps, ndeps, &wp));
    cudaGraph_t body = wp.conditional.phGraph_out[0];
    CK(cudaStreamUpdateCaptureDependencies(s, &wnode, 1, cudaStreamSetCaptureDependencies));
    cudaGraph_t gout = nullptr;
    CK(cudaStreamEndCapture(s, &gout));
    // WHILE body: step A (parity 0) + boundary, IF node, loop condition
    cudaGraphConditionalHandle h_if;
    CK(cudaGraphConditionalHandleCreate(&h_if, body, 0, cudaGraphCondAssignDefault));
    CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    int rc = capture_step(L, fc, 0, grid_p, grid_o, body, s, s2, kernels);
    if (rc == DPR_OK) {
        StepEndArgs e = make_step_end(L, std::vector<int>(L.size(), 0), 1, barrier);
        e.more_slot = 0;
        e.set_if = 1;
        e.h_if = h_if;
        launch_step_end(e, s);
        kernels++;
        CK(cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, &deps, &ndeps));
    }
    cudaGraphNodeParams ip = {};
    cudaGraphNode_t inode;
    if (rc == DPR_OK) {
        ip.type = cudaGraphNodeTypeConditional;
        ip.conditional.handle = h_if;
        ip.conditional.type = cudaGraphCondTypeIf;
        ip.conditional.size = 1;
        CK(cudaGraphAddNode(&inode, cg, deps, ndeps, &ip));
        CK(cudaStreamUpdateCaptureDependencies(s, &inode, 1, cudaStreamSetCaptureDependencies));
        launch_loop_cond(P<uint32_t>(d0->b_more), h_loop, 0, s);
        kernels++;
    }
    CK(cudaStreamEndCapture(s, &gout));
    RET(rc);
    // IF body: step B (parity 1) + boundary
    cudaGraph_t ibody = ip.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(s, ibody, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    rc = capture_step(L, fc, 1, grid_p, grid_o, ibody, s, s2, kernels);
    if (rc == DPR_OK) {
        StepEndArgs e = make_step_end(L, std::vector<int>(L.size(), 1), 1, barrier);
        e.more_slot = 1;
        launch_step_end(e, s);
        kernels++;
    }
    CK(cudaStreamEndCapture(s, &gout));
    RET(rc);
    CK(cudaGraphInstantiate(&d0->gexec, g, 0));
    d0->graph = g;
    d0->graph_kernels = kernels;
    d0->graph_builds++;
    for (Dev *d : L) { d->tpl = 0; d->tol = 0; }  // launch_step counted the captured launches
    return DPR_OK;
}

// a7 in host-collective mode: rank 0 sums the peers' framebuffers (and dumps) through the IPC
// mappings after a barrier; a second barrier keeps the peers from clearing them too early.
int hc_reduce(Dev *d, int64_t P_, size_t nd, bool dumps, int64_t &launches) {
    RET(hc_barrier(d));
    if (d->rank == 0)
        for (int r = 1; r < d->nranks; ++r) {
            launch_fb_accumulate(P<float4>(d->b_fb), d->peer_fb[r], P_, d->stream);
            launches++;
            if (dumps) {
                launch_u32_accumulate(P<uint32_t>(d->b_events), d->peer_events[r], nd, d->stream);
                launch_u32_accumulate(P<uint32_t>(d->b_occl), d->peer_occl_dump[r], nd, d->stream);
                launches += 2;
            }
        }
    return hc_barrier(d);
}

int render_group(std::vector<Dev *> &L) {
    Nvtx nv_frame("dpr_render_frame");
    Dev *d0 = L[0];
    const int N = d0->nranks;
    for (Dev *d : L) {
        if (d->broken) return fail(DPR_ERR_NCCL, "communicator was aborted; release the device");
        if (!d->world_ready) return fail(DPR_ERR_STATE, "dpr_commit_world has not been called");
        if (!d->cam_set || !d->fr_set) return fail(DPR_ERR_STATE, "camera and frame must be set before rendering");
        d->ev_used = 0;
        d->frame_done = 0;
        d->dumps_valid = false;
    }
    const dpr_frame_desc &f = d0->fr;
    for (Dev *d : L) { d->frame_exch_bytes = 0; d->tpl = 0; d->tol = 0; }
    cudaEvent_t ev_f0 = next_event(d0), ev_f1;
    CK(cudaEventRecord(ev_f0, d0->stream));
    FrameCtx fc;
    memset(&fc.R, 0, sizeof(fc.R));
    {
        Nvtx r("frame_setup");
        RET(frame_setup(L, fc));
        for (Dev *d : L) RET(frame_buffers(d, fc));
    }
    bool fused = d0->exch != 0;
    if (fused) {
        const int rc = fused_peers(L);
        if (rc == FUSED_UNAVAILABLE) {
            // collective fallback (decided identically on every rank): NCCL send/recv from now on
            for (Dev *d : L) d->exch = 0;
            for (Dev *d : L) RET(frame_buffers(d, fc));
            fused = false;
        } else {
            RET(rc);
        }
    }
    // device-driven step loop: fused exchange, not the host-collective transport
    const bool dev_loop = fused && d0->step_loop && !d0->has_hc;
    const bool barrier = dev_loop && !d0->group && (N > 1 || d0->comm);
    const int64_t P_ = (int64_t)f.W * f.H;
    const int nb = (f.spp + f.spp_batch - 1) / f.spp_batch;
    int64_t launches = 0;
    std::vector<int> cur(L.size(), 0);
    std::vector<int> grid_p(L.size()), grid_o(L.size());
    for (size_t i = 0; i < L.size(); ++i) {
        grid_p[i] = std::max(1, trace_path_occupancy(TRACE_BLOCK)) * L[i]->nsm;
        grid_o[i] = std::max(1, trace_occl_occupancy(TRACE_BLOCK)) * L[i]->nsm;
    }
    if (dev_loop) {
        const uint64_t key = graph_key(L, fc, grid_p, grid_o, barrier);
        if (!d0->gexec || key != d0->gkey) {
            Nvtx r("build_step_graph");
            RET(build_step_graph(L, fc, grid_p, grid_o, barrier));
            d0->gkey = key;
        }
    }
    StepTimers tm;
    double ms_sync_host = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> t_exch, t_gen;
    std::vector<int64_t> C;
    for (int b = 0; b < nb; ++b) {
        Nvtx nv_batch("spp_batch");
        int s0 = b * f.spp_batch, ns = std::min(f.spp_batch, f.spp - s0);
        for (size_t i = 0; i < L.size(); ++i) {
            Dev *d = L[i];
            // fused: every batch starts with its primaries in parity 0 (all tails are 0 here)
            if (fused) cur[i] = 1;
            else CK(cudaMemsetAsync(d->b_counts.p, 0, sizeof(uint32_t) * (2 * N + 1), d->stream));
            StepArgs a = make_args(d, fc, cur[i]);
            cudaEvent_t e0 = next_event(d), e1 = next_event(d);
            CK(cudaEventRecord(e0, d->stream));
            launch_gen_primary(a, s0, ns, d->spw, d->stream);
            CK(cudaEventRecord(e1, d->stream));
            if (i == 0) t_gen.push_back({e0, e1});
            launches++;
            CK(cudaGetLastError());
        }
        if (dev_loop) {
            // the whole lock-step loop of the batch on the device: no host round trip per step
            Nvtx r("step_loop_graph");
            CK(cudaGraphLaunch(d0->gexec, d0->stream));
            continue;
        }
        {   // host loops: the boundary kernel before the first step (timestamps, fetch heads)
            StepEndArgs e = make_step_end(L, std::vector<int>(L.size(), 1), 0, false);
            launch_step_end(e, d0->stream);
            launches++;
        }
        while (fused) {
            Nvtx nv_step("step");
            // step boundary: every rank's next-queue counts (the allgather is the barrier)
            std::vector<uint32_t> in;
            int64_t total = 0;
            unsigned ovf = 0;
            RET(fused_sync(L, in, total, ovf, ms_sync_host));
            if (getenv("DPR_DEBUG_STEPS")) {
                fprintf(stderr, "[dpr rank %d] step boundary:", d0->rank);
                for (int r = 0; r < N; ++r) fprintf(stderr, " r%d{%u,%u}", r, in[2 * r], in[2 * r + 1]);
                fprintf(stderr, " ovf %u\n", ovf);
            }
            if (ovf & 1u) return fail(DPR_ERR_QUEUE_OVERFLOW, "ray queue capacity exceeded; lower spp_batch");
            if (ovf & 2u) return fail(DPR_ERR_STATE, "BVH traversal stack overflow");
            if (ovf & 4u) return fail(DPR_ERR_STATE, "device bounds check failed (DPR_CHECKS build)");
            if (total == 0) break;
            for (size_t i = 0; i < L.size(); ++i) {
                Dev *d = L[i];
                cur[i] ^= 1;
                const uint32_t n_path = in[2 * d->rank], n_occl = in[2 * d->rank + 1];
                RET(launch_step(d, fc, cur[i], n_path, n_occl, grid_p[i], grid_o[i], i == 0 ? &tm : nullptr,
                                launches));
            }
            // boundary: per-step snapshot, consumed tails (append targets of the step after next)
            // and fetch heads reset
            StepEndArgs e = make_step_end(L, cur, 1, false);
            launch_step_end(e, d0->stream);
            launches++;
        }
        while (!fused) {
            Nvtx nv_step("step");
            unsigned ovf = 0;
            RET(gather_counts(L, C, ovf));
            if (ovf & 1u) return fail(DPR_ERR_QUEUE_OVERFLOW, "ray queue capacity exceeded; lower spp_batch");
            if (ovf & 2u) return fail(DPR_ERR_STATE, "BVH traversal stack overflow");
            if (ovf & 4u) return fail(DPR_ERR_STATE, "device bounds check failed (DPR_CHECKS build)");
            int64_t total = 0;
            for (int64_t v : C) total += v;
            if (total == 0) break;
            // exchange: records for other ranks -> their next input queues
            Nvtx nv_x("exchange");
            cudaEvent_t ex0 = next_event(d0), ex1 = next_event(d0);
            CK(cudaEventRecord(ex0, d0->stream));
            std::vector<std::vector<int64_t>> offs(L.size() * 2);
            for (size_t i = 0; i < L.size(); ++i) {
                Dev *d = L[i];
                for (int k = 0; k < 2; ++k) {
                    std::vector<int64_t> off(N);
                    int64_t tin = 0, gt = 0;
                    int64_t cap = k == 0 ? d->path_cap : d->occl_cap;
                    int rc = dpr_exchange_plan(N, d->rank, C.data() + (size_t)k * N * N, cap, off.data(), &tin, &gt);
                    if (rc != DPR_OK) return fail(rc, "ray queue capacity exceeded on receive; lower spp_batch");
                    d->h_in[k] = (uint32_t)tin;
                    offs[2 * i + k] = off;
                }
            }
            if (N > 1 || d0->comm) {
                const size_t rs[2] = {sizeof(PathRec), sizeof(OcclRec)};
                if (d0->group) {
                    for (size_t i = 0; i < L.size(); ++i) {
                        Dev *dst = L[i];
                        int nxt = cur[i] ^ 1;
                        for (int k = 0; k < 2; ++k) {
                            char *base = k == 0 ? P<char>(dst->b_path[nxt]) : P<char>(dst->b_occlq[nxt]);
                            for (int src = 0; src < N; ++src) {
                                if (src == dst->rank) continue;
                                int64_t cnt = C[((size_t)k * N + src) * N + dst->rank];
                                if (!cnt) continue;
                                Dev *sd = L[src];
                                const void *from = k == 0 ? sd->b_send_path[dst->rank].p : sd->b_send_occl[dst->rank].p;
                                CK(cudaMemcpyAsync(base + offs[2 * i + k][src] * rs[k], from, cnt * rs[k],
                                                   cudaMemcpyDeviceToDevice, dst->stream));
                                sd->frame_exch_bytes += cnt * rs[k];
                            }
                        }
                    }
                } else {
                    Dev *d = d0;
                    int nxt = cur[0] ^ 1;
                    NK(ncclGroupStart());
                    for (int k = 0; k < 2; ++k) {
                        char *base = k == 0 ? P<char>(d->b_path[nxt]) : P<char>(d->b_occlq[nxt]);
                        for (int peer = 0; peer < N; ++peer) {
                            if (peer == d->rank) continue;
                            int64_t sc = C[((size_t)k * N + d->rank) * N + peer];
                            int64_t rc = C[((size_t)k * N + peer) * N + d->rank];
                            if (sc) {
                                const void *from = k == 0 ? d->b_send_path[peer].p : d->b_send_occl[peer].p;
                                NK(ncclSend(from, sc * rs[k], ncclUint8, peer, d->comm, d->stream));
                                d->frame_exch_bytes += sc * rs[k];
                            }
                            if (rc) NK(ncclRecv(base + offs[k][peer] * rs[k], rc * rs[k], ncclUint8, peer, d->comm, d->stream));
                        }
                    }
                    NK(ncclGroupEnd());
                }
            }
            CK(cudaEventRecord(ex1, d0->stream));
            t_exch.push_back({ex0, ex1});
            // next step: swap queues, trace
            for (size_t i = 0; i < L.size(); ++i) {
                Dev *d = L[i];
                cur[i] ^= 1;
                CK(cudaMemcpyAsync(d->b_in_count.p, d->h_in, sizeof(uint32_t) * 2, cudaMemcpyHostToDevice, d->stream));
                CK(cudaMemsetAsync(d->b_counts.p, 0, sizeof(uint32_t) * (2 * N + 1), d->stream));
                RET(launch_step(d, fc, cur[i], d->h_in[0], d->h_in[1], grid_p[i], grid_o[i], i == 0 ? &tm : nullptr,
                                launches));
            }
            StepEndArgs e = make_step_end(L, cur, 1, false);
            launch_step_end(e, d0->stream);
            launches++;
        }
    }
    // a7: framebuffer (+ dumps) reduction to rank 0, normalisation by spp
    Nvtx nv_red("reduce");
    cudaEvent_t r0 = next_event(d0), r1 = next_event(d0);
    CK(cudaEventRecord(r0, d0->stream));
    const size_t nd = (size_t)f.spp * f.max_depth * P_;
    const bool dumps = f.flags & DPR_FLAG_DEBUG_DUMPS;
    if (N > 1 && d0->group) {
        Dev *root = L[0];
        for (int r = 1; r < N; ++r) {
            launch_fb_accumulate(P<float4>(root->b_fb), P<float4>(L[r]->b_fb), P_, root->stream);
            launches++;
            if (dumps) {
                launch_u32_accumulate(P<uint32_t>(root->b_events), P<uint32_t>(L[r]->b_events), nd, root->stream);
                launch_u32_accumulate(P<uint32_t>(root->b_occl), P<uint32_t>(L[r]->b_occl), nd, root->stream);
                launches += 2;
            }
        }
    } else if (d0->has_hc) {
        RET(hc_reduce(d0, P_, nd, dumps, launches));
    } else if (d0->comm) {
        Dev *d = d0;
        NK(ncclGroupStart());
        NK(ncclReduce(d->b_fb.p, d->b_fb.p, 4 * P_, ncclFloat, ncclSum, 0, d->comm, d->stream));
        if (dumps) {
            NK(ncclReduce(d->b_events.p, d->b_events.p, nd, ncclUint32, ncclSum, 0, d->comm, d->stream));
            NK(ncclReduce(d->b_occl.p, d->b_occl.p, nd, ncclUint32, ncclSum, 0, d->comm, d->stream));
        }
        NK(ncclGroupEnd());
    }
    for (Dev *d : L) {
        if (d->rank != 0) continue;
        launch_fb_normalize(P<float4>(d->b_fb_out), P<float4>(d->b_fb), P_, (float)f.spp, d->stream);
        launches++;
        d->dumps_valid = dumps;
    }
    CK(cudaEventRecord(r1, d0->stream));
    ev_f1 = next_event(d0);
    CK(cudaEventRecord(ev_f1, d0->stream));
    RET(wait_stream(d0));
    CK(cudaGetLastError());
    // stats
    auto sum_ms = [](std::vector<std::pair<cudaEvent_t, cudaEvent_t>> &v) {
        double t = 0;
        for (auto &e : v) { float ms = 0; cudaEventElapsedTime(&ms, e.first, e.second); t += ms; }
        return t;
    };
    float fms = 0;
    cudaEventElapsedTime(&fms, ev_f0, ev_f1);
    std::vector<StatsMsg> msgs(L.size());
    std::vector<Counters> ctr(L.size());
    std::vector<StepRec> rec(L.size());
    for (size_t i = 0; i < L.size(); ++i) {
        CK(cudaMemcpy(&ctr[i], L[i]->b_ctr.p, sizeof(Counters), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&rec[i], L[i]->b_rec.p, sizeof(StepRec), cudaMemcpyDeviceToHost));
    }
    for (size_t i = 0; i < L.size(); ++i) {
        if (rec[i].err & 0x100u) return abort_comm(L[i], "step barrier timed out (a peer did not reach the step boundary)");
        if (rec[i].err & 1u) return fail(DPR_ERR_QUEUE_OVERFLOW, "ray queue capacity exceeded; lower spp_batch");
        if (rec[i].err & 2u) return fail(DPR_ERR_STATE, "BVH traversal stack overflow");
        if (rec[i].err & 4u) return fail(DPR_ERR_STATE, "device bounds check failed (DPR_CHECKS build)");
    }
    const int64_t steps = rec[0].step;
    const int nrec = (int)std::min<int64_t>(steps, MAX_STEP_REC);
    // trace kernels: first-CTA-start .. last-CTA-end globaltimer spans of the launches that
    // traced rays (the device loop also launches them on empty queues; they exit at once)
    double kt_ms[2] = {0, 0}, sync_ms = 0;
    int64_t kt_n[2] = {0, 0};
    for (int k = 0; k < nrec; ++k) {
        for (int q = 0; q < 2; ++q) {
            const unsigned long long a = ~rec[0].kt[k][q][0], e = rec[0].kt[k][q][1];
            const bool work = rec[0].rin[k][q] > (k ? rec[0].rin[k - 1][q] : 0ull);
            if (work && rec[0].kt[k][q][0] && e >= a) { kt_ms[q] += (double)(e - a) * 1e-6; kt_n[q]++; }
        }
        sync_ms += rec[0].t_sync[k] * 1e-6;
    }
    for (size_t i = 0; i < L.size(); ++i) {
        StatsMsg &m = msgs[i];
        memset(&m, 0, sizeof(m));
        for (int k = 0; k < 3; ++k) {
            m.V[k] = (int64_t)ctr[i].V[k];
            m.gen[k] = (int64_t)ctr[i].gen[k];
            for (int r = 0; r < N; ++r) m.S[k][r] = (int64_t)ctr[i].S[k][r];
        }
        m.ms_frame = fms;
        m.nsteps = nrec;
        for (int k = 0; k < nrec; ++k) {
            for (int q = 0; q < 3; ++q) {
                for (int r = 0; r < N; ++r) m.stepS[k][q][r] = (int64_t)rec[i].S[k][q][r];
                m.stepV[k][q] = (int64_t)rec[i].V[k][q];
            }
            m.step_ms[k] = (double)(rec[i].t_end[k] - rec[i].t_begin[k]) * 1e-6;
            m.step_sync_ms[k] = rec[i].t_sync[k] * 1e-6;
        }
    }
    std::vector<const void *> sends;
    for (auto &m : msgs) sends.push_back(&m);
    std::vector<std::vector<char>> out;
    RET(allgather_host(L, sends, sizeof(StatsMsg), out));
    const StatsMsg *all = reinterpret_cast<const StatsMsg *>(out[0].data());
    for (size_t i = 0; i < L.size(); ++i) {
        Dev *d = L[i];
        dpr_stats &st = d->stats;
        memset(&st, 0, sizeof(st));
        st.nranks = N;
        st.rank = d->rank;
        st.kernel_launches_local = d->build_launches + (i == 0 ? launches : 0);
        st.exchanged_bytes_local = d->frame_exch_bytes;
        if (fused) {  // records written into peers' queues, from this rank's routing row
            int64_t eb = 0;
            for (int q = 0; q < N; ++q)
                if (q != d->rank)
                    eb += all[d->rank].S[0][q] * (int64_t)sizeof(PathRec) +
                          (all[d->rank].S[1][q] + all[d->rank].S[2][q]) * (int64_t)sizeof(OcclRec);
            st.exchanged_bytes_local = eb;
        }
        st.trace_path_launches = d->tpl;
        st.trace_occl_launches = d->tol;
        st.steps = steps;
        double mx = 0;
        for (int r = 0; r < N; ++r) {
            for (int k = 0; k < 3; ++k) {
                st.V[k][r] = all[r].V[k];
                st.rays[k] += all[r].gen[k];
                for (int q = 0; q < N; ++q) st.S[k][r][q] = all[r].S[k][q];
            }
            mx = std::max(mx, all[r].ms_frame);
        }
        // per-step matrices: deltas of the cumulative snapshots, every rank's row
        d->nsteps_rec = nrec;
        d->step_S.assign((size_t)nrec * 3 * N * N, 0);
        d->step_V.assign((size_t)nrec * 3 * N, 0);
        d->step_ms.assign(nrec, 0.0);
        d->step_sync_ms.assign(nrec, 0.0);
        for (int k = 0; k < nrec; ++k)
            for (int r = 0; r < N; ++r) {
                const StatsMsg &m = all[r];
                for (int q = 0; q < 3; ++q) {
                    for (int c = 0; c < N; ++c)
                        d->step_S[(((size_t)k * 3 + q) * N + r) * N + c] =
                            m.stepS[k][q][c] - (k ? m.stepS[k - 1][q][c] : 0);
                    d->step_V[((size_t)k * 3 + q) * N + r] = m.stepV[k][q] - (k ? m.stepV[k - 1][q] : 0);
                }
                d->step_ms[k] = std::max(d->step_ms[k], m.step_ms[k]);
                d->step_sync_ms[k] = std::max(d->step_sync_ms[k], m.step_sync_ms[k]);
            }
        const KernelCounters &a = ctr[i].kc[0], &o = ctr[i].kc[1];
        st.node_visits_local = (int64_t)(a.nodes + o.nodes);
        st.tri_tests_local = (int64_t)(a.tris + o.tris);
        st.sphere_tests_local = (int64_t)(a.sphs + o.sphs);
        st.vol_samples_local = (int64_t)(a.vols + o.vols);
        st.records_in_local = (int64_t)(a.rin + o.rin);
        st.records_out_local = (int64_t)(a.rout_path + a.rout_occl + o.rout_occl);
        // algorithmic bytes: records read + written, node fetches
        // (80 B wide nodes), triangle tests (48 B), sphere tests (16 B), volume samples (8 voxels, 32 B)
        st.path_bytes_alg_local = (int64_t)(a.rin * 64 + a.rout_path * 64 + a.rout_occl * 48 +
                                            a.nodes * 80 + a.tris * 48 + a.sphs * 16 + a.vols * 32);
        st.occl_bytes_alg_local = (int64_t)(o.rin * 48 + o.rout_occl * 48 + o.nodes * 80 +
                                            o.tris * 48 + o.sphs * 16 + o.vols * 32);
        for (int k = 0; k < 2; ++k) {
            const KernelCounters &kc = ctr[i].kc[k];
            st.kernel_rays_local[k] = (int64_t)kc.rin;
            st.kernel_nodes_local[k] = (int64_t)kc.nodes;
            st.kernel_tris_local[k] = (int64_t)kc.tris;
            st.kernel_sphs_local[k] = (int64_t)kc.sphs;
            st.kernel_vols_local[k] = (int64_t)kc.vols;
        }
        st.bvh_nodes_local = d->wnodes_count;
        st.bvh_levels_local = d->bvh_levels;
        st.ms_frame = fms;
        st.ms_frame_max = mx;
        st.step_loop_device = dev_loop ? 1 : 0;
        if (i == 0) {
            st.ms_kernel_span[0] = kt_ms[0];
            st.ms_kernel_span[1] = kt_ms[1];
        }
        st.graph_builds = d0->graph_builds;
        if (d->comm) {
            int cn = 0;
            if (ncclCommCount(d->comm, &cn) == ncclSuccess) st.comm_nranks = cn;
        }
        if (i == 0) {
            st.ms_gen = sum_ms(t_gen);
            if (dev_loop) {
                st.ms_trace_path = kt_ms[0];
                st.ms_trace_occl = kt_ms[1];
                st.ms_exchange = sync_ms;  // fused: appends are inside the kernels; the barrier
                st.trace_path_launches = kt_n[0];  // launches that traced rays
                st.trace_occl_launches = kt_n[1];
                // graph: per batch 2 (initial boundary + condition); per step k_set_ifs, the
                // kernel groups that ran and the boundary; per WHILE iteration one condition
                // kernel (iterations and group kernels counted on the device)
                uint32_t cnt[2] = {0, 0};
                CK(cudaMemcpy(cnt, P<uint32_t>(d0->b_more) + 2, sizeof(cnt), cudaMemcpyDeviceToHost));
                st.kernel_launches_local = d->build_launches + launches + (int64_t)nb * 2 + steps * 2 + cnt[0] + cnt[1];
            } else {
                st.ms_trace_path = sum_ms(tm.path);
                st.ms_trace_occl = sum_ms(tm.occl);
                // send-recv: grouped send/recv (CUDA events); fused host loop: the host-side
                // boundary collective (after the local stream is idle), wall clock
                st.ms_exchange = fused ? ms_sync_host : sum_ms(t_exch);
            }
            float rms = 0;
            cudaEventElapsedTime(&rms, r0, r1);
            st.ms_reduce = rms;
        }
        d->frame_done = 1;
        d->mapped_w = d->rank == 0 ? f.W : 0;
        d->mapped_h = d->rank == 0 ? f.H : 0;
        d->frame_out = d->rank == 0 ? P<float>(d->b_fb_out) : nullptr;
        d->replicated_frame = false;
    }
    return DPR_OK;
}

int check_part(const dpr_part_desc *p) {
    if (!p) return fail(DPR_ERR_INVALID_ARG, "null part");
    if (p->memory != DPR_MEMORY_HOST && p->memory != DPR_MEMORY_DEVICE && p->memory != DPR_MEMORY_HOST_ASYNC)
        return fail(DPR_ERR_INVALID_ARG, "bad memory kind");
    switch (p->kind) {
    case DPR_PART_TRIANGLES:
        if (p->n_tris < 0 || p->n_verts < 0 || (p->n_tris > 0 && (!p->verts || !p->idx)))
            return fail(DPR_ERR_INVALID_ARG, "triangle part: bad arrays");
        break;
    case DPR_PART_SPHERES:
        if (p->n_spheres < 0 || (p->n_spheres > 0 && !p->spheres)) return fail(DPR_ERR_INVALID_ARG, "sphere part: bad arrays");
        break;
    case DPR_PART_BRICK:
        if (!p->voxels || !p->tf) return fail(DPR_ERR_INVALID_ARG, "brick part: null voxels/tf");
        for (int c = 0; c < 3; ++c)
            if (p->cell_lo[c] < 0 || p->cell_hi[c] <= p->cell_lo[c] || p->cell_hi[c] > p->gdims[c] - 1 || !(p->spacing[c] > 0))
                return fail(DPR_ERR_INVALID_ARG, "brick part: bad cell range / spacing");
        if (!(p->tf_hi > p->tf_lo)) return fail(DPR_ERR_INVALID_ARG, "brick part: tf_hi must exceed tf_lo");
        if ((int64_t)(p->cell_hi[1] - p->cell_lo[1] + 1) * (p->cell_hi[2] - p->cell_lo[2] + 1) >= ((int64_t)1 << 31))
            return fail(DPR_ERR_INVALID_ARG, "brick part: more than 2^31 - 1 voxel rows (y * z extent)");
        break;
    default:
        return fail(DPR_ERR_INVALID_ARG, "bad part kind");
    }
    return DPR_OK;
}

// Bricks (read by the render kernels) and device sources: stream-ordered on the library
// stream; host sources are complete when this returns.
int copy_in(Dev *d, Buf &b, const void *src, size_t bytes, int memory) {
    RET(ensure(d, b, bytes));
    if (!bytes) return DPR_OK;
    CK(cudaMemcpyAsync(b.p, src, bytes, memory == DPR_MEMORY_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                       d->stream));
    if (memory != DPR_MEMORY_DEVICE) CK(cudaStreamSynchronize(d->stream));
    return DPR_OK;
}

// Triangle / sphere arrays (read only by the build): a recycled buffer (its last reader, a
// build, has completed: dpr_commit_world waits for it) or a new one; host sources are copied
// on the side copy stream, which overlaps a render still running on the library stream.
int copy_in_geom(Dev *d, Buf &b, const void *src, size_t bytes, int memory) {
    if (!bytes) return DPR_OK;
    int best = -1;
    for (size_t i = 0; i < d->part_pool.size(); ++i)
        if (d->part_pool[i].bytes >= bytes && (best < 0 || d->part_pool[i].bytes < d->part_pool[best].bytes))
            best = (int)i;
    bool fresh = best < 0;
    if (!fresh) {
        b = d->part_pool[best];
        d->part_pool.erase(d->part_pool.begin() + best);
    } else {
        RET(ensure(d, b, bytes));
    }
    if (memory == DPR_MEMORY_DEVICE) {
        if (d->copy_pending) CK(cudaStreamWaitEvent(d->stream, d->copy_ev, 0));  // recycled buffer
        CK(cudaMemcpyAsync(b.p, src, bytes, cudaMemcpyDeviceToDevice, d->stream));
        return DPR_OK;
    }
    if (fresh) {  // a new allocation is stream-ordered on the library stream: order after it
        CK(cudaEventRecord(d->order_ev, d->stream));
        CK(cudaStreamWaitEvent(d->cstream, d->order_ev, 0));
    }
    CK(cudaMemcpyAsync(b.p, src, bytes, cudaMemcpyHostToDevice, d->cstream));
    CK(cudaEventRecord(d->copy_ev, d->cstream));
    d->copy_pending = true;
    if (memory == DPR_MEMORY_HOST) CK(cudaEventSynchronize(d->copy_ev));
    return DPR_OK;
}

int init_dev(Dev *d, int rank, int nranks, int cuda_device, void *stream, const dpr_allocator *alloc) {
    d->rank = rank;
    d->nranks = nranks;
    d->cuda_dev = cuda_device;
    d->stream = (cudaStream_t)stream;
    if (alloc && alloc->alloc && alloc->free) { d->alloc = *alloc; d->has_alloc = true; }
    CK(cudaSetDevice(cuda_device));
    CK(cudaDeviceGetAttribute(&d->nsm, cudaDevAttrMultiProcessorCount, cuda_device));
    CK(cudaStreamCreateWithFlags(&d->cstream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&d->copy_ev, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&d->order_ev, cudaEventDisableTiming));
    for (int c = 0; c < 3; ++c) { d->box[c] = INFINITY; d->box[3 + c] = -INFINITY; }
    if (const char *e = getenv("DPR_SPW")) d->spw = std::max(1, atoi(e));
    if (const char *e = getenv("DPR_BUILDER"))
        d->builder = strcmp(e, "ploc") == 0 ? 0 : strcmp(e, "karras") == 0 ? 2 : 1;
    if (const char *e = getenv("DPR_EXCHANGE")) d->exch = strcmp(e, "sendrecv") == 0 ? 0 : 1;
    if (const char *e = getenv("DPR_STEP_LOOP")) d->step_loop = strcmp(e, "host") == 0 ? 0 : 1;
    if (const char *e = getenv("DPR_TIMEOUT_S")) d->timeout_s = std::max(0.001, atof(e));
    return DPR_OK;
}

void release_local_view(Dev *d);

void release_bufs(Dev *d) {
    release_local_view(d);
    Buf *cb[] = {&d->b_depth, &d->b_frag_rgba, &d->b_frag_z, &d->b_comp, &d->b_comp_out};
    for (Buf *b : cb) dfree(d, *b);
    for (auto &p : d->parts) { dfree(d, p.verts); dfree(d, p.idx); dfree(d, p.spheres); dfree(d, p.vox); dfree(d, p.tf); dfree(d, p.mc); }
    d->parts.clear();
    for (auto &b : d->retired) dfree(d, b);
    d->retired.clear();
    Buf *bs[] = {&d->b_prims_u, &d->b_blo, &d->b_bhi, &d->b_keys[0], &d->b_keys[1], &d->b_vals[0],
                 &d->b_vals[1], &d->b_tile, &d->b_left, &d->b_right, &d->b_parent, &d->b_rlo, &d->b_rhi,
                 &d->b_nlo, &d->b_nhi, &d->b_arrive, &d->b_prims, &d->b_slo, &d->b_shi,
                 &d->b_bounds, &d->b_chunks, &d->b_hist, &d->b_wnodes, &d->b_prims_w, &d->b_items[0], &d->b_items[1], &d->b_wcnt, &d->b_wperm, &d->b_witems[0], &d->b_witems[1], &d->b_size, &d->b_bn, &d->b_fb, &d->b_fb_out, &d->b_events, &d->b_occl, &d->b_ctr,
                 &d->b_counts, &d->b_in_count, &d->b_fetch, &d->b_part_lo, &d->b_part_alb, &d->b_scratch,
                 &d->b_path[0], &d->b_path[1], &d->b_occlq[0], &d->b_occlq[1]};
    for (Buf *b : bs) dfree(d, *b);
    for (int r = 0; r < DPR_MAX_RANKS; ++r) { dfree(d, d->b_send_path[r]); dfree(d, d->b_send_occl[r]); }
    for (void *p : d->ipc_opened) cudaIpcCloseMemHandle(p);
    d->ipc_opened.clear();
    dfree(d, d->b_tails);
    if (d->h_counts) cudaFreeHost(d->h_counts);
    if (d->h_in) cudaFreeHost(d->h_in);
    if (d->h_app) cudaFreeHost(d->h_app);
    d->h_app = nullptr;
    d->h_counts = nullptr;
    d->h_in = nullptr;
    for (auto e : d->ev_pool) cudaEventDestroy(e);
    d->ev_pool.clear();
    if (d->gexec) cudaGraphExecDestroy(d->gexec);
    if (d->graph) cudaGraphDestroy(d->graph);
    if (d->gstream) cudaStreamDestroy(d->gstream);
    if (d->gstream2) cudaStreamDestroy(d->gstream2);
    d->gstream2 = nullptr;
    d->gexec = nullptr;
    d->graph = nullptr;
    d->gstream = nullptr;
    Buf *xs[] = {&d->b_rec, &d->b_more, &d->b_mbox, &d->b_seq};
    for (Buf *b : xs) dfree(d, *b);
}

// ---------------------------------------------------------------------------------------
// Compositing contrast device.
// ---------------------------------------------------------------------------------------
// A single-rank view of d's world (shares the world buffers, owns its frame buffers).
Dev *local_view(Dev *d, bool replicated = false) {
    if (!d->lv) {
        Dev *v = new Dev();
        v->rank = 0; v->nranks = 1; v->cuda_dev = d->cuda_dev; v->nsm = d->nsm; v->stream = d->stream;
        v->alloc = d->alloc; v->has_alloc = d->has_alloc; v->exch = d->exch; v->spw = d->spw;
        v->step_loop = d->step_loop;
        d->lv = v;
    }
    Dev *v = d->lv;
    v->parts = d->parts;  // non-owning copies (detached before release)
    v->wbricks = d->wbricks; v->amax_local = d->amax_local;
    v->world_ready = d->world_ready; v->nprims = d->nprims; memcpy(v->box, d->box, sizeof(v->box));
    v->nonempty = d->nonempty; v->b_wnodes = d->b_wnodes; v->b_prims_w = d->b_prims_w; v->b_prims_u = d->b_prims_u;
    v->local_parts = d->local_parts; v->wnodes_count = d->wnodes_count; v->bvh_levels = d->bvh_levels;
    v->build_launches = 0;
    v->cam = d->cam; v->cam_set = d->cam_set;
    v->fr = d->fr; v->fr_set = d->fr_set;
    if (replicated) {
        v->want_depth = false;
        v->pix_rank = d->rank;
        v->pix_nranks = d->nranks;
    } else {
        v->fr.flags |= DPR_FLAG_NO_BACKGROUND;
        v->want_depth = true;
        v->pix_rank = 0;
        v->pix_nranks = 1;
    }
    return v;
}

// Data-replicated mode: local renders of disjoint pixel sets, summed to rank 0.
int render_replicated(std::vector<Dev *> &L) {
    Dev *d0 = L[0];
    const int N = d0->nranks;
    for (Dev *d : L) {
        if (!d->world_ready) return fail(DPR_ERR_STATE, "dpr_commit_world has not been called");
        if (!d->cam_set || !d->fr_set) return fail(DPR_ERR_STATE, "camera and frame must be set before rendering");
        d->frame_done = 0;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    CK(cudaEventRecord(e0, d0->stream));
    {
        FrameCtx fc;
        memset(&fc.R, 0, sizeof(fc.R));
        RET(frame_setup(L, fc));  // collective digest check
    }
    for (Dev *d : L) {
        Dev *v = local_view(d, true);
        std::vector<Dev *> one = {v};
        RET(render_group(one));
    }
    const dpr_frame_desc &f = d0->fr;
    const int64_t P_ = (int64_t)f.W * f.H;
    const bool dumps = f.flags & DPR_FLAG_DEBUG_DUMPS;
    const size_t nd = (size_t)f.spp * f.max_depth * P_;
    if (!d0->comm) {
        Dev *root = L[0];
        for (size_t i = 1; i < L.size(); ++i) {
            launch_fb_accumulate(P<float4>(root->lv->b_fb_out), P<float4>(L[i]->lv->b_fb_out), P_, root->stream);
            if (dumps) {
                launch_u32_accumulate(P<uint32_t>(root->lv->b_events), P<uint32_t>(L[i]->lv->b_events), nd, root->stream);
                launch_u32_accumulate(P<uint32_t>(root->lv->b_occl), P<uint32_t>(L[i]->lv->b_occl), nd, root->stream);
            }
        }
    } else {
        Dev *d = d0;
        NK(ncclGroupStart());
        NK(ncclReduce(d->lv->b_fb_out.p, d->lv->b_fb_out.p, 4 * P_, ncclFloat, ncclSum, 0, d->comm, d->stream));
        if (dumps) {
            NK(ncclReduce(d->lv->b_events.p, d->lv->b_events.p, nd, ncclUint32, ncclSum, 0, d->comm, d->stream));
            NK(ncclReduce(d->lv->b_occl.p, d->lv->b_occl.p, nd, ncclUint32, ncclSum, 0, d->comm, d->stream));
        }
        NK(ncclGroupEnd());
    }
    CK(cudaEventRecord(e1, d0->stream));
    CK(cudaStreamSynchronize(d0->stream));
    CK(cudaGetLastError());
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    // rays: sum of every rank's local count
    std::vector<int64_t> mine(L.size() * 3);
    std::vector<const void *> sends;
    for (size_t i = 0; i < L.size(); ++i) {
        for (int k = 0; k < 3; ++k) mine[3 * i + k] = L[i]->lv->stats.rays[k];
        sends.push_back(&mine[3 * i]);
    }
    std::vector<std::vector<char>> out;
    RET(allgather_host(L, sends, sizeof(int64_t) * 3, out));
    const int64_t *all = reinterpret_cast<const int64_t *>(out[0].data());
    for (Dev *d : L) {
        d->stats = d->lv->stats;
        d->stats.nranks = N;
        d->stats.rank = d->rank;
        for (int k = 0; k < 3; ++k) {
            d->stats.rays[k] = 0;
            for (int r = 0; r < N; ++r) d->stats.rays[k] += all[3 * r + k];
        }
        d->stats.ms_frame = ms;
        d->stats.ms_frame_max = ms;
        d->frame_done = 1;
        d->dumps_valid = d->rank == 0 && dumps;
        d->mapped_w = d->rank == 0 ? f.W : 0;
        d->mapped_h = d->rank == 0 ? f.H : 0;
        d->frame_out = d->rank == 0 ? P<float>(d->lv->b_fb_out) : nullptr;
        d->replicated_frame = true;
    }
    return DPR_OK;
}

void release_bufs(Dev *d);

void release_local_view(Dev *d) {
    Dev *v = d->lv;
    if (!v) return;
    v->parts.clear();
    v->b_wnodes = Buf();
    v->b_prims_w = Buf();
    v->b_prims_u = Buf();
    release_bufs(v);
    delete v;
    d->lv = nullptr;
}

int render_composite(std::vector<Dev *> &L) {
    Dev *d0 = L[0];
    const int N = d0->nranks;
    for (Dev *d : L) {
        if (!d->world_ready) return fail(DPR_ERR_STATE, "dpr_commit_world has not been called");
        if (!d->cam_set || !d->fr_set) return fail(DPR_ERR_STATE, "camera and frame must be set before rendering");
        d->frame_done = 0;
    }
    cudaEvent_t e0, e1, e2;
    cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
    CK(cudaEventRecord(e0, d0->stream));
    {   // collective consistency check (same digest on all ranks)
        FrameCtx fc;
        memset(&fc.R, 0, sizeof(fc.R));
        RET(frame_setup(L, fc));
    }
    // 1. local renders: each rank sees only its own parts
    int64_t rays = 0;
    for (Dev *d : L) {
        Dev *v = local_view(d);
        std::vector<Dev *> one = {v};
        RET(render_group(one));
        rays += v->stats.rays[0] + v->stats.rays[1] + v->stats.rays[2];
    }
    CK(cudaEventRecord(e1, d0->stream));
    const dpr_frame_desc &f = d0->fr;
    const int64_t P_ = (int64_t)f.W * f.H, S = (P_ + N - 1) / N;
    auto span_count = [&](int r) { return std::max<int64_t>(0, std::min<int64_t>(P_, (int64_t)(r + 1) * S) - (int64_t)r * S); };
    for (Dev *d : L) {
        RET(ensure(d, d->b_frag_rgba, sizeof(float4) * N * S));
        RET(ensure(d, d->b_frag_z, sizeof(float) * N * S));
        RET(ensure(d, d->b_comp, sizeof(float4) * S));
        if (d->rank == 0) RET(ensure(d, d->b_comp_out, sizeof(float4) * P_));
    }
    // 2. parallel direct send: rank r receives every rank's fragments of its span
    if (!d0->comm) {
        for (Dev *dst : L)
            for (Dev *src : L) {
                int64_t c = span_count(dst->rank);
                if (!c) continue;
                CK(cudaMemcpyAsync(P<float4>(dst->b_frag_rgba) + (int64_t)src->rank * S,
                                   P<float4>(src->lv->b_fb_out) + (int64_t)dst->rank * S, sizeof(float4) * c,
                                   cudaMemcpyDeviceToDevice, dst->stream));
                CK(cudaMemcpyAsync(P<float>(dst->b_frag_z) + (int64_t)src->rank * S,
                                   P<float>(src->lv->b_depth) + (int64_t)dst->rank * S, sizeof(float) * c,
                                   cudaMemcpyDeviceToDevice, dst->stream));
            }
    } else {
        Dev *d = d0;
        const int64_t mine = span_count(d->rank);
        NK(ncclGroupStart());
        for (int q = 0; q < N; ++q) {
            const int64_t cq = span_count(q);
            if (q == d->rank) continue;
            if (cq) {
                NK(ncclSend(P<float4>(d->lv->b_fb_out) + (int64_t)q * S, 4 * cq, ncclFloat, q, d->comm, d->stream));
                NK(ncclSend(P<float>(d->lv->b_depth) + (int64_t)q * S, cq, ncclFloat, q, d->comm, d->stream));
            }
            if (mine) {
                NK(ncclRecv(P<float4>(d->b_frag_rgba) + (int64_t)q * S, 4 * mine, ncclFloat, q, d->comm, d->stream));
                NK(ncclRecv(P<float>(d->b_frag_z) + (int64_t)q * S, mine, ncclFloat, q, d->comm, d->stream));
            }
        }
        NK(ncclGroupEnd());
        if (mine) {
            CK(cudaMemcpyAsync(P<float4>(d->b_frag_rgba) + (int64_t)d->rank * S, P<float4>(d->lv->b_fb_out) + (int64_t)d->rank * S,
                               sizeof(float4) * mine, cudaMemcpyDeviceToDevice, d->stream));
            CK(cudaMemcpyAsync(P<float>(d->b_frag_z) + (int64_t)d->rank * S, P<float>(d->lv->b_depth) + (int64_t)d->rank * S,
                               sizeof(float) * mine, cudaMemcpyDeviceToDevice, d->stream));
        }
    }
    // 3. composite each rank's span
    for (Dev *d : L)
        launch_composite(P<float4>(d->b_frag_rgba), P<float>(d->b_frag_z), N, S, span_count(d->rank), f.B[0],
                         f.B[1], f.B[2], P<float4>(d->b_comp), d->stream);
    // 4. gather the spans to rank 0
    if (!d0->comm) {
        for (Dev *d : L) {
            int64_t c = span_count(d->rank);
            if (c) CK(cudaMemcpyAsync(P<float4>(L[0]->b_comp_out) + (int64_t)d->rank * S, d->b_comp.p, sizeof(float4) * c,
                                      cudaMemcpyDeviceToDevice, L[0]->stream));
        }
    } else {
        Dev *d = d0;
        NK(ncclGroupStart());
        if (d->rank == 0) {
            for (int q = 1; q < N; ++q)
                if (span_count(q)) NK(ncclRecv(P<float4>(d->b_comp_out) + (int64_t)q * S, 4 * span_count(q), ncclFloat, q, d->comm, d->stream));
        } else if (span_count(d->rank)) {
            NK(ncclSend(d->b_comp.p, 4 * span_count(d->rank), ncclFloat, 0, d->comm, d->stream));
        }
        NK(ncclGroupEnd());
        if (d->rank == 0 && span_count(0))
            CK(cudaMemcpyAsync(d->b_comp_out.p, d->b_comp.p, sizeof(float4) * span_count(0), cudaMemcpyDeviceToDevice, d->stream));
    }
    CK(cudaEventRecord(e2, d0->stream));
    CK(cudaStreamSynchronize(d0->stream));
    CK(cudaGetLastError());
    float ms_all = 0, ms_local = 0;
    cudaEventElapsedTime(&ms_all, e0, e2);
    cudaEventElapsedTime(&ms_local, e0, e1);
    cudaEventDestroy(e0); cudaEventDestroy(e1); cudaEventDestroy(e2);
    for (Dev *d : L) {
        d->stats = d->lv->stats;
        d->stats.nranks = N;
        d->stats.rank = d->rank;
        d->stats.ms_frame = ms_all;
        d->stats.ms_frame_max = ms_all;
        d->stats.ms_exchange = ms_all - ms_local;  // direct send + composite + gather
        d->frame_done = 1;
        d->dumps_valid = false;
        d->mapped_w = d->rank == 0 ? f.W : 0;
        d->mapped_h = d->rank == 0 ? f.H : 0;
        d->frame_out = d->rank == 0 ? P<float>(d->b_comp_out) : nullptr;
        d->replicated_frame = false;
    }
    (void)rays;
    return DPR_OK;
}

}  // namespace

struct dpr_device_s {
    Dev d;
};

// =======================================================================================
// C ABI
// =======================================================================================
extern "C" {

int dpr_get_unique_id(uint8_t out[DPR_UNIQUE_ID_BYTES]) {
    if (!out) return fail(DPR_ERR_INVALID_ARG, "null out");
    ncclUniqueId id;
    NK(ncclGetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == DPR_UNIQUE_ID_BYTES, "unique id size");
    memcpy(out, &id, DPR_UNIQUE_ID_BYTES);
    return DPR_OK;
}

int dpr_create_device(int rank, int nranks, int cuda_device, const uint8_t *uid, void *cuda_stream,
                      const dpr_allocator *alloc, dpr_device *out) {
    if (!out || nranks < 1 || nranks > DPR_MAX_RANKS || rank < 0 || rank >= nranks)
        return fail(DPR_ERR_INVALID_ARG, "bad rank/nranks/out");
    if (nranks > 1 && !uid) return fail(DPR_ERR_INVALID_ARG, "uid required for nranks > 1");
    dpr_device h = new dpr_device_s();
    int rc = init_dev(&h->d, rank, nranks, cuda_device, cuda_stream, alloc);
    if (rc != DPR_OK) { delete h; return rc; }
    // DPR_FORCE_NCCL=1: use NCCL even for a single rank (exercises the collective code paths
    // -- allgathers, grouped exchange, reduce -- on a one-GPU box)
    const char *force = getenv("DPR_FORCE_NCCL");
    const bool use_nccl = nranks > 1 || (force && force[0] == '1');
    if (use_nccl) {
        ncclUniqueId id;
        if (nranks > 1) memcpy(&id, uid, DPR_UNIQUE_ID_BYTES);
        else if (ncclGetUniqueId(&id) != ncclSuccess) { delete h; return fail(DPR_ERR_NCCL, "ncclGetUniqueId failed"); }
        ncclResult_t r = ncclCommInitRank(&h->d.comm, nranks, id, rank);
        if (r != ncclSuccess) {
            delete h;
            return fail(DPR_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
        }
    }
    *out = h;
    return DPR_OK;
}

int dpr_create_device_hostcoll(int rank, int nranks, int cuda_device, const dpr_host_collectives *coll,
                               void *cuda_stream, const dpr_allocator *alloc, dpr_device *out) {
    if (!out || !coll || !coll->allgather || nranks < 1 || nranks > DPR_MAX_RANKS || rank < 0 || rank >= nranks)
        return fail(DPR_ERR_INVALID_ARG, "bad rank/nranks/collectives/out");
    dpr_device h = new dpr_device_s();
    int rc = init_dev(&h->d, rank, nranks, cuda_device, cuda_stream, alloc);
    if (rc != DPR_OK) { delete h; return rc; }
    h->d.hc = *coll;
    h->d.has_hc = true;
    h->d.exch = 1;  // ray records move only by the fused (peer-memory) exchange
    *out = h;
    return DPR_OK;
}

int dpr_get_step_stats(dpr_device dev, int max_steps, int64_t *S_out, int64_t *V_out, double *ms_out,
                       double *sync_ms_out, int *nsteps) {
    if (!valid_dev(dev) || max_steps < 0 || !nsteps) return fail(DPR_ERR_INVALID_ARG, "null argument");
    Dev *d = &dev->d;
    if (!d->frame_done) return fail(DPR_ERR_STATE, "no frame rendered");
    const int N = d->nranks;
    const int n = (int)std::min<int64_t>(d->nsteps_rec, max_steps);
    if (S_out) memcpy(S_out, d->step_S.data(), sizeof(int64_t) * (size_t)n * 3 * N * N);
    if (V_out) memcpy(V_out, d->step_V.data(), sizeof(int64_t) * (size_t)n * 3 * N);
    if (ms_out) memcpy(ms_out, d->step_ms.data(), sizeof(double) * n);
    if (sync_ms_out) memcpy(sync_ms_out, d->step_sync_ms.data(), sizeof(double) * n);
    *nsteps = (int)d->nsteps_rec;
    return DPR_OK;
}

int dpr_test_step_barrier(int cuda_device, int nranks, int iters, int64_t *mismatches) {
    if (nranks < 1 || nranks > DPR_MAX_RANKS || iters < 0 || !mismatches)
        return fail(DPR_ERR_INVALID_ARG, "bad arguments");
    CK(cudaSetDevice(cuda_device));
    const size_t mb = sizeof(uint32_t) * (size_t)nranks * 2 * DPR_MAX_RANKS * 4;
    char *buf = nullptr;
    CK(cudaMalloc(&buf, mb + sizeof(uint32_t) * (nranks + 1)));
    uint32_t *mbox = (uint32_t *)buf, *seq = (uint32_t *)(buf + mb), *bad = seq + nranks;
    cudaError_t e = cudaMemset(buf, 0, mb + sizeof(uint32_t) * (nranks + 1));
    if (e == cudaSuccess) e = (cudaError_t)test_step_barrier(nranks, iters, mbox, seq, bad, 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    uint32_t hb = 0;
    if (e == cudaSuccess) e = cudaMemcpy(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost);
    cudaFree(buf);
    if (e != cudaSuccess) return fail(DPR_ERR_CUDA, std::string("step barrier test: ") + cudaGetErrorString(e));
    *mismatches = hb;
    return DPR_OK;
}

int dpr_test_radix_sort(int cuda_device, const uint32_t *keys, int64_t n, uint32_t *perm_out) {
    if (n < 0 || n > ((int64_t)1 << 30) || (n > 0 && (!keys || !perm_out)))
        return fail(DPR_ERR_INVALID_ARG, "bad arguments");
    if (n == 0) return DPR_OK;
    static_assert(sizeof(mkey_t) == sizeof(uint32_t), "32-bit Morton keys");
    CK(cudaSetDevice(cuda_device));
    const int64_t ntiles = radix_tiles(n);
    char *buf = nullptr;
    const size_t kv = sizeof(uint32_t) * (size_t)n;
    CK(cudaMalloc(&buf, 4 * kv + sizeof(uint32_t) * 256 * (ntiles + 1)));
    mkey_t *k[2] = {(mkey_t *)buf, (mkey_t *)(buf + kv)};
    uint32_t *v[2] = {(uint32_t *)(buf + 2 * kv), (uint32_t *)(buf + 3 * kv)};
    uint32_t *tile = (uint32_t *)(buf + 4 * kv);
    cudaError_t e = cudaMemcpy(k[0], keys, kv, cudaMemcpyDeviceToDevice);
    if (e == cudaSuccess) {
        launch_iota(v[0], n, 0);
        e = cudaGetLastError();
    }
    int launches = 0, cur = 0;
    for (int pass = 0; pass < MKEY_DIGITS && e == cudaSuccess; ++pass) {
        launch_radix_pass(k[cur], v[cur], k[cur ^ 1], v[cur ^ 1], n, 8 * pass, tile, 0, &launches);
        cur ^= 1;
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(perm_out, v[cur], kv, cudaMemcpyDeviceToDevice);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaFree(buf);
    if (e != cudaSuccess) return fail(DPR_ERR_CUDA, std::string("radix sort test: ") + cudaGetErrorString(e));
    return DPR_OK;
}

int dpr_create_loopback_group(int nranks, int cuda_device, void *cuda_stream, const dpr_allocator *alloc,
                              dpr_device *out) {
    if (!out || nranks < 1 || nranks > DPR_MAX_RANKS) return fail(DPR_ERR_INVALID_ARG, "bad nranks/out");
    LoopGroup *g = new LoopGroup();
    for (int r = 0; r < nranks; ++r) {
        dpr_device h = new dpr_device_s();
        int rc = init_dev(&h->d, r, nranks, cuda_device, cuda_stream, alloc);
        if (rc != DPR_OK) return rc;
        h->d.group = g;
        if (!getenv("DPR_EXCHANGE")) h->d.exch = 1;  // loopback default: fused appends
        g->devs.push_back(&h->d);
        out[r] = h;
    }
    return DPR_OK;
}

int dpr_release_device(dpr_device dev) {
    if (!valid_dev(dev)) return fail(DPR_ERR_INVALID_ARG, "null device");
    Dev *d = &dev->d;
    cudaSetDevice(d->cuda_dev);
    cudaStreamSynchronize(d->stream);
    if (d->cstream) cudaStreamSynchronize(d->cstream);
    for (auto &b : d->part_pool) dfree(d, b);
    d->part_pool.clear();
    release_bufs(d);
    cudaStreamSynchronize(d->stream);
    if (d->cstream) cudaStreamDestroy(d->cstream);
    if (d->copy_ev) cudaEventDestroy(d->copy_ev);
    if (d->order_ev) cudaEventDestroy(d->order_ev);
    if (d->comm) ncclCommDestroy(d->comm);
    if (d->group) {
        auto &v = d->group->devs;
        v[d->rank] = nullptr;
        bool empty = true;
        for (auto *x : v) if (x) empty = false;
        if (empty) delete d->group;
    }
    delete dev;
    return DPR_OK;
}

int dpr_commit_part(dpr_device dev, const dpr_part_desc *part) {
    if (!valid_dev(dev)) return fail(DPR_ERR_INVALID_ARG, "null device");
    RET(check_part(part));
    Dev *d = &dev->d;
    CK(cudaSetDevice(d->cuda_dev));
    PartStore p;
    p.kind = part->kind;
    for (int c = 0; c < 3; ++c) p.albedo[c] = part->albedo[c];
    p.has_hint = part->has_bounds_hint;
    for (int c = 0; c < 6; ++c) p.hint[c] = part->bounds_hint[c];
    if (p.kind == DPR_PART_TRIANGLES) {
        p.nv = part->n_verts;
        p.nt = part->n_tris;
        RET(copy_in_geom(d, p.verts, part->verts, sizeof(float) * 3 * p.nv, part->memory));
        RET(copy_in_geom(d, p.idx, part->idx, sizeof(int32_t) * 3 * p.nt, part->memory));
    } else if (p.kind == DPR_PART_SPHERES) {
        p.ns = part->n_spheres;
        RET(copy_in_geom(d, p.spheres, part->spheres, sizeof(float) * 4 * p.ns, part->memory));
    } else {
        for (int c = 0; c < 3; ++c) {
            p.gdims[c] = part->gdims[c]; p.lo[c] = part->cell_lo[c]; p.hi[c] = part->cell_hi[c];
            p.origin[c] = part->origin[c]; p.spacing[c] = part->spacing[c];
        }
        for (auto &q : d->parts)
            if (q.kind == DPR_PART_BRICK)
                for (int c = 0; c < 3; ++c)
                    if (q.gdims[c] != p.gdims[c] || q.origin[c] != p.origin[c] || q.spacing[c] != p.spacing[c])
                        return fail(DPR_ERR_INVALID_ARG, "bricks of one world must share gdims/origin/spacing");
        int nb = 0;
        for (auto &q : d->parts) nb += q.kind == DPR_PART_BRICK;
        if (nb >= MAX_BRICKS) return fail(DPR_ERR_INVALID_ARG, "too many bricks on one rank");
        p.tf_lo = part->tf_lo; p.tf_hi = part->tf_hi; p.dscale = part->density_scale;
        size_t nvox = (size_t)(p.hi[0] - p.lo[0] + 1) * (p.hi[1] - p.lo[1] + 1) * (p.hi[2] - p.lo[2] + 1);
        RET(copy_in(d, p.vox, part->voxels, sizeof(float) * nvox, part->memory));
        RET(copy_in(d, p.tf, part->tf, sizeof(float) * 4 * 256, part->memory));
        std::vector<float> tfh(4 * 256);
        CK(cudaMemcpyAsync(tfh.data(), p.tf.p, sizeof(float) * 4 * 256, cudaMemcpyDeviceToHost, d->stream));
        CK(cudaStreamSynchronize(d->stream));
        for (int j = 0; j < 256; ++j) p.amax = std::max(p.amax, std::min(1.0f, tfh[4 * j + 3] * p.dscale));
    }
    d->parts.push_back(p);
    return DPR_OK;
}

int dpr_clear_parts(dpr_device dev) {
    if (!valid_dev(dev)) return fail(DPR_ERR_INVALID_ARG, "null device");
    Dev *d = &dev->d;
    // buffers freed below are stream-ordered on the library stream: order them after any
    // upload still in flight on the copy stream
    if (d->copy_pending) CK(cudaStreamWaitEvent(d->stream, d->copy_ev, 0));
    for (auto &p : d->parts) {
        // geometry arrays are recycled for the next commit (bounded pool); bricks are freed
        // stream-ordered (a render may still read them)
        for (Buf *b : {&p.verts, &p.idx, &p.spheres})
            if (b->p) {
                if (d->part_pool.size() < 64) { d->part_pool.push_back(*b); *b = Buf(); }
                else dfree(d, *b);
            }
        // bricks: the committed world still renders from them until the next build
        for (Buf *b : {&p.vox, &p.tf, &p.mc})
            if (b->p) { d->retired.push_back(*b); *b = Buf(); }
    }
    d->parts.clear();
    return DPR_OK;
}

int dpr_commit_world(dpr_device dev) {
    if (!valid_dev(dev)) return fail(DPR_ERR_INVALID_ARG, "null device");
    Dev *d = &dev->d;
    CK(cudaSetDevice(d->cuda_dev));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, d->stream);
    int rc = build_world(d);
    cudaEventRecord(e1, d->stream);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    d->ms_build = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return rc;
}

int dpr_get_world_bounds(dpr_device dev, float lohi_host[6]) {
    if (!valid_dev(dev) || !lohi_host) return fail(DPR_ERR_INVALID_ARG, "null argument");
    Dev *d = &dev->d;
    if (!d->world_ready) return fail(DPR_ERR_STATE, "dpr_commit_world has not been called");
    std::vector<Dev *> L;
    if (d->group) {
        for (Dev *x : d->group->devs) if (!x || !x->world_ready) return fail(DPR_ERR_STATE, "group member world not ready");
        L = d->group->devs;
    } else {
        L = {d};
    }
    std::vector<const void *> sends;
    for (Dev *x : L) sends.push_back(x->box);
    std::vector<std::vector<char>> out;
    RET(allgather_host(L, sends, sizeof(float) * 6, out));
    const float *b = reinterpret_cast<const float *>(out[0].data());
    for (int c = 0; c < 3; ++c) { lohi_host[c] = INFINITY; lohi_host[3 + c] = -INFINITY; }
    for (int r = 0; r < d->nranks; ++r)
        for (int c = 0; c < 3; ++c) {
            lohi_host[c] = fminf(lohi_host[c], b[6 * r + c]);
            lohi_host[3 + c] = fmaxf(lohi_host[3 + c], b[6 * r + 3 + c]);
        }
    return DPR_OK;
}

int dpr_set_camera(dpr_device dev, const dpr_camera_basis *cam) {
    if (!valid_dev(dev) || !cam) return fail(DPR_ERR_INVALID_ARG, "null argument");
    if (!(cam->lens_radius >= 0.0f) || (cam->lens_radius > 0.0f && !(cam->focus_dist > 0.0f)))
        return fail(DPR_ERR_INVALID_ARG, "lens_radius must be >= 0 and focus_dist > 0 when lens_radius > 0");
    dev->d.cam = *cam;
    dev->d.cam_set = true;
    return DPR_OK;
}

int dpr_set_frame(dpr_device dev, const dpr_frame_desc *fr) {
    if (!valid_dev(dev) || !fr) return fail(DPR_ERR_INVALID_ARG, "null argument");
    if (fr->W <= 0 || fr->H <= 0 || fr->spp <= 0 || fr->spp > 65535 || fr->spp_batch <= 0 || fr->max_depth <= 0 ||
        fr->max_depth > 200 || fr->ao_k < 0 || fr->ao_k > 30)
        return fail(DPR_ERR_INVALID_ARG, "bad frame parameters");
    dpr_frame_desc &f = dev->d.fr;  // field by field: the caller's padding bytes are not copied
    memset(&f, 0, sizeof(f));
    f.W = fr->W; f.H = fr->H; f.spp = fr->spp; f.spp_batch = std::min(fr->spp_batch, fr->spp);
    f.max_depth = fr->max_depth; f.ao_k = fr->ao_k; f.ao_radius = fr->ao_radius;
    for (int c = 0; c < 3; ++c) {
        f.light_dir[c] = fr->light_dir[c]; f.E[c] = fr->E[c]; f.A[c] = fr->A[c]; f.B[c] = fr->B[c];
    }
    f.dt = fr->dt; f.seed = fr->seed; f.flags = fr->flags;
    dev->d.fr_set = true;
    return DPR_OK;
}

int dpr_render_frame(dpr_device dev) {
    if (!valid_dev(dev)) return fail(DPR_ERR_INVALID_ARG, "null device");
    Dev *d = &dev->d;
    if (d->group) return fail(DPR_ERR_STATE, "loopback devices render with dpr_render_frame_group");
    CK(cudaSetDevice(d->cuda_dev));
    std::vector<Dev *> L = {d};
    return render_group(L);
}

int dpr_render_frame_group(dpr_device *devs, int n) {
    if (!devs || n < 1) return fail(DPR_ERR_INVALID_ARG, "bad group");
    std::vector<Dev *> L;
    for (int i = 0; i < n; ++i) {
        if (!devs[i] || !devs[i]->d.group || devs[i]->d.rank != i || devs[i]->d.nranks != n)
            return fail(DPR_ERR_INVALID_ARG, "devices must be a full loopback group in rank order");
        L.push_back(&devs[i]->d);
    }
    CK(cudaSetDevice(L[0]->cuda_dev));
    return render_group(L);
}

int dpr_render_frame_composite(dpr_device dev) {
    if (!valid_dev(dev)) return fail(DPR_ERR_INVALID_ARG, "null device");
    Dev *d = &dev->d;
    if (d->group) return fail(DPR_ERR_STATE, "loopback devices use dpr_render_frame_composite_group");
    CK(cudaSetDevice(d->cuda_dev));
    std::vector<Dev *> L = {d};
    return render_composite(L);
}

int dpr_render_frame_composite_group(dpr_device *devs, int n) {
    if (!devs || n < 1) return fail(DPR_ERR_INVALID_ARG, "bad group");
    std::vector<Dev *> L;
    for (int i = 0; i < n; ++i) {
        if (!devs[i] || !devs[i]->d.group || devs[i]->d.rank != i || devs[i]->d.nranks != n)
            return fail(DPR_ERR_INVALID_ARG, "devices must be a full loopback group in rank order");
        L.push_back(&devs[i]->d);
    }
    CK(cudaSetDevice(L[0]->cuda_dev));
    return render_composite(L);
}

int dpr_render_frame_replicated(dpr_device dev) {
    if (!valid_dev(dev)) return fail(DPR_ERR_INVALID_ARG, "null device");
    Dev *d = &dev->d;
    if (d->group) return fail(DPR_ERR_STATE, "loopback devices use dpr_render_frame_replicated_group");
    CK(cudaSetDevice(d->cuda_dev));
    std::vector<Dev *> L = {d};
    return render_replicated(L);
}

int dpr_render_frame_replicated_group(dpr_device *devs, int n) {
    if (!devs || n < 1) return fail(DPR_ERR_INVALID_ARG, "bad group");
    std::vector<Dev *> L;
    for (int i = 0; i < n; ++i) {
        if (!devs[i] || !devs[i]->d.group || devs[i]->d.rank != i || devs[i]->d.nranks != n)
            return fail(DPR_ERR_INVALID_ARG, "devices must be a full loopback group in rank order");
        L.push_back(&devs[i]->d);
    }
    CK(cudaSetDevice(L[0]->cuda_dev));
    return render_replicated(L);
}

int dpr_frame_ready(dpr_device dev, int wait) {
    (void)wait;
    if (!valid_dev(dev)) return fail(DPR_ERR_INVALID_ARG, "null device");
    return dev->d.frame_done;
}

int dpr_map_frame(dpr_device dev, const float **rgba, int *w, int *h, int *undefined) {
    if (!valid_dev(dev) || !rgba || !w || !h || !undefined) return fail(DPR_ERR_INVALID_ARG, "null argument");
    Dev *d = &dev->d;
    if (!d->frame_done) return fail(DPR_ERR_STATE, "no frame rendered");
    if (d->rank != 0) {
        *rgba = nullptr; *w = 0; *h = 0; *undefined = 1;
        return DPR_OK;
    }
    *rgba = d->frame_out;
    *w = d->mapped_w;
    *h = d->mapped_h;
    *undefined = 0;
    return DPR_OK;
}

int dpr_get_debug(dpr_device dev, const uint32_t **events, const uint32_t **occl) {
    if (!valid_dev(dev) || !events || !occl) return fail(DPR_ERR_INVALID_ARG, "null argument");
    Dev *d = &dev->d;
    if (d->rank != 0 || !d->dumps_valid) return fail(DPR_ERR_STATE, "no debug dumps (rank 0, DPR_FLAG_DEBUG_DUMPS)");
    Dev *src = d->replicated_frame ? d->lv : d;
    *events = P<uint32_t>(src->b_events);
    *occl = P<uint32_t>(src->b_occl);
    return DPR_OK;
}

int dpr_get_stats(dpr_device dev, dpr_stats *out) {
    if (!valid_dev(dev) || !out) return fail(DPR_ERR_INVALID_ARG, "null argument");
    *out = dev->d.stats;
    out->ms_build = dev->d.ms_build;
    return DPR_OK;
}

const char *dpr_last_error(dpr_device dev) {
    (void)dev;
    return g_err.c_str();
}

int dpr_exchange_plan(int nranks, int rank, const int64_t *counts, int64_t capacity, int64_t *recv_offset,
                      int64_t *total_in, int64_t *global_total) {
    if (nranks < 1 || rank < 0 || rank >= nranks || !counts || !recv_offset || !total_in || !global_total)
        return fail(DPR_ERR_INVALID_ARG, "bad exchange plan arguments");
    int64_t g = 0;
    for (int i = 0; i < nranks * nranks; ++i) {
        if (counts[i] < 0) return fail(DPR_ERR_INVALID_ARG, "negative count");
        g += counts[i];
    }
    int64_t off = counts[(int64_t)rank * nranks + rank];
    for (int src = 0; src < nranks; ++src) {
        if (src == rank) { recv_offset[src] = 0; continue; }
        recv_offset[src] = off;
        off += counts[(int64_t)src * nranks + rank];
    }
    *total_in = off;
    *global_total = g;
    if (off > capacity) return fail(DPR_ERR_QUEUE_OVERFLOW, "receive exceeds queue capacity");
    return DPR_OK;
}

}  // extern "C"
