/*
 * dpr.h -- C ABI of the B200-native data-parallel wavefront ray tracer (libdpr.so).
 *
 * What this library is (PAPER.md = P:<line>, paper section in parentheses):
 *   A data-parallel ANARI-style device in the sense of S3: every rank (one
 *   process per GPU) commits ONLY ITS OWN part of the world -- "everything under World is
 *   defined locally within the rank" (S3.1.2) -- and a COLLECTIVE renderFrame
 *   (S3.2) path-traces the union of all parts by ray forwarding: "rays are sent
 *   to the node(s) that may have geometry that may intersect a given ray ... each ray will
 *   always find its respectively closest intersection no matter which rank ... holds that
 *   respective geometry" (S5.2), one lock-step ray wave-front at a time "until
 *   all wave-fronts contain zero rays" (S2.2).  The final framebuffer is
 *   provided on rank 0 only (S3.1.3).  The arithmetic the paper leaves open is
 *   pinned in SURVEY.md 8(c) (P1-P13) and listed as readings in DESIGN.md.
 *
 * Conventions for every call:
 *   - Returns dpr_status (0 = DPR_OK).  Nothing throws across the ABI.  On failure
 *     dpr_last_error(dev) returns a NUL-terminated message (thread-local, valid until the
 *     next call on that thread).
 *   - COLLECTIVE calls must be made by every rank of the device group in the same order
 *     (as in S3.2).  Calling one on a subset of ranks deadlocks; this is not
 *     detected.  A collective consistency failure is reported on EVERY rank.
 *   - LOCAL calls involve no communication.
 *   - All GPU work is issued on the stream passed to dpr_create_device, in order.
 *   - Pointers named *_host are host memory; device pointers are CUDA global memory on the
 *     device's GPU.  Sizes are element counts unless named *_bytes.
 */
#ifndef DPR_H
#define DPR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define DPR_API __attribute__((visibility("default")))
#else
#define DPR_API
#endif

#define DPR_MAX_RANKS 16
#define DPR_UNIQUE_ID_BYTES 128

typedef struct dpr_device_s *dpr_device; /* opaque; one per rank */

typedef enum {
    DPR_OK = 0,
    DPR_ERR_INVALID_ARG = -1,   /* bad pointer/size/enum; nothing was changed */
    DPR_ERR_STATE = -2,         /* call not valid now (e.g. render before commit_world) */
    DPR_ERR_CUDA = -3,          /* a CUDA runtime error; the device should be released */
    DPR_ERR_NCCL = -4,          /* an NCCL error, incl. asynchronous ones (polled with
                                   ncclCommGetAsyncError while waiting), a collective that did not
                                   complete within DPR_TIMEOUT_S seconds (default 600), or a
                                   device step barrier that did not complete within
                                   min(DPR_TIMEOUT_S, 60) s (a dead peer): the communicator is
                                   aborted; every later collective returns this; release the device */
    DPR_ERR_CONSISTENCY = -5,   /* camera/frame parameters differ between ranks */
    DPR_ERR_OOM = -6,           /* device allocation failed */
    DPR_ERR_QUEUE_OVERFLOW = -7 /* a ray queue exceeded its capacity; lower spp_batch */
} dpr_status;

typedef enum { DPR_PART_TRIANGLES = 0, DPR_PART_SPHERES = 1, DPR_PART_BRICK = 2 } dpr_part_kind;
/* HOST: copied before dpr_commit_part returns.  DEVICE: device-to-device copy, stream-ordered.
 * HOST_ASYNC: (pinned) host memory read by the copy engine on a side stream, overlapping
 * whatever the device is still rendering; the array must stay valid and unchanged until the
 * next dpr_commit_world returns (which waits for the copies).  Triangle / sphere arrays only;
 * bricks are copied as HOST. */
typedef enum { DPR_MEMORY_HOST = 0, DPR_MEMORY_DEVICE = 1, DPR_MEMORY_HOST_ASYNC = 2 } dpr_memory;

/* frame flags */
#define DPR_FLAG_JITTER_CENTER 1u  /* camera jitter fixed at 0.5 (test mode) */
#define DPR_FLAG_DEBUG_DUMPS 2u    /* record P13 event / occlusion dumps (parity mode) */
#define DPR_FLAG_RING 8u            /* ring schedule instead of the visit rule ("wave-fronts
                                      are exchanged in a ring buffer"; reading R-RING):
                                      every ray of pixel p starts at rank floor(p*N/(W*H)), is
                                      traced by every rank in ring order without culling or
                                      early-out, resolves at the last one; children go home.
                                      Same image, events and occlusion bits as the visit rule */
#define DPR_FLAG_DELTA 16u          /* volumes by delta tracking with one global majorant instead
                                      of the P10 per-sample march (NEXT f4; DESIGN.md readings
                                      R-DELTA, R-LOG): extinction alpha(x)/dt, majorant amax/dt,
                                      tentative points from the ray's entry into the global grid
                                      domain, event id VOL_BIT | tentative index */
#define DPR_FLAG_NO_BACKGROUND 4u  /* misses add no background (set internally for the local
                                      renders of the compositing contrast device) */

/* Device memory provider.  NULL allocator -> stream-ordered cudaMallocAsync.
 * The Python binding passes PyTorch's caching allocator (north_star: PyTorch owns device
 * memory).  alloc returns NULL on failure (-> DPR_ERR_OOM). */
typedef struct {
    void *(*alloc)(void *ctx, size_t bytes, void *cuda_stream);
    void (*free)(void *ctx, void *ptr, size_t bytes, void *cuda_stream);
    void *ctx;
} dpr_allocator;

/* One rank-local world part.  Arrays are COPIED at commit (ANARI commit
 * semantics): the caller may free them when dpr_commit_part returns (except
 * DPR_MEMORY_HOST_ASYNC, see dpr_memory).
 *   TRIANGLES: verts float[n_verts][3] (finite), idx int32[n_tris][3] (indices into verts).
 *              A triangle whose binary32 cross(v1-v0, v2-v0) is exactly zero (no area, no
 *              normal) is never hit (reading R-DEGEN).
 *   SPHERES:   spheres float[n_spheres][4] = centre xyz, radius (finite, > 0).
 *   Indices, finiteness and radii are validated on the GPU by dpr_commit_world
 *   (DPR_ERR_INVALID_ARG).
 *   BRICK:     a brick of one global structured grid: gdims (points per axis), origin,
 *              spacing (> 0); the brick owns cells [cell_lo, cell_hi) (half-open) and
 *              stores voxels [cell_lo, cell_hi] INCLUSIVE (one ghost layer), x fastest;
 *              tf float[256][4] rgba over [tf_lo, tf_hi], alpha scaled by density_scale
 *              (SURVEY P10).  All bricks of a world must share gdims/origin/spacing.
 *              A brick stores fewer than 2^31 voxel rows (y extent * z extent, each
 *              cell_hi - cell_lo + 1; else DPR_ERR_INVALID_ARG).
 *   albedo: matte rgb for TRIANGLES / SPHERES.
 *   bounds_hint: optional app-provided box (S8.2 "box3 boundingBox"); it is
 *   only VALIDATED to contain the part (DPR_ERR_INVALID_ARG otherwise), never used for
 *   routing (routing uses the exact computed bounds; reading A14). */
typedef struct {
    int32_t kind;   /* dpr_part_kind */
    int32_t memory; /* dpr_memory of all array pointers below */
    float albedo[3];
    int64_t n_verts;
    const float *verts;
    int64_t n_tris;
    const int32_t *idx;
    int64_t n_spheres;
    const float *spheres;
    int32_t gdims[3];
    float origin[3];
    float spacing[3];
    int32_t cell_lo[3];
    int32_t cell_hi[3];
    const float *voxels;
    const float *tf;
    float tf_lo, tf_hi, density_scale;
    int32_t has_bounds_hint;
    float bounds_hint[6]; /* lo xyz, hi xyz */
} dpr_part_desc;

/* Camera basis, float32, identical on all ranks.  Primary ray through pixel
 * (x,y) (bottom-left origin, row-major) with jitter (jx,jy):
 *   q = L + ((x+jx)/W)*U + ((y+jy)/H)*V;  dir = normalize(q), origin E.
 * Depth of field ("rendered with depth of field"; reading R-DOF): with
 * lens_radius > 0 the origin is a point of the thin lens (radius lens_radius, in the plane
 * spanned by U and V, sampled by Philox purpose 1) and the ray passes through the point
 * E + focus_dist*q of the focal plane (distance focus_dist along the view axis).
 * lens_radius == 0 is the pinhole camera bit for bit; focus_dist must then be ignored. */
typedef struct { float E[3], L[3], U[3], V[3]; float lens_radius, focus_dist; } dpr_camera_basis;

/* Frame / renderer parameters, identical on all ranks.
 *   W,H pixels; spp samples per pixel, traced in batches of spp_batch samples (bounded
 *   queue memory); max_depth shaded path vertices; ao_k AO rays per surface vertex with
 *   length ao_radius; light_dir unit vector TOWARD the light with irradiance E; ambient A;
 *   background B; dt volume sample spacing (world units); seed the Philox key; flags. */
typedef struct {
    int32_t W, H, spp, spp_batch, max_depth, ao_k;
    float ao_radius;
    float light_dir[3], E[3], A[3], B[3];
    float dt;
    uint64_t seed;
    uint32_t flags;
} dpr_frame_desc;

/* Per-frame statistics.  Matrices are GLOBAL (gathered over all ranks at the end of the
 * collective render); kinds are 0 path, 1 shadow, 2 ambient-occlusion.
 *   S[k][src][dst]  rays of kind k forwarded src -> dst (P8 routing)
 *   V[k][r]         visits (local traces) of kind k at rank r
 *   rays[k]         rays generated (primaries counted once + every spawned ray)
 *   steps           lock-step wavefront steps with >= 1 ray traced anywhere (P8b)
 *   the *_local counters and ms_* timers are THIS rank's; ms_* are CUDA-event device times */
typedef struct {
    int32_t nranks, rank;
    int64_t S[3][DPR_MAX_RANKS][DPR_MAX_RANKS];
    int64_t V[3][DPR_MAX_RANKS];
    int64_t rays[3];
    int64_t steps;
    int64_t node_visits_local, tri_tests_local, sphere_tests_local, vol_samples_local;
    int64_t records_in_local, records_out_local;
    int64_t exchanged_bytes_local;
    int64_t kernel_launches_local;
    int64_t trace_path_launches, trace_occl_launches;
    double ms_frame, ms_build, ms_gen, ms_trace_path, ms_trace_occl, ms_exchange, ms_reduce;
    double ms_frame_max; /* max over ranks of ms_frame */
    int64_t path_bytes_alg_local, occl_bytes_alg_local; /* algorithmic bytes */
    /* per trace kernel (0 = k_trace_path, 1 = k_trace_occl), this rank: rays traced, wide-node
     * visits, triangle tests, sphere tests, volume samples */
    int64_t kernel_rays_local[2], kernel_nodes_local[2], kernel_tris_local[2], kernel_sphs_local[2],
        kernel_vols_local[2];
    int64_t bvh_nodes_local, bvh_levels_local; /* wide-BVH size of this rank's world */
    int64_t step_loop_device; /* 1: the lock-step loop ran on the device (CUDA graph, no host
                                 round trip per step); ms_trace_* are then globaltimer spans
                                 (first CTA start .. last CTA end) and ms_exchange the time in
                                 the step barrier */
    int64_t graph_builds;     /* step-loop graphs captured so far on this device */
    int64_t comm_nranks;      /* ranks of the NCCL communicator (ncclCommCount), 0 without NCCL */
    double ms_kernel_span[2]; /* k_trace_path / k_trace_occl: sum over launches that traced rays
                                 of the globaltimer span first CTA start .. last CTA end */
} dpr_stats;

/* Host-collective transport: a blocking, collective all-gather supplied by the caller (e.g.
 * torch.distributed over gloo).  Every rank calls it with the same `bytes`; recv_host receives
 * nranks*bytes, rank-major; returns 0 on success.  Called from the thread that called the
 * dpr_* function. */
typedef struct {
    int (*allgather)(void *ctx, const void *send_host, void *recv_host, size_t bytes);
    void *ctx;
} dpr_host_collectives;

/* ---- device lifetime ------------------------------------------------------------------ */

/* LOCAL, rank 0 only: create an NCCL unique id to broadcast to all ranks (the harness uses
 * torch.distributed for the broadcast).  out must hold DPR_UNIQUE_ID_BYTES bytes. */
DPR_API int dpr_get_unique_id(uint8_t out[DPR_UNIQUE_ID_BYTES]);

/* COLLECTIVE (P:460-461 collaborative device creation): rank in [0,nranks), one CUDA device
 * per rank; uid from dpr_get_unique_id (ignored when nranks == 1: no NCCL is used, and the
 * device behaves exactly like a non-parallel renderer).  cuda_stream: a
 * cudaStream_t (NULL = legacy default stream).  alloc may be NULL.  *out receives the
 * handle; release it with dpr_release_device. */
DPR_API int dpr_create_device(int rank, int nranks, int cuda_device, const uint8_t *uid,
                      void *cuda_stream, const dpr_allocator *alloc, dpr_device *out);

/* COLLECTIVE: a rank whose control collectives (frame setup, step counts, barriers) go
 * through `coll` instead of NCCL, and whose ray records move by the fused exchange only:
 * shading / resolve kernels append straight into the destination rank's queues through CUDA
 * IPC mappings (system-scope tail atomics), and rank 0 sums the peers' framebuffers through
 * the same mappings (a7).  Processes may share one GPU (IPC works within a device), which is
 * how the cross-process data plane is tested on a one-GPU box.  The step loop runs on the
 * host in this mode (no kernel ever waits for another process).  coll is copied. */
DPR_API int dpr_create_device_hostcoll(int rank, int nranks, int cuda_device, const dpr_host_collectives *coll,
                               void *cuda_stream, const dpr_allocator *alloc, dpr_device *out);

/* LOCAL test fixture: nranks virtual ranks in ONE process on ONE GPU (exchange by
 * device-to-device copies instead of NCCL).  out[nranks] receives the handles.  Render
 * them with dpr_render_frame_group; every other call is per handle as usual. */
DPR_API int dpr_create_loopback_group(int nranks, int cuda_device, void *cuda_stream,
                              const dpr_allocator *alloc, dpr_device *out);

/* COLLECTIVE (P:428-431 lock-step release).  Frees everything the device owns. */
DPR_API int dpr_release_device(dpr_device dev);

/* ---- world (local content) ------------------------------------------------- */

/* LOCAL: copy one part (see dpr_part_desc).  Parts are numbered in commit order; global
 * primitive ids are base_rank + local index.  Parts describe the NEXT world:
 * the world of the last dpr_commit_world stays renderable while parts are cleared and
 * committed (so uploads of frame k+1 can overlap the render of frame k). */
DPR_API int dpr_commit_part(dpr_device dev, const dpr_part_desc *part);

/* LOCAL: drop all committed parts (the next commit_world builds an empty world; the current
 * world, including its bricks, remains renderable until then). */
DPR_API int dpr_clear_parts(dpr_device dev);

/* LOCAL: (re)build the rank's acceleration structures from the committed parts, on the
 * GPU: per-prim AABBs, 30-bit Morton codes, LSD radix sort, agglomerative LBVH (the Karras
 * hierarchy + refit or PLOC with env DPR_BUILDER=karras|ploc), collapse into a compressed
 * 8-wide BVH ("negligible pre-processing time") and brick macrocells.  May be called again to rebuild
 * from the resident parts.  DPR_ERR_INVALID_ARG if a triangle index is out of range,
 * a coordinate is not finite or a sphere radius is not > 0 (validated on the GPU here, not at
 * commit_part) or a bounds_hint does not contain its part; the world is then not ready. */
DPR_API int dpr_commit_world(dpr_device dev);

/* COLLECTIVE (getProperty(WAIT) on the world): union of all ranks' world
 * bounds (exact, unpadded).  lohi_host[6] = lo xyz, hi xyz (+inf/-inf if empty). */
DPR_API int dpr_get_world_bounds(dpr_device dev, float lohi_host[6]);

/* ---- frame ---------------------------------------------------------------------------- */
DPR_API int dpr_set_camera(dpr_device dev, const dpr_camera_basis *cam);  /* LOCAL */
DPR_API int dpr_set_frame(dpr_device dev, const dpr_frame_desc *frame);   /* LOCAL */

/* COLLECTIVE renderFrame.  Blocks until the frame is complete and the reduced
 * framebuffer is on rank 0.  Fails with DPR_ERR_CONSISTENCY on every rank if camera/frame
 * digests differ. */
DPR_API int dpr_render_frame(dpr_device dev);

/* LOOPBACK only: one collective render over all virtual ranks of the group. */
DPR_API int dpr_render_frame_group(dpr_device *devs, int n);

/* COLLECTIVE: the contrast device of P:534-647 (S5.1 ANARI-Composite): every rank renders
 * ONLY its local parts (local shading: no cross-rank shadows/AO/bounces) into colour +
 * depth buffers (depth = min over samples of the primary hit distance), then deep
 * compositing: parallel direct send of RGBA-z fragments so rank r receives all ranks'
 * fragments of its pixel span [r*S, (r+1)*S), S = ceil(W*H/N); per pixel sort by depth (ties:
 * lower rank) and composite front to back with "over" on premultiplied colour, background
 * last; spans gathered to rank 0 (P:568-582 S5.1.1).  dpr_map_frame then returns this image. */
DPR_API int dpr_render_frame_composite(dpr_device dev);
DPR_API int dpr_render_frame_composite_group(dpr_device *devs, int n);  /* loopback */

/* COLLECTIVE: Barney's data-REPLICATED mode: every rank has committed
 * the WHOLE world; pixel p is rendered only by rank (p*N)/(W*H) against its local copy (no
 * forwarding), and the disjoint framebuffers (and P13 dumps) are summed to rank 0.  The image
 * equals the data-parallel render of the same world. */
DPR_API int dpr_render_frame_replicated(dpr_device dev);
DPR_API int dpr_render_frame_replicated_group(dpr_device *devs, int n);  /* loopback */

/* LOCAL: 1 if the last render completed (renders are synchronous; wait is ignored). */
DPR_API int dpr_frame_ready(dpr_device dev, int wait);

/* LOCAL: rank 0 gets a DEVICE pointer to float RGBA [H][W] (bottom-left
 * origin; rgb = radiance/spp, a = coverage), valid until the next render or release.
 * Other ranks get *rgba=NULL, *w=*h=0, *undefined=1 and DPR_OK ("undefined ... not an
 * error"). */
DPR_API int dpr_map_frame(dpr_device dev, const float **rgba, int *w, int *h, int *undefined);

/* LOCAL, rank 0, frames rendered with DPR_FLAG_DEBUG_DUMPS: DEVICE pointers to the P13
 * dumps events[spp][max_depth][H*W] and occl[spp][max_depth][H*W] (uint32), valid until
 * the next render.  events: 0 not reached, 1 miss, 2+id surface, 0x80000000|i volume
 * sample i; occl: bit0 shadow unoccluded, bit(1+k) AO ray k unoccluded. */
DPR_API int dpr_get_debug(dpr_device dev, const uint32_t **events, const uint32_t **occl);

/* LOCAL: statistics of the last render (see dpr_stats). */
DPR_API int dpr_get_stats(dpr_device dev, dpr_stats *out);

/* LOCAL: per-step records of the last render (P8b lock-step steps, in order over all spp
 * batches; GLOBAL, gathered over all ranks).  For step k < min(*nsteps, max_steps):
 *   S_out[k][kind][src][dst]  rays forwarded / spawned src -> dst in step k (int64, N x N)
 *   V_out[k][kind][r]         traces (visits) at rank r in step k
 *   ms_out[k]                 step latency: max over ranks of the time from the step's start
 *                             to its completed step boundary (globaltimer, ms)
 *   sync_ms_out[k]            max over ranks of the time spent in the step barrier (device
 *                             loop with peers; 0 otherwise)
 * Any output may be NULL.  *nsteps = steps recorded (the last slot accumulates beyond 256). */
DPR_API int dpr_get_step_stats(dpr_device dev, int max_steps, int64_t *S_out, int64_t *V_out, double *ms_out,
                       double *sync_ms_out, int *nsteps);

/* LOCAL: last error message of this thread ("" if none). */
DPR_API const char *dpr_last_error(dpr_device dev);

/* LOCAL test of the step barrier of the device-driven loop (the mailbox protocol ranks use
 * over NVLink peer memory): nranks ranks emulated as the blocks of ONE cooperative kernel on
 * cuda_device (ranks that spin on each other must be co-resident), iters boundaries with
 * skewed arrival; *mismatches = boundaries whose gathered sums were wrong (0 expected). */
DPR_API int dpr_test_step_barrier(int cuda_device, int nranks, int iters, int64_t *mismatches);

/* LOCAL test of the LBVH builder's key sort (north star subsystem (1): "Morton codes, radix
 * sort"): the library's LSD radix passes (all four 8-bit digits, the default scatter kernel)
 * over n 32-bit keys.  keys, perm_out: DEVICE pointers on cuda_device (n elements each; the keys
 * are not modified).  perm_out[i] = index of the i-th key in ascending order, equal keys in
 * input order (stable), i.e. the order the build's Morton sort produces.  n >= 0; n > 2^30 or
 * NULL pointers with n > 0 -> DPR_ERR_INVALID_ARG.  Synchronous. */
DPR_API int dpr_test_radix_sort(int cuda_device, const uint32_t *keys, int64_t n, uint32_t *perm_out);

/* ---- host-side exchange planning (pure function; used by the render loop) ------------ */

/* Given the gathered per-destination counts of one ray kind, counts[src*nranks + dst]
 * (rays rank src queued for rank dst in this step, self entries included), compute THIS
 * rank's next input layout: [self-queued | from rank 0 | from rank 1 | ...] (skipping
 * self).  recv_offset[src] = first record index of src's rays; *total_in = next input
 * count; *global_total = sum over all entries (0 -> the wavefront loop is finished).
 * Returns DPR_ERR_QUEUE_OVERFLOW if *total_in > capacity, DPR_ERR_INVALID_ARG on bad
 * arguments.  Host memory only; needs no GPU. */
DPR_API int dpr_exchange_plan(int nranks, int rank, const int64_t *counts, int64_t capacity,
                      int64_t *recv_offset, int64_t *total_in, int64_t *global_total);

#ifdef __cplusplus
}
#endif
#endif /* DPR_H */
