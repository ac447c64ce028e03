/*
 * torus.h -- C-ABI of libtorus.so, the B200-native 2D-Torus all-reduce.
 *
 * Method (Sec. 2.2, Mikami et al., arXiv 1811.05233): the N = X*Y GPUs are
 * arranged in a 2D grid; "all-reduce consists of three steps: reduce-scatter, all-reduce,
 * and all-gather ... Firstly, reduce-scatter is performed horizontally. Then, all-reduce
 * is performed vertically. Finally, all-gather is performed horizontally."  The problem
 * it solves is the data-parallel step that must "synchronize and average gradients
 * across participating GPUs"; gradients are communicated in FP16
 * (PAPER.md:121).
 *
 * Ranks are row-major: rank = row * X + col, X = GPUs per row ("horizontal"),
 * Y = GPUs per column ("vertical")  (PAPER.md:70 defines X and Y; row-major is the
 * reading R1 in DESIGN.md).
 *
 * All functions return a torus_result_t (0 = TORUS_OK) unless stated.  No function
 * takes or returns a torch type; pointers are plain host or device pointers as stated.
 * Nothing here is thread-safe per comm; distinct comms may be used from distinct threads.
 */
#ifndef TORUS_H
#define TORUS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define TORUS_API __attribute__((visibility("default")))
#else
#define TORUS_API
#endif

#define TORUS_VERSION_MAJOR 0
#define TORUS_VERSION_MINOR 1

typedef struct torus_comm* torus_comm_t;
typedef void* torus_stream_t; /* a cudaStream_t (CUstream); NULL = the legacy default stream */

typedef enum { TORUS_F32 = 0, TORUS_F16 = 1, TORUS_BF16 = 2, TORUS_I32 = 3 } torus_dtype_t;
typedef enum { TORUS_SUM = 0, TORUS_MEAN = 1 } torus_op_t;

typedef enum {
    TORUS_OK = 0,
    TORUS_ERR_INVALID_ARG = 1, /* null pointer, bad enum, count overflow, misaligned buffer  */
    TORUS_ERR_GRID = 2,        /* X*Y != world, rank outside [0, world), grid too large     */
    TORUS_ERR_UNSUPPORTED = 3, /* e.g. wire wider than the buffer, i32 with a float wire     */
    TORUS_ERR_CUDA = 4,        /* an underlying CUDA call failed; see torus_last_error()     */
    TORUS_ERR_PEER = 5,        /* no P2P access to a peer, or IPC open failed                */
    TORUS_ERR_TIMEOUT = 6,     /* async: a device spin-wait exceeded its budget (watchdog)   */
    TORUS_ERR_MISMATCH = 7     /* peers disagree on the call (count/dtype/op/config)         */
} torus_result_t;

/* An exported workspace slab: the 64-byte cudaIpcMemHandle_t plus its size in bytes. */
typedef struct {
    unsigned char bytes[64];
    unsigned long long offset; /* always 0 in this version                                 */
    unsigned long long size;   /* slab size in bytes; must be equal on every rank          */
} torus_ipc_handle_t;

/* ---------------------------------------------------------------------------------------
 * Setup (multi-process: one process per GPU)
 * ------------------------------------------------------------------------------------- */

/* Allocate this rank's symmetric workspace slab on `device` (cudaMalloc, zeroed) and
 * export it for CUDA IPC.  `bytes` = 0 selects the default (env TORUS_WS_BYTES, else
 * 320 MiB), enough to reduce the 25.6M-element fp16 ResNet-50 buffer in a single round
 * on every grid.  The slab is owned by the library and adopted by the comm that
 * torus_comm_init builds from it; release it with torus_workspace_release only if no
 * comm was created.  out: host pointer, written on success. */
TORUS_API int torus_workspace_alloc(int device, size_t bytes, torus_ipc_handle_t* out);
TORUS_API int torus_workspace_release(const torus_ipc_handle_t* h);

/* Build this rank's communicator (collective in the sense that every rank must call it
 * with the same world, X, Y and the same handle array before any rank calls
 * torus_allreduce).  ipc_handles: host array [world] of every rank's exported slab, in
 * rank order (ipc_handles[rank] must be a slab this process allocated).  X = Y = 0 lets
 * the topology layer choose the grid (torus_pick_grid).  The handles are copied.
 * Uses the current CUDA device of the slab.  out: written on success. */
TORUS_API int torus_comm_init(int rank, int world, int X, int Y, const torus_ipc_handle_t* ipc_handles,
                    torus_comm_t* out);

/* Single-GPU emulation of a whole X*Y grid ("virtual ranks"): all N
 * ranks' workspaces live on `device` and one cooperative launch runs every rank's CTAs,
 * so the cross-rank flag protocol and the peer-pointer paths of the product kernel are
 * exercised without N GPUs.  ctas = CTAs per virtual rank (0 = auto, sized so all N*ctas
 * CTAs are co-resident); ws_bytes per rank (0 = default). */
TORUS_API int torus_vcomm_init(int device, int X, int Y, int ctas, size_t ws_bytes, torus_comm_t* out);

/* Collective teardown: waits for every collective this comm enqueued on any stream
 * (device synchronize), then a device barrier among all ranks (so no peer still reads
 * this rank's slab), then unmap peers, free the slab.  NULL is a no-op. */
TORUS_API int torus_comm_destroy(torus_comm_t comm);

/* Non-collective teardown for a comm whose peers never finished init (or are gone):
 * drains this rank's own work, frees its resources, no barrier.  NULL is a no-op. */
TORUS_API int torus_comm_abort(torus_comm_t comm);

/* Buffer registration (zero-copy): a collective promise that `ptr` (a device buffer of
 * `bytes` bytes on the comm's device) is the buffer every rank passes to later calls.
 * Step 1, local: torus_buffer_export(ptr, bytes, &h) -> h = the IPC handle of the
 * allocation containing ptr + ptr's offset in it.  Step 2: all-gather h over the ranks
 * (host side, e.g. torch.distributed).  Step 3: torus_register_buffer(comm, ptr, bytes,
 * handles[world]) maps every peer's buffer.  Afterwards calls whose buf == ptr (and
 * dtype == wire) let the pull kernel read the row peers' inputs straight from their
 * buffers (TMA over NVLink): no pre-pass copy into the slab (SURVEY 8(d) HBM table).
 * Ownership: the caller keeps ptr allocated until torus_deregister_buffer (peer mappings
 * are closed at destroy).  Errors: MISMATCH if sizes differ across ranks, PEER if a
 * mapping fails.  Every rank must register / deregister the same buffers in the same
 * order, and call with the registered buffer on every rank or on none. */
TORUS_API int torus_buffer_export(const void* ptr, size_t bytes, torus_ipc_handle_t* out);
TORUS_API int torus_register_buffer(torus_comm_t comm, void* ptr, size_t bytes,
                                    const torus_ipc_handle_t* handles /*[world]*/);
TORUS_API int torus_deregister_buffer(torus_comm_t comm, void* ptr);

/* Configuration fingerprint: writes up to n words that must be EQUAL on every
 * rank for the flag protocol to line up -- grid, CTA count, slab layout, routing
 * thresholds, kernel choice and tiling knobs (all read from the environment once, at
 * init).  Returns the number of meaningful words (<= n) or a negative error.  The Python
 * binding all-gathers it right after init and fails with TORUS_ERR_MISMATCH if ranks
 * differ.  words: host array [n]. */
TORUS_API int torus_comm_config(torus_comm_t comm, unsigned long long* words, int n);

/* Which kernel a torus_allreduce_ex call with these arguments runs ("torus_pull_kernel",
 * "torus_kernel", "ll_kernel", "ll2_kernel", "castscale_kernel", "none"); a static
 * string.  The routing is a pure function of (count, dtype, wire) and the comm's
 * configuration, so it is the same on every rank. */
TORUS_API const char* torus_comm_route(torus_comm_t comm, size_t count, torus_dtype_t dtype,
                                       torus_dtype_t wire);

/* ---------------------------------------------------------------------------------------
 * The all-reduce
 * ------------------------------------------------------------------------------------- */

/* In-place all-reduce of `count` elements of `dtype` at device pointer `buf` (on the
 * comm's device), enqueued on `stream`; returns once enqueued (asynchronous, CUDA-graph
 * capturable: no host sync, no allocation).  Every rank must call it in the same order
 * with the same count, dtype and op.  Result on every rank: the
 * element-wise sum, or for TORUS_MEAN the sum times f32(1/N) rounded once (i32: the
 * wrapped sum / N truncated toward zero).  The wire type equals dtype.
 * count == 0: TORUS_OK, nothing enqueued.  buf must be element-aligned; 16-byte
 * alignment selects the 128-bit vector path.  The caller keeps buf valid until the
 * stream work completes.  Errors: INVALID_ARG / UNSUPPORTED before anything is
 * enqueued; CUDA if a launch fails; TIMEOUT is reported asynchronously.
 * Messages of at most torus_comm_ll_max_bytes() wire bytes take the one-shot
 * small-message kernel (every rank broadcasts, then folds locally in the same torus
 * order: the result is bit-identical to the multi-phase path); up to
 * torus_comm_ll2_max_bytes() the two-shot kernel (N >= 3); larger ones the
 * multi-phase kernel, in rounds of torus_comm_round_elems() elements. */
TORUS_API int torus_allreduce(torus_comm_t comm, void* buf, size_t count, torus_dtype_t dtype,
                    torus_op_t op, torus_stream_t stream);

/* As torus_allreduce with an explicit wire type ("the communication to
 * synchronize gradients [is] conducted in half precision float (FP16)" while LARS runs
 * in FP32).  Supported: wire == dtype, or dtype F32 with wire F16 / BF16: the f32 buffer
 * is cast to the wire type on the first read (round-to-nearest-even) and cast back on the
 * last write -- no separate pack/unpack kernels. */
TORUS_API int torus_allreduce_ex(torus_comm_t comm, void* buf, size_t count, torus_dtype_t dtype,
                       torus_dtype_t wire, torus_op_t op, torus_stream_t stream);

/* End-to-end all-reduce of a HOST buffer (PAPER.md:54's all-reduce of the gradients,
 * starting and ending in host memory): the `count` elements of `dtype` at host pointer
 * `host` are copied to the device buffer `dev` (>= count elements on the comm's device,
 * owned by the caller), all-reduced in place as torus_allreduce_ex(dev + k*piece, piece,
 * dtype, wire, op) for each piece k in order, and copied back to `host`.  The three steps
 * are pipelined over the pieces on two internal copy streams (piece k+1 travels host ->
 * device and piece k-1 device -> host while piece k is reduced); `stream` is forked at the
 * call and joined after the last copy, so work queued on `stream` afterwards sees the
 * result in `host` once the stream reaches it.  piece == 0 or >= count: one piece.
 * `host` should be pinned (cudaHostAlloc / cudaHostRegister): pageable memory works but
 * its copies do not overlap.  The result equals torus_allreduce_ex on each piece, bit for
 * bit (each piece is its own message: its own partition and fold order).
 * Every rank must call it with the same count, piece, dtype, wire and op.
 * Not for virtual comms (INVALID_ARG); not capturable in a CUDA graph.  Errors as
 * torus_allreduce_ex, plus CUDA for a failed copy or event. */
TORUS_API int torus_allreduce_host(torus_comm_t comm, void* host, void* dev, size_t count, size_t piece,
                                   torus_dtype_t dtype, torus_dtype_t wire, torus_op_t op,
                                   torus_stream_t stream);

/* Virtual-rank variant (comm from torus_vcomm_init): bufs is a HOST array [N] of device
 * pointers, one buffer per virtual rank, all on the comm's device. */
TORUS_API int torus_vallreduce(torus_comm_t comm, void* const* bufs, size_t count, torus_dtype_t dtype,
                     torus_dtype_t wire, torus_op_t op, torus_stream_t stream);

/* Bucketed multi-tensor all-reduce (NEXT-1, BASELINE.json config 5: "layer-bucketed
 * ResNet-50 gradients (161 tensors fused into buckets) fp16 with fused cast/scale").
 * ptrs / counts: HOST arrays [ntensors] of device pointers and element counts.  The
 * result equals torus_allreduce_ex on the concatenation of the tensors (same partition,
 * fold order and rounding).  When the concatenation takes the multi-phase route the call
 * is FUSED: the kernel reads the tensors through a device table of (pointer, count,
 * offset) with the dtype -> wire cast fused into its first read, and writes them back with
 * the up-cast fused into its last write -- no staging buffer, no pack / unpack kernels.
 * The first call with a new bucket (pointer list) uploads its table (allocates,
 * synchronizes); later calls with the same bucket are capturable.  Smaller buckets (the
 * one-shot / two-shot routes) pack into the comm's staging buffer, all-reduce it and
 * unpack (that buffer grows on first use; reserve it with torus_comm_reserve).
 * Concurrent buckets need one comm each, with CTA budgets that sum to at most the SM
 * count (spin-waiting kernels of different comms must co-reside). */
TORUS_API int torus_allreduce_multi(torus_comm_t comm, void* const* ptrs, const size_t* counts,
                                    int ntensors, torus_dtype_t dtype, torus_dtype_t wire,
                                    torus_op_t op, torus_stream_t stream);
TORUS_API int torus_comm_reserve(torus_comm_t comm, size_t staging_bytes);

/* Virtual-rank variant of the fused bucket call: ptrs is a HOST array [N * ntensors] of
 * device pointers, rank-major (rank r's tensor i at ptrs[r * ntensors + i]); counts
 * [ntensors] is shared.  Only the multi-phase route (UNSUPPORTED otherwise). */
TORUS_API int torus_vallreduce_multi(torus_comm_t comm, void* const* ptrs, const size_t* counts,
                                     int ntensors, torus_dtype_t dtype, torus_dtype_t wire,
                                     torus_op_t op, torus_stream_t stream);

/* Flat ring all-reduce over the rank ring 0 -> 1 -> ... -> N-1 -> 0 -- the BASELINE the
 * torus replaces ("Ring all-reduce scheme executes 2(N-1) GPU-to-GPU
 * operations", ref [14]).  N-1 reduce-scatter then N-1 all-gather steps, each a push
 * to the next rank; every message is rounded to the wire type (HOP policy),
 * the mean is applied once by the chunk's owner.  Same comm, arguments, ownership and
 * errors as torus_allreduce_ex; rounds of torus_comm_ring_round_elems() elements. */
TORUS_API int torus_ring_allreduce(torus_comm_t comm, void* buf, size_t count, torus_dtype_t dtype,
                                   torus_dtype_t wire, torus_op_t op, torus_stream_t stream);
TORUS_API int torus_vring_allreduce(torus_comm_t comm, void* const* bufs, size_t count,
                                    torus_dtype_t dtype, torus_dtype_t wire, torus_op_t op,
                                    torus_stream_t stream);
TORUS_API size_t torus_comm_ring_round_elems(torus_comm_t comm, torus_dtype_t wire);

/* Hierarchical all-reduce [6] -- the other baseline the paper compares against
 * ("the hierarchical all-reduce also does the same amount of GPU-to-GPU
 * operation as the 2D-Torus all-reduce, [but] the data size of the second step ... is X
 * times" larger).  Per row of X ranks a chain reduce of the FULL buffer to column 0, a
 * ring all-reduce of the full buffer among the Y leaders, a chain broadcast back (SPEC.md
 * 234-242); HOP rounding; mean applied once.  Same conventions as torus_ring_allreduce;
 * rounds of torus_comm_hier_round_elems() elements. */
TORUS_API int torus_hier_allreduce(torus_comm_t comm, void* buf, size_t count, torus_dtype_t dtype,
                                   torus_dtype_t wire, torus_op_t op, torus_stream_t stream);
TORUS_API int torus_vhier_allreduce(torus_comm_t comm, void* const* bufs, size_t count,
                                    torus_dtype_t dtype, torus_dtype_t wire, torus_op_t op,
                                    torus_stream_t stream);
TORUS_API size_t torus_comm_hier_round_elems(torus_comm_t comm, torus_dtype_t wire);

/* NVLS variant (NEXT-4): all-reduce with NVLink-SHARP in-switch reduction over ALL ranks
 * (multimem.ld_reduce with f32 accumulation + multimem.st on a multicast object), per GPU
 * about (N+1)/N*S bytes each way instead of 2(N-1)/N*S.  The switch's summation order is
 * unspecified: results match the oracle within the float tolerance, not bit for bit.
 * Wires f16 / bf16 / f32 (no i32).  Setup is collective and takes two host exchanges:
 *   prepare(bytes) -> blob[2] (rank 0: {pid, fd} of the exported multicast object)
 *   all ranks: attach(blob of rank 0)  -- imports the fd (pidfd_getfd), adds the device
 *   barrier; all ranks: bind()         -- binds the staging memory, maps the multicast VA
 *   barrier; then torus_nvls_allreduce.  `bytes` = staging per rank (rounds above it). */
TORUS_API int torus_nvls_prepare(torus_comm_t comm, size_t bytes, long long* blob /*[2]*/);
TORUS_API int torus_nvls_attach(torus_comm_t comm, const long long* blob0 /*[2]*/);
TORUS_API int torus_nvls_bind(torus_comm_t comm);
TORUS_API int torus_nvls_allreduce(torus_comm_t comm, void* buf, size_t count, torus_dtype_t dtype,
                                   torus_dtype_t wire, torus_op_t op, torus_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * Queries, topology, host logic, errors
 * ------------------------------------------------------------------------------------- */

/* Async error word written by the device watchdog (TORUS_ERR_TIMEOUT) -- readable without
 * synchronizing; 0 when healthy.  A comm that reported an async error must be destroyed. */
TORUS_API int torus_comm_get_async_error(torus_comm_t comm);

TORUS_API int torus_comm_grid(torus_comm_t comm, int* X, int* Y);  /* host out-pointers */
TORUS_API int torus_comm_rank(torus_comm_t comm, int* rank, int* world);
TORUS_API int torus_comm_ctas(torus_comm_t comm);                  /* CTAs per rank per launch, or -1 */

/* Elements per round for a wire type: calls longer than this run as consecutive rounds
 * (one kernel launch each), each partitioned independently.  0 on error. */
TORUS_API size_t torus_comm_round_elems(torus_comm_t comm, torus_dtype_t wire);

/* Small-message threshold: calls with count * sizeof(wire) <= this many bytes run the
 * one-shot kernel (NEXT-2; the latency term of PAPER.md:68).  Set at
 * init from env TORUS_LL_MAX_BYTES (default 6 MiB at N = 2, 1.5 MiB / (N-1) at N >= 3;
 * 0 disables) -- it must be the same on every rank, like the grid.  0 if disabled or
 * comm is NULL.  The region it needs, 4 * N * threshold bytes, comes out of the slab
 * (both LL paths are disabled if their region would exceed a quarter of it). */
TORUS_API size_t torus_comm_ll_max_bytes(torus_comm_t comm);

/* Mid-size threshold (N >= 3): calls above the one-shot threshold and up to this many
 * wire bytes run the two-shot kernel -- each rank sends every sub-chunk C_{c,s} to its
 * torus owner (s, c), the owner folds it in the torus order and broadcasts it back;
 * bit-identical to the multi-phase path.  Env TORUS_LL2_MAX_BYTES (default 4 MiB at
 * N >= 3; 0 disables; same on every rank); needs ~8x that many bytes of slab region.
 * 0 if disabled, N < 3 or comm is NULL. */
TORUS_API size_t torus_comm_ll2_max_bytes(torus_comm_t comm);

/* Kernel launches one torus_allreduce_ex call with these arguments enqueues (0 for
 * count == 0 or a no-op N == 1 call).  Returns -1 on invalid arguments. */
TORUS_API int torus_comm_launches(torus_comm_t comm, size_t count, torus_dtype_t dtype,
                        torus_dtype_t wire);

/* Topology layer (north_star (3); SPEC.md:303-311 costmodel): an
 * alpha-beta model predicts the time of an all-reduce of `bytes` on an X-by-Y grid
 * (ranks row-major, rows = horizontal groups) and the grid with the smallest prediction
 * wins.
 *   algo 0 torus, 1 flat ring, 2 hierarchical [6].
 *   schedule 0: the paper's ring phases, sum over phases of steps * (alpha + step bytes /
 *     beta): 2(X-1) horizontal steps of S/X, 2(Y-1) vertical steps of S/(XY);
 *   schedule 1: this library's one-shot phases (one dependent hand-off per phase, every
 *     peer of the phase at once): 2 * (alpha + (X-1)/X*S/beta_h) + 2 * (alpha +
 *     (Y-1)/Y*S/X/beta_v).
 * beta of a phase = the slowest link inside its row (or column) groups, from bw_gbs, a host
 * row-major [X*Y*X*Y] matrix of GB/s (0 = no P2P path: that grid is infeasible); bw_gbs
 * NULL = every link beta_default_gbs.  alpha_us: one hand-off in microseconds.  Result in
 * *out_us (host).  Errors: INVALID_ARG, GRID (infeasible grid). */
TORUS_API int torus_predict_time(int X, int Y, double bytes, double alpha_us, const double* bw_gbs,
                                 double beta_default_gbs, int algo, int schedule, double* out_us);

/* Choose the grid for `world` ranks: every factorization X*Y = world is predicted with the
 * schedule-1 model above and the fastest wins (ties: the larger X, i.e. fewer vertical
 * hand-offs).  Writes X, Y and, if pred_us is not NULL, the prediction. */
TORUS_API int torus_pick_grid_model(int world, const double* bw_gbs, double alpha_us,
                                    double beta_default_gbs, double bytes, int* X, int* Y,
                                    double* pred_us);

/* Topology discovery for torus_comm_init(X = Y = 0): p2p = host row-major [world*world]
 * relative link bandwidths (1 = one NVLink domain, 0 = no P2P), or NULL to query the
 * CUDA driver (cudaDeviceCanAccessPeer + the P2P performance rank of devices 0..world-1);
 * the calibrated alpha (4 us per hand-off) and beta (560 GB/s per GPU)
 * and the 51.1 MB north-star message feed torus_pick_grid_model.  On one NVSwitch
 * domain every grid moves 2(N-1)/N*S bytes per rank and the widest grid has the fewest
 * hand-offs (X = N); GPUs that share no P2P domain end up in different rows. */
TORUS_API int torus_pick_grid(int world, const int* p2p, int* X, int* Y);

/* Host logic export (tests): the nested quantum-aligned partition used by every launch
 * (SURVEY C3): split n into `parts` ranges with quantum q.  off/len: host arrays
 * [parts]. */
TORUS_API int torus_partition(unsigned long long n, int parts, int q, unsigned long long* off,
                    unsigned long long* len);

/* Device trace (tracing subsystem): with env TORUS_TRACE=1 at init, every launch records
 * globaltimer stamps per CTA and pipeline iteration -- host array [ctas][64][8] u64
 * (events: 0 poll start, 1 poll done, 2 DONE synced, 3 READY arrived, 4 flags raised,
 * 5 worker READY passed, 6 worker data done).  Synchronizes the device.  UNSUPPORTED if
 * tracing is off. */
TORUS_API int torus_comm_trace(torus_comm_t comm, unsigned long long* host, size_t bytes);

/* Device trace of the last pull-kernel launch (TORUS_TRACE=1 at init): host array
 * [ctas][64][8] u64 globaltimer stamps, CTAs of all local ranks in launch order; per job
 * n < 63 of each CTA: 0 producer saw the inputs' flags, 1 operands landed in shared
 * memory, 2 consumers done, 3 flags raised, 4 bulk stores issued, 5 stores read the
 * shared memory; [63][0..1] = CTA start / end.  Also writes
 * the CTAs per rank and the split over the CTA kinds (S0, R, VR, VA, H, SIG).
 * Synchronizes the device. */
TORUS_API int torus_comm_pull_trace(torus_comm_t comm, unsigned long long* host, size_t bytes,
                                    int* ctas_per_rank, int* kinds /*[6]*/);

/* Calibration probes (not part of the all-reduce; SURVEY.md 8(d) "Calibration"), enqueued
 * on `stream` with `ctas` CTAs (0 = the comm's count).  mode 0: push `bytes` split over
 * the N-1 peers' slabs; 1: pull the same; 2: flag ping-pong between ranks 0 and 1,
 * `iters` round trips, elapsed ns written to *ns_out (host; the call then synchronizes);
 * 3: local slab-to-slab copy of `bytes`; 4 / 5: push / pull as 0 / 1 but with TMA bulk
 * copies (cp.async.bulk, 16 KiB, 8-deep shared-memory ring, one thread per CTA).  Overwrites the data region of the slabs: never
 * run concurrently with an all-reduce on the same comm. */
TORUS_API int torus_probe(torus_comm_t comm, int mode, size_t bytes, int iters, int ctas,
                          unsigned long long* ns_out, torus_stream_t stream);

/* Static string for a result code. */
TORUS_API const char* torus_strerror(int code);
/* Thread-local text of the last error raised in this thread (CUDA message included). */
TORUS_API const char* torus_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* TORUS_H */
