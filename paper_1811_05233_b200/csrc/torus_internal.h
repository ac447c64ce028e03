// torus_internal.h -- layout and launch structures shared by the product's host code
// (torus_abi.cu) and kernels (torus_kernels.cu).  Not part of the public ABI.
//
// Notation follows PAPER.md:70: N = X * Y ranks, X per row (horizontal), Y per column
// (vertical); rank = rho * X + c (row rho, column c).
#pragma once
#include <cstddef>
#include <cstdint>

#include <cuda.h>  // driver-API types only (NVLS); the library does not link libcuda
#include <cuda_runtime.h>

namespace torus {

constexpr int kMaxRanks = 64;     // N <= 64 (a single NVLink domain has at most 72 GPUs)
constexpr int kMaxDim = 64;       // X, Y <= 64
constexpr int kMaxLocal = 16;     // virtual ranks per launch (single-GPU emulation)
constexpr int kThreads = 512;     // threads per CTA of the torus kernel
constexpr int kVecBytes = 16;     // 128-bit vectors (LDG/STG.E.128)
constexpr int kFlagPhases = 4;    // H-RS, V-RS, V-AG, H-AG handshakes
constexpr int kTraceIters = 64;   // trace: iterations recorded per CTA
constexpr int kTraceEvents = 8;   // trace: events per iteration (see torus_kernels.cu)

// Flag kinds (PAPER.md:70 phases; one u32 epoch per (kind, source, CTA)).
enum FlagKind : int {
  kFlagH = 0,   // row peer pushed its share of my chunk into my h_in        (phase 1)
  kFlagV = 1,   // column peer pushed its phase-1 result into my v_in        (phase 2 RS)
  kFlagAG = 2,  // column peer pushed its reduced sub-chunk into my chunk     (phase 2 AG)
  kFlagR = 3,   // row peer's chunk is complete: I may pull it                (phase 3)
};

// Workspace slab layout (identical on every rank; byte offsets from the slab base):
//   [0, flags_bytes)          flags[kind][src < kMaxDim][cta < G]  (u32 epochs)
//   [bar_off, +kMaxRanks*4)   barrier flags for init/destroy
//   [data_off, size)          data region, carved per call by wire type:
//        h_in[X][Lc]   (X > 1 only) shares of MY chunk pushed by each row peer
//        v_in[Y][Lcs]  phase-1 results of MY sub-chunk pushed by each column peer
//        chunk[Lc]     MY chunk, complete after phase 2 (pulled by row peers in phase 3)
//   [ll_off, +2*N*ll_slot)    small-message one-shot region (ll_kernel): [parity][src]
//                             slots of ll_slot bytes (0 when the LL path is disabled)
//   [pull_flag_off, data_off) pull-kernel per-tile flags (torus_pull.cu)
struct SlabLayout {
  size_t flags_bytes;
  size_t bar_off;
  size_t ll_off;
  size_t ll_slot;
  size_t ll_region;   // bytes of the LL region (two parity halves)
  size_t pull_flag_off;  // pull-kernel flag region (torus_pull.cu), up to kPullFlagBytes
  size_t data_off;
  size_t size;
};

// Per-(rank) static description, uploaded once at init (device memory).
struct RankDev {
  int rank, rho, c;
  int X, Y, N;
  int G;                         // CTAs per rank per launch
  char* ws[kMaxRanks];           // every rank's slab base as mapped in THIS process
  uint32_t* epoch;               // [G] local per-CTA call counters (device memory)
  uint32_t* bar_epoch;           // [1] barrier counter
  int* err;                      // host-mapped async error word
  uint32_t* ll_ctr;              // [2] one-shot kernel: epoch, CTAs done in the current call
  uint32_t* pull_ctr;            // [2] pull kernel: call epoch, CTAs done in the current call
};

// Per-launch (per-round) arguments, passed by value.
struct LaunchArgs {
  const RankDev* ranks;          // device array [nlocal]
  void* buf[kMaxLocal];          // user buffer of each local rank
  unsigned long long n;          // elements in this round
  unsigned long long buf_off;    // element offset of the round inside the user buffers
  unsigned long long hin_off, hin_stride;   // bytes (from slab base / between slots)
  unsigned long long vin_off, vin_stride;
  unsigned long long chunk_off;
  unsigned long long timeout_ns;
  int nlocal;
  int G;
  int q;                         // partition quantum in elements (16 B / sizeof(wire))
  int op;                        // 0 sum, 1 mean
  float inv_n;                   // f32(1/N)
  int aligned;                   // all user buffers 16-byte aligned -> vector path
  unsigned long long* trace;     // optional [G][kTraceIters][kTraceEvents] globaltimer stamps
  int T;                         // pipeline tiles per CTA slice (same on every rank)
  int tile_vecs;                 // vectors per tile piece
  int nbufs;                     // > 0: TMA-staged kernel with this many ring buffers
  // TMA kernel: per data CTA, the last tile each stage has completed (5 words, stride 8),
  // published at gpu scope for the signal CTA(s), and the signal lane's end-of-call ack
  uint32_t* done_local;          // [nlocal * G * 8]
  uint32_t* sig_ack;             // [nlocal * G]
  int nsig;                      // signal CTAs appended after the nlocal * G data CTAs
  int chunk_vecs;                // TMA kernel: vectors per ring buffer (a tile piece is
                                 // streamed through the ring in chunks of this size)
  int fence_early;               // default kernel: fence before releasing the next iteration
  unsigned long long ll_off, ll_slot;  // one-shot kernel region (SlabLayout)
  unsigned long long ll_half;    // bytes per parity half of the LL region
  int ll_two_shot;               // 1: ll2_kernel (two-shot) instead of ll_kernel
  unsigned poll_sleep;           // default kernel: ns of back-off between flag polls
  int sd1;                       // default kernel: stage distance 1 even with T > 1
  // NEXT-1 fused multi-tensor call: the "user buffer" of local rank l is the concatenation
  // of nseg tensors described by segs[l * nseg .. (l + 1) * nseg) (device memory, sorted by
  // offset); nseg == 0: buf[l] is one flat buffer
  const struct MultiSeg* segs;
  int nseg;
};

// one tensor of a fused multi-tensor call (device memory)
struct MultiSeg {
  void* ptr;
  unsigned long long count;   // elements
  unsigned long long offset;  // element offset of the tensor in the concatenation
};

// TMA kernel shared memory: nbufs ring buffers of one piece each (tile_vecs 16-byte wire
// vectors, or the same elements in the user dtype: `ratio` = sizeof(dtype)/sizeof(wire),
// at least 1) + 3 mbarriers per buffer
constexpr int kTmaSmemMax = 227 * 1024 - 2048;  // dynamic part; static smem needs the rest
inline int tma_buf_bytes(int tile_vecs, int ratio) { return tile_vecs * 16 * (ratio > 1 ? ratio : 1); }
inline int tma_smem_bytes(int nbufs, int tile_vecs, int ratio) {
  return nbufs * tma_buf_bytes(tile_vecs, ratio) + nbufs * 24;
}


// Nested quantum-aligned partition (SPEC.md:67-75 when q == 1).  Host and
// device use this one definition; the oracle has its own, independent one.
__host__ __device__ inline void qpart(unsigned long long n, int parts, int q, int i,
                                      unsigned long long* off, unsigned long long* len) {
  const unsigned long long Q = (n + q - 1) / q;
  const unsigned long long base = Q / parts, rem = Q % parts;
  const unsigned long long ui = (unsigned long long)i;
  const unsigned long long start = ui * base + (ui < rem ? ui : rem);
  const unsigned long long cnt = base + (ui < rem ? 1 : 0);
  unsigned long long a = start * q, b = (start + cnt) * q;
  if (a > n) a = n;
  if (b > n) b = n;
  *off = a;
  *len = b - a;
}

// Pipeline geometry for a round of n elements (host and device agree by construction):
// CTA b owns slice b of every sub-chunk; each slice is cut into T tiles of tile_vecs
// 16-byte vectors.  T is sized from the largest sub-chunk (qpart puts it first).
__host__ __device__ inline void tile_geometry(unsigned long long n, int X, int Y, int q, int G,
                                              int tile_vecs, int* T) {
  unsigned long long o, l0, s0;
  const int VE = q;  // the quantum is one 16-byte vector
  qpart(n, X, q, 0, &o, &l0);
  qpart(l0, Y, q, 0, &o, &s0);
  const unsigned long long nv = (s0 + VE - 1) / VE;
  const unsigned long long slice = (nv + G - 1) / G;
  unsigned long long t = (slice + tile_vecs - 1) / tile_vecs;
  *T = (int)(t < 1 ? 1 : t);
}

inline size_t flags_bytes_for(int G) {
  size_t b = (size_t)kFlagPhases * kMaxDim * (size_t)G * sizeof(uint32_t);
  return (b + 65535) & ~(size_t)65535;
}

// Multi-tensor table passed by value (kernel parameter space): up to kMultiMax tensors
// per launch (161 ResNet-50 tensors fit in two).
constexpr int kMultiMax = 96;
struct MultiTable {
  void* ptr[kMultiMax];
  unsigned long long count[kMultiMax];
  unsigned long long offset[kMultiMax];  // element offset in the staging buffer
};

// NVLS (multicast) state of one rank (torus_nvls.cu)
struct NvlsState {
  CUmemGenericAllocationHandle mem = 0;        // my physical staging memory
  CUmemGenericAllocationHandle mc_handle = 0;  // the multicast object
  CUdeviceptr uc = 0;                          // unicast view of my staging
  CUdeviceptr mc = 0;                          // multicast view (everyone's staging)
  size_t size = 0, gran = 0;
  CUdevice dev = 0;
  int export_fd = -1;
  bool have_mc = false, ready = false;
};
int nvls_prepare(int device, int rank, size_t bytes, int world, NvlsState* st, long long blob[2]);
int nvls_attach(NvlsState* st, const long long blob0[2]);
int nvls_bind(NvlsState* st);
void nvls_release(NvlsState* st);
cudaError_t launch_nvls(const RankDev* ranks, const NvlsState* st, void* buf, unsigned long long n,
                        unsigned long long buf_off, int dtype, int wire, int op, float inv_n, int G,
                        unsigned long long timeout_ns, cudaStream_t s);

// ---- launch wrappers implemented in torus_kernels.cu ----
cudaError_t launch_torus(const LaunchArgs& a, int dtype, int wire, bool cooperative,
                         cudaStream_t stream);
cudaError_t launch_castscale(void* buf, unsigned long long n, int dtype, int wire,
                             cudaStream_t stream);
bool castscale_use_tma();  // env TORUS_CS_KERNEL=tma: the TMA ring instead of the one-shot LDG/STG kernel
cudaError_t launch_castscale_tma(void* buf, unsigned long long n, int wire, cudaStream_t stream);
cudaError_t launch_barrier(const RankDev* ranks, int nlocal, unsigned long long bar_off,
                           unsigned long long timeout_ns, cudaStream_t stream);
int torus_kernel_max_ctas_per_sm(int dtype, int wire);
cudaError_t launch_ring(const LaunchArgs& a, int dtype, int wire, bool cooperative, cudaStream_t stream);
cudaError_t launch_hier(const LaunchArgs& a, int dtype, int wire, bool cooperative, cudaStream_t stream);
cudaError_t launch_ll(const LaunchArgs& a, int dtype, int wire, bool cooperative, cudaStream_t stream);
cudaError_t launch_multi_copy(const MultiTable& tab, int n, int dtype, int wire, void* staging,
                              bool pack, cudaStream_t stream);
cudaError_t launch_probe(const RankDev* ranks, unsigned long long data_off, unsigned long long bytes,
                         int mode, int iters, int ctas, unsigned long long* out, cudaStream_t stream);

}  // namespace torus
