// torus_abi.cu -- host side of libtorus.so: the C-ABI declared in include/torus.h.
//
// Responsibilities: symmetric workspace slabs exported/opened through CUDA IPC, the
// communicator (grid, peer table, device epochs, async error word), argument
// validation, round splitting, the topology layer (grid choice) and kernel
// launches.  PyTorch never appears here; the Python binding passes plain pointers.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/torus.h"
#include "torus_internal.h"
#include "torus_ll128.h"
#include "torus_pull.h"

using namespace torus;

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char msg[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(msg, sizeof msg, fmt, ap);
  va_end(ap);
  g_last_error = std::string(torus_strerror(code)) + ": " + msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(TORUS_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

#define CU(call)                                         \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);  \
  } while (0)

size_t env_size(const char* name, size_t dflt) {
  const char* v = getenv(name);
  if (!v || !*v) return dflt;
  return (size_t)strtoull(v, nullptr, 10);
}

constexpr size_t kDefaultSlab = 512ull << 20;   // real ranks (f32 51M-element rounds fit)
constexpr size_t kDefaultVirtualSlab = 320ull << 20;  // per virtual rank (N slabs on one GPU)
constexpr size_t kPullTraceBytes = (size_t)kMaxLocal * 512 * kPullTraceJobs * kPullTraceEv * 8;
constexpr int kLLThreadsHost = 256;  // ll_kernel block size (torus_kernels.cu)

struct Slab {
  int device;
  void* ptr;
  size_t size;
  cudaIpcMemHandle_t handle;
};
std::mutex g_mu;
std::vector<Slab> g_slabs;  // exported, not yet adopted by a comm

size_t wire_size(int t) { return (t == TORUS_F16 || t == TORUS_BF16) ? 2 : 4; }
bool valid_dtype(int t) { return t >= TORUS_F32 && t <= TORUS_I32; }
bool valid_pair(int dtype, int wire) {
  if (!valid_dtype(dtype) || !valid_dtype(wire)) return false;
  if (dtype == wire) return true;
  return dtype == TORUS_F32 && (wire == TORUS_F16 || wire == TORUS_BF16);
}

}  // namespace

struct torus_comm {
  int rank = 0, world = 1, X = 1, Y = 1;
  int device = 0;
  int G = 0;
  int tile_vecs = 0;        // vectors per tile piece (env TORUS_TILE); 0 = auto
  bool tma = false;         // env TORUS_KERNEL=tma selects the TMA-staged kernel
  int nlocal = 1;           // > 1: virtual ranks on one device
  bool virt = false;
  size_t slab_size = 0;
  SlabLayout layout{};
  unsigned long long timeout_ns = 0;
  std::vector<void*> own_slabs;   // slabs this process allocated (freed at destroy)
  std::vector<void*> opened;      // IPC-opened peer bases (closed at destroy)
  std::vector<int> local_ranks;   // ranks hosted by this process
  RankDev* d_ranks = nullptr;     // device [nlocal]
  uint32_t* d_epochs = nullptr;   // device [nlocal * G] + [nlocal] barrier counters
  int* h_err = nullptr;           // host-mapped async error word
  int* d_err = nullptr;
  bool poisoned = false;
  unsigned long long* d_trace = nullptr;  // TORUS_TRACE=1: [G][kTraceIters][kTraceEvents]
  uint32_t* d_done_local = nullptr;       // TMA kernel: [nlocal][G][8] stage tiles done
  uint32_t* d_sig_ack = nullptr;          // TMA kernel: [nlocal][G] signal-lane acks
  void* d_staging = nullptr;              // multi-tensor staging buffer (wire type)
  size_t staging_bytes = 0;
  NvlsState nvls;                         // NVLS (multicast) variant, NEXT-4
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;  // torus_allreduce_host copy streams (lazy)
  cudaEvent_t ev_fork = nullptr, ev_h2d = nullptr, ev_red = nullptr, ev_d2h = nullptr;
  size_t ll2_max = 0;                     // two-shot LL up to this many wire bytes (N >= 3)
  // ---- knobs, read ONCE at init (they must agree across ranks: torus_comm_config) ----
  int mode = 3;                           // kModeLL128 (default) / kModePush / kModePull / kModeTma
  unsigned long long one_tile_max = 4096; // push kernel: single-tile threshold (vectors)
  unsigned long long mid_tiles = 1;       // push kernel: tiles per slice below it
  int fence_early = 0;                    // push kernel experiment
  unsigned poll_sleep = 64;               // push kernel poll back-off (ns)
  int pull_tv = 0;                        // pull kernel: vectors per tile (0 = auto)
  int pull_slots = 0;                     // pull kernel: shared-memory ring slots (0 = auto)
  int pull_ctas = 0;                      // pull kernel: CTA budget per rank (0 = all resident)
  int pull_fence = 0;                     // pull kernel publish fence (see PullArgs::fence)
  int pull_zc = 1;                        // pull kernel: zero-copy from registered buffers
  int ll128_ctas = 0;                     // LL128 kernel: CTAs per rank (0 = one per SM)
  float ll128_w[5] = {1.f, 1.f, 1.f, 1.f, 1.f};  // LL128 kernel: warp weight per stage
  int ll128_lane = 16;                    // LL128 kernel: bytes per lane per line store (16 / 32)
  int check = 0;                          // TORUS_CHECK=1: per-call header check (MISMATCH)
  int fault = 0;                          // TORUS_FAULT: negative-control fault injection (tests)
  unsigned delay_ns = 0;                  // TORUS_DELAY_NS: random per-CTA start delay (tests)
  unsigned call_seq = 0;                  // calls issued (header check sequence number)
  struct Reg {                            // a registered user buffer (torus_register_buffer)
    char* ptr;
    size_t bytes;
    bool aligned;                         // 16-byte aligned on every rank
    std::vector<char*> peer;              // every rank's buffer, mapped here
  };
  std::vector<Reg> regs;
  struct SegTable {                       // NEXT-1: device copy of a bucket's tensor table
    std::vector<MultiSeg> host;           // [nlocal * ntensors]
    MultiSeg* dev;
  };
  std::vector<SegTable> seg_tables;
  std::vector<std::pair<std::string, void*>> ipc_opened;  // IPC handle -> mapped base
  float pull_w[5] = {0.5f, 1.f, 1.f, 1.f, 1.f};  // pull kernel: CTA weight per kind
  uint32_t* d_pull_ctr = nullptr;         // [nlocal][2] pull call epochs
  unsigned long long* d_pull_trace = nullptr;  // TORUS_TRACE=1: pull kernel stamps
  int last_data_kernel = 0;               // kernel that last used the shared data region
  int last_pull_gsum = 0, last_pull_g[6] = {0, 0, 0, 0, 0, 0};  // CTA split of the last pull launch
  unsigned long long* d_pull_pub = nullptr;  // pull kernel fence mode 3: [nlocal * 1024] job counts
  int ctas_req = 0;                       // CTA count requested at init (0 = auto)
};

namespace {

enum { kModePull = 0, kModePush = 1, kModeTma = 2, kModeLL128 = 3 };
// kernels that share the slab's data region (a switch between them needs a barrier)
enum { kDataNone = 0, kDataPull = 1, kDataPush = 2, kDataRing = 3, kDataHier = 4, kDataLL128 = 5 };

size_t pull_flag_bytes(size_t slab_size) {
  size_t b = std::min<size_t>(kPullFlagBytes, slab_size / 16);
  b = std::max<size_t>(b, 65536);
  return (b + 65535) & ~(size_t)65535;
}

// ll_max: largest message (wire bytes per rank) for the one-shot small-message kernel;
// its region is dropped when it would take more than a quarter of the slab.
// ll2_max: largest message for the two-shot variant (N >= 3); per parity it needs 2N
// slots of two LL lines per vector of the largest sub-chunk, ~4 * ll2_max bytes.
SlabLayout make_layout(size_t slab_size, int G, int N, size_t ll_max, size_t ll2_max) {
  SlabLayout L;
  L.flags_bytes = flags_bytes_for(G);
  L.bar_off = L.flags_bytes;
  L.ll_off = L.bar_off + 65536;
  size_t slot = 2 * ((ll_max + 15) & ~(size_t)15);  // two LL lines per 16-byte vector
  size_t region = (N >= 2 && ll_max) ? 2 * (size_t)N * slot : 0;
  if (N >= 3 && ll2_max) region = std::max(region, 8 * ll2_max + 64 * (size_t)N * 32);
  region = (region + 65535) & ~(size_t)65535;
  if (region > slab_size / 4) region = slot = 0;
  L.ll_slot = region ? slot : 0;
  L.ll_region = region;
  L.pull_flag_off = L.ll_off + region;
  L.data_off = L.pull_flag_off + pull_flag_bytes(slab_size);
  L.size = slab_size;
  return L;
}

// Default threshold: the one-shot kernel moves 2(N-1) * S bytes per rank (LL lines, one
// copy per peer) against the multi-phase kernel's 2(N-1)/N * S plus four dependent
// hand-offs.  Measured on B200 (profiles/r01_ll_*, r01_single_tile_sizes.jsonl): it beats
// the multi-phase kernel (single-tile mode) up to ~6.5 MB at N = 2 and ~3.6 MB at N = 4,
// so at N = 2 the default is 6 MiB (a 48 MiB slab region).
// With N >= 3 the two-shot variant takes over above 1.5 MiB / (N-1) (512 KiB at N=4,
// where both take ~14 us) and runs up to 8 MiB (profiles/r01_ll2_*: 13-33 us from 256 KB
// to 4 MB at 2x2 vs NCCL's 21-43); at N = 2 it would move the same bytes as the one-shot.
size_t ll_max_env(int N) {
  size_t dflt = 0;
  if (N == 2) dflt = 6ull << 20;
  else if (N >= 3) dflt = ((3ull << 19) / (N - 1)) & ~(size_t)15;
  return env_size("TORUS_LL_MAX_BYTES", dflt);
}
// two-shot up to 4 MiB at N >= 3: above it the LL128 multi-phase kernel is faster (8 MB at
// 2x2: 45 us vs 58, profiles/r02_thresholds.txt)
size_t ll2_max_env(int N) { return env_size("TORUS_LL2_MAX_BYTES", N >= 3 ? (4ull << 20) : 0); }

// Round capacity for a wire type (elements): R = k * q * X * Y with
// h_in (X>1: X slots of R/X) + v_in (Y slots of R/(XY)) + chunk (R/X) in the data region.
unsigned long long round_elems(const torus_comm* c, int wire) {
  const unsigned long long sw = wire_size(wire), q = kVecBytes / sw;
  if (c->slab_size <= c->layout.data_off + 4096) return 0;
  const unsigned long long data_elems = (c->slab_size - c->layout.data_off - 4096) / sw;
  const unsigned long long X = (unsigned long long)c->X, Y = (unsigned long long)c->Y;
  // R = k * q * X * Y elements.
  // push kernel: h_in (X > 1: X slots of R/X) + v_in (Y slots of R/(XY)) + chunk (R/X)
  // pull kernel, per call parity: win (R) + P1 (R/X, if X > 1 and Y > 1) + chunk (R/X)
  unsigned long long per_k;
  if (c->mode == kModePull) {
    per_k = 2 * q * (X * Y + ((X > 1 && Y > 1) ? 2 : 1) * Y);
  } else if (c->mode == kModeLL128 && X * Y > 1) {
    // per parity: H and HAG inboxes (X > 1) R each, V and AG inboxes (Y > 1) R/X each, as
    // 128-byte lines holding 120 bytes (x 16/15) -- plus a 10% margin for stream padding
    const unsigned long long slots = (X > 1 ? 2 * X * Y : 0) + (Y > 1 ? 2 * Y : 0);
    per_k = (2 * q * slots * 16 * 11 + 149) / 150;
  } else {
    per_k = q * Y * ((X > 1 ? X : 0) + 2);
  }
  const unsigned long long k = data_elems / per_k;
  return k * q * X * Y;
}

// Pull-kernel slab regions for a round capacity R (identical on every rank).
struct PullLayout {
  unsigned long long win[2], p1[2], chunk[2];
};
PullLayout pull_layout(const torus_comm* c, unsigned long long R, unsigned long long sw) {
  const unsigned long long X = (unsigned long long)c->X, Y = (unsigned long long)c->Y;
  auto up = [](unsigned long long b) { return (b + 255) & ~255ull; };
  const unsigned long long win = up(R * sw + 64), lc = up((R / X) * sw + 64);
  PullLayout p;
  unsigned long long off = c->layout.data_off;
  for (int par = 0; par < 2; ++par) {
    p.win[par] = off;
    off += win;
    p.p1[par] = off;
    if (X > 1 && Y > 1) off += lc;
    p.chunk[par] = off;
    off += lc;
  }
  return p;
}

// Flat ring baseline: 2(N-1) slots of one chunk (R/N elements) per round.
unsigned long long ring_round_elems(const torus_comm* c, int wire) {
  const unsigned long long sw = wire_size(wire), q = kVecBytes / sw;
  const unsigned long long N = (unsigned long long)c->world;
  if (N < 2 || c->slab_size <= c->layout.data_off) return 0;
  const unsigned long long data_elems = (c->slab_size - c->layout.data_off) / sw;
  const unsigned long long k = data_elems / (2 * (N - 1) * q);
  return k * q * N;
}

// Hierarchical baseline: chain slot [R] + broadcast slot [R] + 2(Y-1) ring slots [R/Y].
unsigned long long hier_round_elems(const torus_comm* c, int wire) {
  const unsigned long long sw = wire_size(wire), q = kVecBytes / sw;
  const unsigned long long Y = (unsigned long long)c->Y;
  if (c->world < 2 || c->slab_size <= c->layout.data_off) return 0;
  const unsigned long long data_elems = (c->slab_size - c->layout.data_off) / sw;
  // R = k*q*Y:  2*R + 2(Y-1)*R/Y = k*q*(2Y + 2(Y-1)) elements
  const unsigned long long k = data_elems / (q * (2 * Y + 2 * (Y - 1)));
  return k * q * Y;
}

int alloc_comm_common(torus_comm* c) {
  const size_t n_ep = (size_t)c->nlocal * c->G + 5 * (size_t)c->nlocal;  // + barrier, ll[2], pull[2]
  CU(cudaMalloc(&c->d_epochs, n_ep * sizeof(uint32_t)));
  CU(cudaMemset(c->d_epochs, 0, n_ep * sizeof(uint32_t)));
  CU(cudaHostAlloc(&c->h_err, sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable));
  *c->h_err = 0;
  CU(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->d_err), c->h_err, 0));
  CU(cudaMalloc(&c->d_ranks, sizeof(RankDev) * c->nlocal));
  CU(cudaMalloc(&c->d_pull_pub, (size_t)c->nlocal * 1024 * sizeof(unsigned long long)));
  CU(cudaMemset(c->d_pull_pub, 0, (size_t)c->nlocal * 1024 * sizeof(unsigned long long)));
  {
    const size_t nd = (size_t)c->nlocal * c->G;
    CU(cudaMalloc(&c->d_done_local, nd * 8 * sizeof(uint32_t)));
    CU(cudaMemset(c->d_done_local, 0, nd * 8 * sizeof(uint32_t)));
    CU(cudaMalloc(&c->d_sig_ack, nd * sizeof(uint32_t)));
    CU(cudaMemset(c->d_sig_ack, 0, nd * sizeof(uint32_t)));
  }
  if (env_size("TORUS_TRACE", 0)) {
    const size_t tb = (size_t)c->G * kTraceIters * kTraceEvents * sizeof(unsigned long long);
    CU(cudaMalloc(&c->d_trace, tb));
    CU(cudaMemset(c->d_trace, 0, tb));
    CU(cudaMalloc(&c->d_pull_trace, kPullTraceBytes));
    CU(cudaMemset(c->d_pull_trace, 0, kPullTraceBytes));
  }
  return TORUS_OK;
}

int upload_ranks(torus_comm* c, const std::vector<char*>& bases) {
  std::vector<RankDev> rd(c->nlocal);
  for (int l = 0; l < c->nlocal; ++l) {
    RankDev& r = rd[l];
    memset(&r, 0, sizeof r);
    r.rank = c->local_ranks[l];
    r.X = c->X;
    r.Y = c->Y;
    r.N = c->X * c->Y;
    r.rho = r.rank / c->X;
    r.c = r.rank % c->X;
    r.G = c->G;
    for (int p = 0; p < c->world; ++p) r.ws[p] = bases[p];
    r.epoch = c->d_epochs + (size_t)l * c->G;
    r.bar_epoch = c->d_epochs + (size_t)c->nlocal * c->G + l;
    r.err = c->d_err;
    r.ll_ctr = c->d_epochs + (size_t)c->nlocal * (c->G + 1) + 2 * (size_t)l;
    r.pull_ctr = c->d_epochs + (size_t)c->nlocal * (c->G + 3) + 2 * (size_t)l;
  }
  CU(cudaMemcpy(c->d_ranks, rd.data(), sizeof(RankDev) * c->nlocal, cudaMemcpyHostToDevice));
  return TORUS_OK;
}

int pick_ctas(int device, int nlocal, int ctas_req) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  int per_sm = torus_kernel_max_ctas_per_sm(TORUS_F32, TORUS_F16);
  for (int d = 0; d < 4; ++d) per_sm = std::min(per_sm, torus_kernel_max_ctas_per_sm(d, d));
  if (per_sm < 1) per_sm = 1;
  const int resident = sms * per_sm;
  int want = ctas_req > 0 ? ctas_req : (int)env_size("TORUS_CTAS", nlocal > 1 ? 16 : sms * per_sm);
  want = std::max(1, want);
  // every CTA of every rank that waits on another must be co-resident
  // the TMA kernel appends one signal CTA on its own SM
  const char* k = getenv("TORUS_KERNEL");
  const int spare = (k && strcmp(k, "tma") == 0) ? 1 : 0;
  return std::min(want, std::max(1, (resident - spare) / nlocal));
}

// Knobs are read once, here; every rank must see the same values (torus_comm_config
// exposes them so the binding can check agreement at init).
void read_knobs(torus_comm* c) {
  c->timeout_ns = env_size("TORUS_TIMEOUT_MS", 30000) * 1000000ull;
  const char* k = getenv("TORUS_KERNEL");
  // default: the LL128 push kernel (fence-free flag-in-data lines; grids with X, Y <= 8) --
  // 100 us vs 120 (push kernel) and 124 (NCCL) at 1x2, 161 vs 175 and 161 at 2x2
  // (profiles/r02_ll128_*); TORUS_KERNEL=push / pull / tma select the others
  c->mode = kModeLL128;
  if (k && (strcmp(k, "push") == 0 || strcmp(k, "ldg") == 0)) c->mode = kModePush;
  if (k && strcmp(k, "pull") == 0) c->mode = kModePull;
  if (k && strcmp(k, "tma") == 0) c->mode = kModeTma;
  if (k && strcmp(k, "ll128") == 0) c->mode = kModeLL128;
  c->tma = c->mode == kModeTma;
  c->tile_vecs = (int)env_size("TORUS_TILE", 0);  // push kernel; 0 = auto (T ~ 3 tiles per slice)
  c->one_tile_max = env_size("TORUS_ONE_TILE_MAX", 4096);
  c->mid_tiles = std::max<size_t>(1, env_size("TORUS_MID_TILES", 1));
  c->fence_early = (int)env_size("TORUS_FENCE_EARLY", 0);
  c->poll_sleep = (unsigned)env_size("TORUS_POLL_SLEEP", 64);
  c->pull_tv = (int)env_size("TORUS_PULL_TILE", 0);
  c->pull_slots = (int)env_size("TORUS_PULL_SLOTS", 0);
  c->pull_ctas = (int)env_size("TORUS_PULL_CTAS", 0);
  c->pull_fence = (int)env_size("TORUS_PULL_FENCE", 3);
  c->pull_zc = (int)env_size("TORUS_PULL_ZC", 1);
  // LL128 CTAs (per device): TORUS_LL128_CTAS, else (one rank per process) the comm's CTA
  // budget TORUS_CTAS, set by TorusComm.init(ctas=...) so that concurrent comms' spinning
  // kernels co-reside, else all SMs
  c->ll128_ctas = (int)env_size("TORUS_LL128_CTAS", c->virt ? 0 : env_size("TORUS_CTAS", 0));
  c->ll128_lane = (int)env_size("TORUS_LL128_LANE", 16) == 32 ? 32 : 16;
  if (const char* w = getenv("TORUS_LL128_W"))
    sscanf(w, "%f,%f,%f,%f,%f", &c->ll128_w[0], &c->ll128_w[1], &c->ll128_w[2], &c->ll128_w[3], &c->ll128_w[4]);
  c->check = (int)env_size("TORUS_CHECK", 0);
  c->fault = (int)env_size("TORUS_FAULT", 0);
  c->delay_ns = (unsigned)env_size("TORUS_DELAY_NS", 0);
  if (const char* w = getenv("TORUS_PULL_W"))
    sscanf(w, "%f,%f,%f,%f,%f", &c->pull_w[0], &c->pull_w[1], &c->pull_w[2], &c->pull_w[3], &c->pull_w[4]);
  c->ll2_max = ll2_max_env(c->world);
}

void destroy_resources(torus_comm* c) {
  nvls_release(&c->nvls);
  for (cudaEvent_t e : {c->ev_fork, c->ev_h2d, c->ev_red, c->ev_d2h})
    if (e) cudaEventDestroy(e);
  if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
  if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
  for (void* p : c->opened) cudaIpcCloseMemHandle(p);
  for (auto& h : c->ipc_opened) cudaIpcCloseMemHandle(h.second);
  for (void* p : c->own_slabs) cudaFree(p);
  if (c->d_ranks) cudaFree(c->d_ranks);
  if (c->d_epochs) cudaFree(c->d_epochs);
  if (c->d_trace) cudaFree(c->d_trace);
  if (c->d_pull_trace) cudaFree(c->d_pull_trace);
  if (c->d_pull_pub) cudaFree(c->d_pull_pub);
  for (auto& t : c->seg_tables) cudaFree(t.dev);
  if (c->d_done_local) cudaFree(c->d_done_local);
  if (c->d_sig_ack) cudaFree(c->d_sig_ack);
  if (c->d_staging) cudaFree(c->d_staging);
  if (c->h_err) cudaFreeHost(c->h_err);
  delete c;
}

}  // namespace

extern "C" {

const char* torus_strerror(int code) {
  switch (code) {
    case TORUS_OK: return "TORUS_OK";
    case TORUS_ERR_INVALID_ARG: return "TORUS_ERR_INVALID_ARG";
    case TORUS_ERR_GRID: return "TORUS_ERR_GRID";
    case TORUS_ERR_UNSUPPORTED: return "TORUS_ERR_UNSUPPORTED";
    case TORUS_ERR_CUDA: return "TORUS_ERR_CUDA";
    case TORUS_ERR_PEER: return "TORUS_ERR_PEER";
    case TORUS_ERR_TIMEOUT: return "TORUS_ERR_TIMEOUT";
    case TORUS_ERR_MISMATCH: return "TORUS_ERR_MISMATCH";
    default: return "TORUS_ERR_UNKNOWN";
  }
}

const char* torus_last_error(void) { return g_last_error.c_str(); }

int torus_partition(unsigned long long n, int parts, int q, unsigned long long* off,
                    unsigned long long* len) {
  if (parts < 1 || q < 1 || !off || !len) return fail(TORUS_ERR_INVALID_ARG, "partition args");
  for (int i = 0; i < parts; ++i) qpart(n, parts, q, i, &off[i], &len[i]);
  return TORUS_OK;
}

int torus_workspace_alloc(int device, size_t bytes, torus_ipc_handle_t* out) {
  if (!out) return fail(TORUS_ERR_INVALID_ARG, "out is NULL");
  if (bytes == 0) bytes = env_size("TORUS_WS_BYTES", kDefaultSlab);
  bytes = (bytes + 65535) & ~(size_t)65535;
  CU(cudaSetDevice(device));
  void* p = nullptr;
  CU(cudaMalloc(&p, bytes));
  cudaError_t e = cudaMemset(p, 0, bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return cuda_fail(e, "workspace export");
  }
  memset(out, 0, sizeof *out);
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(out->bytes, &h, 64);
  out->offset = 0;
  out->size = bytes;
  std::lock_guard<std::mutex> g(g_mu);
  g_slabs.push_back(Slab{device, p, bytes, h});
  return TORUS_OK;
}

int torus_workspace_release(const torus_ipc_handle_t* h) {
  if (!h) return fail(TORUS_ERR_INVALID_ARG, "handle is NULL");
  std::lock_guard<std::mutex> g(g_mu);
  for (size_t i = 0; i < g_slabs.size(); ++i)
    if (memcmp(&g_slabs[i].handle, h->bytes, 64) == 0) {
      cudaSetDevice(g_slabs[i].device);
      cudaFree(g_slabs[i].ptr);
      g_slabs.erase(g_slabs.begin() + i);
      return TORUS_OK;
    }
  return fail(TORUS_ERR_INVALID_ARG, "no such local workspace");
}

}  // extern "C"

// ---------------------------------------------------------------------------------------
// Topology layer: an alpha-beta cost model picks the grid (SPEC.md:303-311 predict_time;
// the ring's cost grows with N "due to network latency", the torus
// replaces 2(N-1) sequential steps by 2(X-1) + 2(Y-1)).
//
// Phases of the X-by-Y torus (rows = ranks rho*X .. rho*X+X-1, columns = ranks i*X + c):
//   H-RS (X-1)/X*S  |  V-RS (Y-1)/Y*S/X  |  V-AG (Y-1)/Y*S/X  |  H-AG (X-1)/X*S   bytes per rank
// schedule 0 (the paper's / SPEC's ring phases): phase p costs steps_p * (alpha + S_p/beta_p),
//   steps = X-1, Y-1, Y-1, X-1 with per-step payloads S/X, S/(XY), S/(XY), S/X;
// schedule 1 (this library's kernels: one-shot phases, every peer at once over NVSwitch):
//   phase p costs alpha + bytes_p/beta_p -- one dependent hand-off per phase.
// beta_p = the slowest link inside the phase's groups (bw[i*world+j] in GB/s; 0 = no P2P
// path: the grid is infeasible).  Ring (algo 1): 2(N-1) steps of S/N on the ring's slowest
// link; hierarchical (algo 2): chain reduce (X-1 steps of S), Y-ring all-reduce on the
// full buffer (2(Y-1) steps of S/Y), chain broadcast (X-1 steps of S).
// ---------------------------------------------------------------------------------------
namespace {

double group_beta(int world, const double* bw, double dflt, const int* ranks, int n) {
  double b = dflt;
  if (!bw) return b;
  b = 1e300;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      if (i != j) b = std::min(b, bw[(size_t)ranks[i] * world + ranks[j]]);
  return n > 1 ? b : dflt;
}

// slowest link over all rows (horizontal) or all columns (vertical) of the grid
double dim_beta(int X, int Y, const double* bw, double dflt, bool rows) {
  const int world = X * Y;
  double b = 1e300;
  std::vector<int> g;
  if (rows) {
    for (int rho = 0; rho < Y; ++rho) {
      g.clear();
      for (int c = 0; c < X; ++c) g.push_back(rho * X + c);
      b = std::min(b, group_beta(world, bw, dflt, g.data(), X));
    }
  } else {
    for (int c = 0; c < X; ++c) {
      g.clear();
      for (int i = 0; i < Y; ++i) g.push_back(i * X + c);
      b = std::min(b, group_beta(world, bw, dflt, g.data(), Y));
    }
  }
  return b;
}

// predicted seconds (negative: infeasible)
double predict(int X, int Y, double S, double alpha, const double* bw, double beta_default, int algo,
               int schedule) {
  const int N = X * Y;
  const double bh = dim_beta(X, Y, bw, beta_default, true) * 1e9;   // bytes/s
  const double bv = dim_beta(X, Y, bw, beta_default, false) * 1e9;
  if (N == 1) return 0.0;
  if (algo == 1) {  // flat ring over ranks 0..N-1
    double b = beta_default * 1e9;
    if (bw) {
      b = 1e300;
      for (int r = 0; r < N; ++r) b = std::min(b, bw[(size_t)r * N + (r + 1) % N] * 1e9);
    }
    if (b <= 0) return -1;
    return 2.0 * (N - 1) * (alpha + S / N / b);
  }
  if ((X > 1 && bh <= 0) || (Y > 1 && bv <= 0)) return -1;
  double t = 0;
  if (algo == 2) {  // hierarchical [6]
    if (X > 1) t += 2.0 * (X - 1) * (alpha + S / bh);
    if (Y > 1) t += 2.0 * (Y - 1) * (alpha + S / Y / bv);
    return t;
  }
  if (schedule == 0) {
    if (X > 1) t += 2.0 * (X - 1) * (alpha + S / X / bh);
    if (Y > 1) t += 2.0 * (Y - 1) * (alpha + S / ((double)X * Y) / bv);
  } else {
    if (X > 1) t += 2.0 * (alpha + (double)(X - 1) / X * S / bh);
    if (Y > 1) t += 2.0 * (alpha + (double)(Y - 1) / Y * S / X / bv);
  }
  return t;
}

// Calibration of this library's kernels on B200 (profiles/r01_probe_*):
// one dependent hand-off = flag one-way ~2.5 us + a system fence ~1.5 us; per-GPU NVLink
// injection with every peer busy ~560 GB/s (SM stores) -- used when no measurement is given.
constexpr double kAlphaUs = 4.0;
constexpr double kBetaGBs = 560.0;

}  // namespace

extern "C" {

int torus_predict_time(int X, int Y, double bytes, double alpha_us, const double* bw_gbs,
                       double beta_default_gbs, int algo, int schedule, double* out_us) {
  // without a link matrix any grid of the paper's scale (Table 4: up to 4096 GPUs) is fine
  if (X < 1 || Y < 1 || (long long)X * Y > (bw_gbs ? kMaxRanks : (1 << 20)) || !out_us || bytes < 0 ||
      alpha_us < 0 || algo < 0 || algo > 2 ||
      schedule < 0 || schedule > 1 || (!bw_gbs && !(beta_default_gbs > 0)))
    return fail(TORUS_ERR_INVALID_ARG, "predict_time args");
  const double t = predict(X, Y, bytes, alpha_us * 1e-6, bw_gbs, beta_default_gbs, algo, schedule);
  if (t < 0) return fail(TORUS_ERR_GRID, "grid %dx%d has a pair without a P2P path", X, Y);
  *out_us = t * 1e6;
  return TORUS_OK;
}

int torus_pick_grid_model(int world, const double* bw_gbs, double alpha_us, double beta_default_gbs,
                          double bytes, int* X, int* Y, double* pred_us) {
  if (world < 1 || world > kMaxRanks || !X || !Y || alpha_us < 0 || bytes < 0 ||
      (!bw_gbs && !(beta_default_gbs > 0)))
    return fail(TORUS_ERR_INVALID_ARG, "pick_grid_model args");
  double best = -1;
  int bx = 0, by = 0;
  for (int x = world; x >= 1; --x) {  // ties: the wider grid (fewer vertical hand-offs) first
    if (world % x) continue;
    const int y = world / x;
    if (x > kMaxDim || y > kMaxDim) continue;
    const double t = predict(x, y, bytes, alpha_us * 1e-6, bw_gbs, beta_default_gbs, 0, 1);
    if (t < 0) continue;
    if (best < 0 || t < best * (1 - 1e-9)) {
      best = t;
      bx = x;
      by = y;
    }
  }
  if (best < 0) return fail(TORUS_ERR_GRID, "no feasible grid for %d ranks", world);
  *X = bx;
  *Y = by;
  if (pred_us) *pred_us = best * 1e6;
  return TORUS_OK;
}

int torus_pick_grid(int world, const int* p2p, int* X, int* Y) {
  if (world < 1 || world > kMaxRanks || !X || !Y) return fail(TORUS_ERR_INVALID_ARG, "pick_grid args");
  std::vector<double> bw((size_t)world * world, 0.0);
  if (p2p) {
    // relative link bandwidths; 0 = no P2P path: traffic stages through the host (or
    // another fabric), modelled as 1/20 of an NVLink domain's bandwidth
    for (size_t i = 0; i < bw.size(); ++i) bw[i] = p2p[i] > 0 ? kBetaGBs * p2p[i] : kBetaGBs / 20.0;
  } else {
    int ndev = 0;
    CU(cudaGetDeviceCount(&ndev));
    if (ndev < world) return fail(TORUS_ERR_GRID, "only %d visible devices for world %d", ndev, world);
    for (int i = 0; i < world; ++i)
      for (int j = 0; j < world; ++j) {
        int ok = (i == j);
        int rank = 0;
        if (i != j) {
          CU(cudaDeviceCanAccessPeer(&ok, i, j));
          if (ok) cudaDeviceGetP2PAttribute(&rank, cudaDevP2PAttrPerformanceRank, i, j);
        }
        // relative performance rank 0 = best; without P2P traffic would stage through the
        // host (modelled as 1/20 of NVLink)
        bw[(size_t)i * world + j] = ok ? kBetaGBs / (1.0 + rank) : kBetaGBs / 20.0;
      }
  }
  for (int i = 0; i < world; ++i) bw[(size_t)i * world + i] = kBetaGBs;
  // the north-star message (ResNet-50 gradients in fp16) sets the bandwidth/latency balance
  return torus_pick_grid_model(world, bw.data(), kAlphaUs, kBetaGBs, 51114064.0, X, Y, nullptr);
}


int torus_comm_init(int rank, int world, int X, int Y, const torus_ipc_handle_t* ipc_handles,
                    torus_comm_t* out) {
  if (!ipc_handles || !out) return fail(TORUS_ERR_INVALID_ARG, "null argument");
  if (world < 1 || world > kMaxRanks) return fail(TORUS_ERR_GRID, "world %d outside [1,%d]", world, kMaxRanks);
  if (rank < 0 || rank >= world) return fail(TORUS_ERR_GRID, "rank %d outside [0,%d)", rank, world);
  if (X == 0 && Y == 0) {
    int rc = torus_pick_grid(world, nullptr, &X, &Y);
    if (rc) return rc;
  }
  if (X < 1 || Y < 1 || X * Y != world || X > kMaxDim || Y > kMaxDim)
    return fail(TORUS_ERR_GRID, "grid %dx%d does not match world %d", X, Y, world);
  for (int r = 1; r < world; ++r)
    if (ipc_handles[r].size != ipc_handles[0].size)
      return fail(TORUS_ERR_MISMATCH, "slab sizes differ across ranks");

  Slab own{};
  {
    std::lock_guard<std::mutex> g(g_mu);
    size_t i = 0;
    for (; i < g_slabs.size(); ++i)
      if (memcmp(&g_slabs[i].handle, ipc_handles[rank].bytes, 64) == 0) break;
    if (i == g_slabs.size()) return fail(TORUS_ERR_INVALID_ARG, "ipc_handles[rank] is not a local slab");
    own = g_slabs[i];
    g_slabs.erase(g_slabs.begin() + i);
  }
  torus_comm* c = new torus_comm();
  c->rank = rank;
  c->world = world;
  c->X = X;
  c->Y = Y;
  c->device = own.device;
  c->nlocal = 1;
  c->local_ranks = {rank};
  c->slab_size = own.size;
  c->own_slabs.push_back(own.ptr);
  read_knobs(c);
  int rc = TORUS_OK;
  std::vector<char*> bases(world, nullptr);
  if (cudaSetDevice(c->device) != cudaSuccess) rc = fail(TORUS_ERR_CUDA, "cudaSetDevice");
  if (!rc) {
    c->G = pick_ctas(c->device, 1, 0);
    c->layout = make_layout(c->slab_size, c->G, world, ll_max_env(world), c->ll2_max);
    if (round_elems(c, TORUS_F32) == 0) rc = fail(TORUS_ERR_INVALID_ARG, "workspace too small");
  }
  for (int p = 0; !rc && p < world; ++p) {
    if (p == rank) {
      bases[p] = static_cast<char*>(own.ptr);
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, ipc_handles[p].bytes, 64);
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      rc = fail(TORUS_ERR_PEER, "cudaIpcOpenMemHandle(rank %d): %s", p, cudaGetErrorString(e));
      break;
    }
    c->opened.push_back(ptr);
    bases[p] = static_cast<char*>(ptr);
  }
  if (!rc) rc = alloc_comm_common(c);
  if (!rc) rc = upload_ranks(c, bases);
  if (rc) {
    destroy_resources(c);
    return rc;
  }
  *out = c;
  return TORUS_OK;
}

int torus_vcomm_init(int device, int X, int Y, int ctas, size_t ws_bytes, torus_comm_t* out) {
  if (!out) return fail(TORUS_ERR_INVALID_ARG, "out is NULL");
  if (X < 1 || Y < 1 || X > kMaxDim || Y > kMaxDim || X * Y > kMaxLocal)
    return fail(TORUS_ERR_GRID, "virtual grid %dx%d (at most %d ranks)", X, Y, kMaxLocal);
  CU(cudaSetDevice(device));
  int coop = 0;
  CU(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
  if (!coop) return fail(TORUS_ERR_UNSUPPORTED, "device lacks cooperative launch");
  torus_comm* c = new torus_comm();
  c->virt = true;
  c->X = X;
  c->Y = Y;
  c->world = X * Y;
  c->nlocal = X * Y;
  c->device = device;
  for (int r = 0; r < c->world; ++r) c->local_ranks.push_back(r);
  if (ws_bytes == 0) ws_bytes = env_size("TORUS_WS_BYTES", kDefaultVirtualSlab);
  c->slab_size = (ws_bytes + 65535) & ~(size_t)65535;
  read_knobs(c);
  c->ctas_req = ctas;
  c->G = pick_ctas(device, c->nlocal, ctas);
  c->layout = make_layout(c->slab_size, c->G, c->world, ll_max_env(c->world), c->ll2_max);
  int rc = TORUS_OK;
  if (round_elems(c, TORUS_F32) == 0) rc = fail(TORUS_ERR_INVALID_ARG, "workspace too small");
  std::vector<char*> bases(c->world, nullptr);
  for (int r = 0; !rc && r < c->world; ++r) {
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, c->slab_size);
    if (e == cudaSuccess) e = cudaMemset(p, 0, c->slab_size);
    if (e != cudaSuccess) {
      rc = cuda_fail(e, "virtual slab");
      break;
    }
    c->own_slabs.push_back(p);
    bases[r] = static_cast<char*>(p);
  }
  if (!rc) rc = alloc_comm_common(c);
  if (!rc) rc = upload_ranks(c, bases);
  if (!rc && cudaDeviceSynchronize() != cudaSuccess) rc = fail(TORUS_ERR_CUDA, "init sync");
  if (rc) {
    destroy_resources(c);
    return rc;
  }
  *out = c;
  return TORUS_OK;
}

int torus_comm_destroy(torus_comm_t c) {
  if (!c) return TORUS_OK;
  int rc = TORUS_OK;
  cudaSetDevice(c->device);
  // Every collective this comm enqueued -- on any stream -- must have finished before
  // the teardown barrier is launched: the barrier's own stream is not ordered after the
  // user's streams, and a 64-thread barrier CTA fits beside a running all-reduce (ADVICE
  // r1).  After the local drain, the barrier tells each rank that no peer still reads it.
  cudaError_t se = cudaDeviceSynchronize();
  if (se != cudaSuccess) rc = cuda_fail(se, "destroy: device synchronize");
  if (!rc && !c->poisoned && *c->h_err == 0 && c->world > 1) {
    cudaStream_t s;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess) {
      cudaError_t e = launch_barrier(c->d_ranks, c->nlocal, c->layout.bar_off, c->timeout_ns, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) rc = cuda_fail(e, "destroy barrier");
      cudaStreamDestroy(s);
    }
    if (*c->h_err) rc = fail(TORUS_ERR_TIMEOUT, "destroy barrier timed out");
  }
  destroy_resources(c);
  return rc;
}

int torus_comm_abort(torus_comm_t c) {
  if (!c) return TORUS_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();  // local work only; no collective barrier
  destroy_resources(c);
  return TORUS_OK;
}

int torus_comm_get_async_error(torus_comm_t c) {
  if (!c) return TORUS_ERR_INVALID_ARG;
  return *reinterpret_cast<volatile int*>(c->h_err);
}

int torus_comm_grid(torus_comm_t c, int* X, int* Y) {
  if (!c || !X || !Y) return fail(TORUS_ERR_INVALID_ARG, "null argument");
  *X = c->X;
  *Y = c->Y;
  return TORUS_OK;
}

int torus_comm_rank(torus_comm_t c, int* rank, int* world) {
  if (!c || !rank || !world) return fail(TORUS_ERR_INVALID_ARG, "null argument");
  *rank = c->rank;
  *world = c->world;
  return TORUS_OK;
}

int torus_comm_ctas(torus_comm_t c) { return c ? c->G : -1; }

int torus_comm_pull_trace(torus_comm_t c, unsigned long long* host, size_t bytes, int* ctas_per_rank,
                          int* kinds /*[6]*/) {
  if (!c || !host) return fail(TORUS_ERR_INVALID_ARG, "null argument");
  if (!c->d_pull_trace) return fail(TORUS_ERR_UNSUPPORTED, "tracing is off (set TORUS_TRACE=1 before init)");
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(host, c->d_pull_trace, std::min(bytes, kPullTraceBytes), cudaMemcpyDeviceToHost));
  if (ctas_per_rank) *ctas_per_rank = c->last_pull_gsum;
  if (kinds)
    for (int k = 0; k < 6; ++k) kinds[k] = c->last_pull_g[k];
  return TORUS_OK;
}

int torus_comm_trace(torus_comm_t c, unsigned long long* host, size_t bytes) {
  if (!c || !host) return fail(TORUS_ERR_INVALID_ARG, "null argument");
  if (!c->d_trace) return fail(TORUS_ERR_UNSUPPORTED, "tracing is off (set TORUS_TRACE=1 before init)");
  const size_t tb = (size_t)c->G * kTraceIters * kTraceEvents * sizeof(unsigned long long);
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(host, c->d_trace, std::min(bytes, tb), cudaMemcpyDeviceToHost));
  return TORUS_OK;
}

int torus_probe(torus_comm_t c, int mode, size_t bytes, int iters, int ctas, unsigned long long* ns_out,
                torus_stream_t stream) {
  if (!c || c->virt || mode < 0 || mode > 11) return fail(TORUS_ERR_INVALID_ARG, "probe args");
  const size_t room = c->slab_size - c->layout.data_off;
  if (mode != 2 && (bytes == 0 || (bytes / 16) * 16 * (size_t)(c->world + 1) > room))
    return fail(TORUS_ERR_INVALID_ARG, "probe bytes %zu exceed the slab", bytes);
  if (mode == 2 && c->world < 2) return fail(TORUS_ERR_INVALID_ARG, "ping-pong needs 2 ranks");
  unsigned long long* d_out = nullptr;
  if (ns_out) CU(cudaMalloc(&d_out, sizeof(unsigned long long)));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const unsigned long long off = mode == 2 ? c->layout.bar_off + 4096 : c->layout.data_off;
  cudaError_t e = launch_probe(c->d_ranks, off, bytes, mode, iters,
                               ctas > 0 ? ctas : c->G, d_out, s);
  if (e == cudaSuccess && ns_out && mode >= 6)
    e = cudaMemcpyAsync(d_out, static_cast<char*>(c->own_slabs[0]) + c->layout.bar_off + 8192, 8,
                        cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess && ns_out) e = cudaMemcpyAsync(ns_out, d_out, 8, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && ns_out) e = cudaStreamSynchronize(s);
  if (d_out) cudaFree(d_out);
  return e == cudaSuccess ? TORUS_OK : cuda_fail(e, "probe");
}

size_t torus_comm_round_elems(torus_comm_t c, torus_dtype_t wire) {
  if (!c || !valid_dtype(wire)) return 0;
  return (size_t)round_elems(c, wire);
}

size_t torus_comm_ll_max_bytes(torus_comm_t c) {
  return c ? c->layout.ll_slot / 2 : 0;
}

size_t torus_comm_ll2_max_bytes(torus_comm_t c) {
  return (c && c->world >= 3 && c->layout.ll_region) ? c->ll2_max : 0;
}

int torus_comm_launches(torus_comm_t c, size_t count, torus_dtype_t dtype, torus_dtype_t wire) {
  if (!c || !valid_pair(dtype, wire)) return -1;
  if (count == 0) return 0;
  if (c->world == 1) return dtype == wire ? 0 : 1;
  const unsigned long long R = round_elems(c, wire);
  if (R == 0) return -1;
  return (int)((count + R - 1) / R);
}

}  // extern "C"

namespace {

// ---- routing: which kernel serves a call (same decision on every rank) ----
enum Route { kRouteNone = 0, kRouteCast, kRouteLL, kRouteLL2, kRoutePull, kRoutePush, kRouteLL128 };
const char* route_name(int r) {
  switch (r) {
    case kRouteCast: return castscale_use_tma() ? "castscale_tma_kernel" : "castscale_kernel";
    case kRouteLL: return "ll_kernel";
    case kRouteLL2: return "ll2_kernel";
    case kRoutePull: return "torus_pull_kernel";
    case kRoutePush: return "torus_kernel";
    case kRouteLL128: return "torus_ll128_kernel";
    default: return "none";
  }
}

// Two-shot slot bytes for a message (0 if it does not fit the LL region).
unsigned long long ll2_slot(const torus_comm* c, size_t count, unsigned long long sw) {
  const int q = (int)(kVecBytes / sw);
  unsigned long long o, l0, s0;
  qpart(count, c->X, q, 0, &o, &l0);
  qpart(l0, c->Y, q, 0, &o, &s0);
  const unsigned long long slot = 2 * ((s0 * sw + kVecBytes - 1) / kVecBytes) * kVecBytes;
  return (2ull * c->world * slot <= c->layout.ll_region / 2) ? slot : 0;
}

// Pull kernel ring and tile (auto: 16 KiB wire tiles, a ring of >= 2 jobs' operands in
// <= ~100 KiB so two CTAs fit per SM).  TV decides tile boundaries and flag indices, so
// it depends only on values every rank shares (grid, dtypes, env).
void pull_ring(const torus_comm* c, int ratio, int* tv, int* ns) {
  const int need = std::max(c->X, c->Y);
  int n = c->pull_slots > 0 ? c->pull_slots : std::max(6, 2 * need);
  n = std::max(n, need + 1);
  int t = c->pull_tv;
  if (t <= 0) {
    t = 1024;
    while (t > 128 && (size_t)n * t * 16 * ratio > (100u << 10)) t /= 2;
  }
  *tv = t;
  *ns = n;
}

unsigned long long pull_kmax(unsigned long long n, int X, int Y, int q, int TV) {
  unsigned long long o, l0, s0;
  qpart(n, X, q, 0, &o, &l0);
  qpart(l0, Y, q, 0, &o, &s0);
  const unsigned long long nv = (s0 + q - 1) / q;
  return (nv + TV - 1) / TV;
}

bool pull_fits(const torus_comm* c, unsigned long long R, int wire, int dtype) {
  if (c->mode != kModePull || c->world < 2 || c->world > kMaxRanks || std::max(c->X, c->Y) > 32) return false;
  const unsigned long long sw = wire_size(wire);
  int tv, ns;
  pull_ring(c, (int)(wire_size(dtype) / sw), &tv, &ns);
  const unsigned long long K = pull_kmax(R, c->X, c->Y, (int)(kVecBytes / sw), tv);
  const unsigned long long X = c->X, Y = c->Y;
  const unsigned long long words = (std::max(X, Y) * Y + 2 * Y + X * Y) * K + kMaxRanks;
  return words * 4 <= c->layout.data_off - c->layout.pull_flag_off;
}

int plan_route(const torus_comm* c, size_t count, int dtype, int wire) {
  if (count == 0) return kRouteNone;
  if (c->world == 1) return dtype == wire ? kRouteNone : kRouteCast;
  const unsigned long long R = round_elems(c, wire), sw = wire_size(wire);
  if (count * sw <= c->layout.ll_slot / 2 && count <= R) return kRouteLL;
  if (c->world >= 3 && c->layout.ll_region && count * sw <= c->ll2_max && count <= R && ll2_slot(c, count, sw))
    return kRouteLL2;
  if (pull_fits(c, R, wire, dtype)) return kRoutePull;
  if (c->mode == kModeLL128 && c->X <= 8 && c->Y <= 8) return kRouteLL128;
  return kRoutePush;
}

// Serialise against the previous kernel of a different kind on the shared data region
// (a ring/hier/push/pull switch must not overwrite slots a slower peer still
// reads).  Every rank issues the same call sequence, so every rank inserts the barrier.
int switch_data_kernel(torus_comm* c, int kind, cudaStream_t stream) {
  if (c->last_data_kernel != kDataNone && c->last_data_kernel != kind) {
    cudaError_t e = launch_barrier(c->d_ranks, c->nlocal, c->layout.bar_off, c->timeout_ns, stream);
    if (e != cudaSuccess) return cuda_fail(e, "algorithm-switch barrier");
  }
  c->last_data_kernel = kind;
  return TORUS_OK;
}

// Zero-copy source table for a call: the peers' user buffers when the call's buffer is a
// registered one (every rank calls with its registered buffer: same decision everywhere),
// or -- virtual ranks -- the local buffers themselves.
bool pull_zero_copy(const torus_comm* c, void* const* bufs, size_t bytes, int dtype, int wire, bool aligned,
                    char** peer) {
  if (!c->pull_zc || dtype != wire) return false;
  if (c->virt) {
    if (!aligned) return false;
    for (int r = 0; r < c->world; ++r) peer[r] = static_cast<char*>(bufs[r]);
    return true;
  }
  for (const auto& g : c->regs)
    if (g.ptr == bufs[0] && bytes <= g.bytes && g.aligned) {
      for (int r = 0; r < c->world; ++r) peer[r] = g.peer[r];
      return true;
    }
  return false;
}

int launch_pull_rounds(torus_comm* c, void* const* bufs, size_t count, int dtype, int wire, int op,
                       bool aligned, cudaStream_t stream) {
  const unsigned long long R = round_elems(c, wire), sw = wire_size(wire);
  const int ratio = (int)(wire_size(dtype) / sw);
  PullArgs a;
  memset(&a, 0, sizeof a);
  a.ranks = c->d_ranks;
  for (int l = 0; l < c->nlocal; ++l) a.buf[l] = bufs[l];
  a.nlocal = c->nlocal;
  a.q = (int)(kVecBytes / sw);
  a.op = op;
  a.inv_n = 1.0f / (float)(c->X * c->Y);
  a.aligned = aligned ? 1 : 0;
  a.timeout_ns = c->timeout_ns;
  const PullLayout L = pull_layout(c, R, sw);
  for (int p = 0; p < 2; ++p) {
    a.win_off[p] = L.win[p];
    a.p1_off[p] = L.p1[p];
    a.chunk_off[p] = L.chunk[p];
  }
  if (L.chunk[1] + (R / c->X) * sw + 64 > c->slab_size) return fail(TORUS_ERR_INVALID_ARG, "pull layout overflow");
  a.flag_off = c->layout.pull_flag_off;
  int tv, ns;
  pull_ring(c, ratio, &tv, &ns);
  a.TV = tv;
  a.nslots = ns;
  a.slot_bytes = tv * 16 * ratio;
  // CTAs per kind, proportional to the bytes each kind moves (SURVEY 8(d) per-kernel
  // table); every CTA of every rank must be co-resident (they spin on each other)
  static int cached_smem = -1, cached_per_sm = 0;
  const int smem = (int)pull_smem_bytes(ns, a.slot_bytes);
  if (smem != cached_smem) {
    cached_per_sm = pull_ctas_per_sm((size_t)smem);
    cached_smem = smem;
  }
  if (cached_per_sm < 1) return fail(TORUS_ERR_UNSUPPORTED, "pull kernel does not fit an SM (%d B smem)", smem);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  int gtot = sms * cached_per_sm / c->nlocal;
  if (c->pull_ctas > 0) gtot = std::min(gtot, c->pull_ctas);
  const int X = c->X, Y = c->Y;
  a.zc = pull_zero_copy(c, bufs, count * wire_size(dtype), dtype, wire, aligned, a.peer_buf) ? 1 : 0;
  const bool own_copy = !(dtype == wire && aligned);  // S0 also copies my own chunk
  double w[6] = {0, 0, 0, 0, 0, 0};
  const double f0 = X > 1 ? (double)(X - 1) / X + (own_copy ? 1.0 / X : 0.0)
                          : (double)(Y - 1) / Y + (own_copy ? 1.0 / Y : 0.0);
  w[0] = a.zc ? 0.02 : c->pull_w[0] * f0 * ratio;  // zero-copy: S0 only copies ragged tails
  if (X > 1) w[1] = c->pull_w[1] * (double)(X - 1) / X;
  if (Y > 1) w[2] = c->pull_w[2] * (double)(Y - 1) / Y / X;
  if (Y > 1) w[3] = c->pull_w[3] * (double)(Y - 1) / Y / X;
  if (X > 1) w[4] = c->pull_w[4] * (double)(X - 1) / X;
  double wsum = 0;
  int kinds = 0;
  for (int k = 0; k < 5; ++k) {
    if (w[k] > 0) ++kinds;
    wsum += w[k];
  }
  if (gtot < kinds) return fail(TORUS_ERR_UNSUPPORTED, "pull kernel needs %d CTAs per rank, %d fit", kinds, gtot);
  // fence mode 3: SIG CTAs (one thread per data CTA, 192 threads, up to 4 each)
  const int nsig_ctas = c->pull_fence == 3 ? std::max(1, (gtot + 4 * 192 - 1) / (4 * 192)) : 0;
  gtot -= nsig_ctas;
  int gs = 0;
  for (int k = 0; k < 5; ++k) {
    a.g[k] = w[k] > 0 ? std::max(1, (int)(gtot * w[k] / wsum)) : 0;
    gs += a.g[k];
  }
  while (gs > gtot) {  // trim the largest kind
    int kb = 0;
    for (int k = 1; k < 5; ++k)
      if (a.g[k] > a.g[kb]) kb = k;
    --a.g[kb];
    --gs;
  }
  a.g[5] = nsig_ctas;
  a.gsum = gs + nsig_ctas;
  a.pub = c->d_pull_pub;
  c->last_pull_gsum = gs;
  for (int k = 0; k < 6; ++k) c->last_pull_g[k] = a.g[k];
  for (unsigned long long r0 = 0; r0 < count; r0 += R) {
    a.n = std::min<unsigned long long>(R, count - r0);
    a.buf_off = r0;
    for (int j = 0; j < X; ++j) {
      unsigned long long cl;
      qpart(a.n, X, a.q, j, &a.g_co[j], &cl);
      for (int s = 0; s < Y; ++s) {
        qpart(cl, Y, a.q, s, &a.g_cs[j * Y + s], &a.g_sl[j * Y + s]);
        const unsigned long long nv = (a.g_sl[j * Y + s] + a.q - 1) / a.q;
        a.g_K[j * Y + s] = (int)((nv + tv - 1) / tv);
      }
    }
    const unsigned long long K = pull_kmax(a.n, X, Y, a.q, tv);
    a.Kmax = (int)std::max<unsigned long long>(1, K);
    a.fl_win = 0;
    a.fl_p1 = (unsigned long long)std::max(X, Y) * Y * a.Kmax;
    a.fl_v = a.fl_p1 + (unsigned long long)Y * a.Kmax;
    a.fl_c = a.fl_v + (unsigned long long)Y * a.Kmax;
    a.fl_pres = a.fl_c + (unsigned long long)X * Y * a.Kmax;
    a.trace = c->d_pull_trace;
    a.fence = c->pull_fence;
    a.fault = c->fault;
    a.delay_ns = c->delay_ns;
    cudaError_t e = launch_pull(a, dtype, wire, c->virt, stream);
    if (e != cudaSuccess) return cuda_fail(e, "pull kernel launch");
  }
  return TORUS_OK;
}

int launch_ll128_rounds(torus_comm* c, void* const* bufs, size_t count, int dtype, int wire, int op,
                        bool aligned, cudaStream_t stream, const MultiSeg* segs = nullptr, int nseg = 0) {
  const unsigned long long R = round_elems(c, wire), sw = wire_size(wire);
  const int X = c->X, Y = c->Y, q = (int)(kVecBytes / sw);
  // 32-byte lanes (TORUS_LL128_LANE=32) for flat calls: 60 vectors per 1 KiB unit, 512-thread
  // CTAs; multi-tensor buckets keep 16-byte lanes (30 vectors per 512-byte unit, 1024 threads)
  const int lane_bytes = (nseg == 0 && c->ll128_lane == 32) ? 32 : 16;
  const unsigned long long UE = (lane_bytes == 32 ? 60ull : 30ull) * q;  // elements per unit
  const unsigned long long unit_bytes = lane_bytes == 32 ? 2ull * kL128Unit : (unsigned long long)kL128Unit;
  L128Args a;
  memset(&a, 0, sizeof a);
  a.ranks = c->d_ranks;
  for (int l = 0; l < c->nlocal; ++l) a.buf[l] = bufs[l];
  a.segs = segs;  // NEXT-1 fused multi-tensor call: the buffer is a concatenation of tensors
  a.nseg = nseg;
  a.nlocal = c->nlocal;
  a.op = op;
  a.inv_n = 1.0f / (float)(X * Y);
  a.aligned = aligned ? 1 : 0;
  a.timeout_ns = c->timeout_ns;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  a.ctas = std::max(1, (c->ll128_ctas > 0 ? std::min(c->ll128_ctas, sms) : sms) / c->nlocal);
  a.lane_bytes = lane_bytes;
  const int warps = a.ctas * (lane_bytes == 32 ? 16 : kL128CtaWarps);
  // warps per stage ~ each stage's loads + stores per unit x units (x TORUS_LL128_W)
  // (B with Y == 1 also pushes its final values to the X-1 row peers)
  double w[5] = {X > 1 ? 2.0 * (X - 1) * Y : 0, (double)Y * (X + (Y > 1 ? 1 : X)), Y > 1 ? 2.0 * Y + X - 1 : 0,
                 Y > 1 ? (double)(Y - 1) * (X + 1) : 0, X > 1 ? 2.0 * (X - 1) * Y : 0};
  // measured at 2x2 (profiles/r02_wsweep2_n4.txt, 3 interleaved repeats): 0.8 x the fold
  // stages B, C and 1.2 x the row all-gather E is 2% faster than the formula alone
  // (150.0 vs 152.9 us); at 1x2 the formula is best (profiles/r02_wsweep_n2.txt)
  if (X > 1 && Y > 1) {
    w[1] *= 0.8;
    w[2] *= 0.8;
    w[4] *= 1.2;
  }
  for (int k = 0; k < 5; ++k) w[k] *= c->ll128_w[k];
  double ws = 0;
  int present = 0;
  for (double v : w) {
    ws += v;
    present += v > 0;
  }
  if (warps < present) return fail(TORUS_ERR_UNSUPPORTED, "ll128 kernel: %d warps for %d stages", warps, present);
  int tot = 0;
  for (int k = 0; k < 5; ++k) {
    a.wk[k] = w[k] > 0 ? std::max(1, (int)(warps * w[k] / ws)) : 0;
    tot += a.wk[k];
  }
  while (tot > warps) {
    int kb = 0;
    for (int k = 1; k < 5; ++k)
      if (a.wk[k] > a.wk[kb]) kb = k;
    --a.wk[kb];
    --tot;
  }
  a.wsum = tot;
  int rc = switch_data_kernel(c, kDataLL128, stream);
  if (rc) return rc;
  for (unsigned long long r0 = 0; r0 < count; r0 += R) {
    a.n = std::min<unsigned long long>(R, count - r0);
    a.buf_off = r0;
    unsigned long long chunk_units_max = 0, umax = 0;
    for (int j = 0; j < X; ++j) {
      unsigned long long cl;
      qpart(a.n, X, q, j, &a.g_co[j], &cl);
      unsigned long long cu = 0;
      for (int s2 = 0; s2 < Y; ++s2) {
        const int js = j * Y + s2;
        qpart(cl, Y, q, s2, &a.g_cs[js], &a.g_sl[js]);
        a.g_U[js] = (int)((a.g_sl[js] + UE - 1) / UE);
        a.g_uoff[js] = (int)cu;
        cu += a.g_U[js];
        umax = std::max<unsigned long long>(umax, a.g_U[js]);
      }
      chunk_units_max = std::max(chunk_units_max, cu);
    }
    a.Umax = (int)umax;
    a.h_stride = a.hag_stride = chunk_units_max * unit_bytes;
    a.v_stride = a.ag_stride = umax * unit_bytes;
    unsigned long long off = c->layout.data_off;
    for (int p = 0; p < 2; ++p) {
      a.h_off[p] = off;
      off += X > 1 ? X * a.h_stride : 0;
      a.hag_off[p] = off;
      off += X > 1 ? X * a.hag_stride : 0;
      a.v_off[p] = off;
      off += Y > 1 ? Y * a.v_stride : 0;
      a.ag_off[p] = off;
      off += Y > 1 ? Y * a.ag_stride : 0;
    }
    if (off > c->slab_size) return fail(TORUS_ERR_INVALID_ARG, "ll128 layout overflow (%llu > %zu)", off, c->slab_size);
    cudaError_t e = launch_ll128(a, dtype, wire, c->virt, stream);
    if (e != cudaSuccess) return cuda_fail(e, "ll128 kernel launch");
  }
  return TORUS_OK;
}

int allreduce_impl(torus_comm* c, void* const* bufs, size_t count, int dtype, int wire, int op,
                   cudaStream_t stream, const MultiSeg* segs = nullptr, int nseg = 0) {
  if (!c) return fail(TORUS_ERR_INVALID_ARG, "comm is NULL");
  if (!valid_pair(dtype, wire))
    return valid_dtype(dtype) && valid_dtype(wire)
               ? fail(TORUS_ERR_UNSUPPORTED, "dtype %d with wire %d", dtype, wire)
               : fail(TORUS_ERR_INVALID_ARG, "bad dtype/wire code");
  if (op != TORUS_SUM && op != TORUS_MEAN) return fail(TORUS_ERR_INVALID_ARG, "bad op %d", op);
  if (c->poisoned || *reinterpret_cast<volatile int*>(c->h_err)) {
    c->poisoned = true;
    return fail(TORUS_ERR_TIMEOUT, "communicator has an async error; destroy it");
  }
  if (count == 0) return TORUS_OK;  // nothing enqueued; empty buffers may be NULL
  const size_t esz = wire_size(dtype);
  bool aligned = true;
  for (int l = 0; l < c->nlocal; ++l) {
    if (!bufs[l]) return fail(TORUS_ERR_INVALID_ARG, "buffer %d is NULL", l);
    const uintptr_t p = reinterpret_cast<uintptr_t>(bufs[l]);
    if (p % esz) return fail(TORUS_ERR_INVALID_ARG, "buffer %d not element-aligned", l);
    if (p % kVecBytes) aligned = false;
  }
  if (count > (size_t)1 << 48) return fail(TORUS_ERR_INVALID_ARG, "count overflow");
  const int route = plan_route(c, count, dtype, wire);
  if (route == kRouteNone) return TORUS_OK;  // sum/mean over one rank of wire values: identity
  if (c->check && c->world > 1) {
    // per-call header: every rank must make the same call
    unsigned desc = 2166136261u;
    const unsigned long long fields[] = {count, (unsigned long long)dtype, (unsigned long long)wire,
                                         (unsigned long long)op, (unsigned long long)route};
    for (unsigned long long f : fields)
      for (int i = 0; i < 8; ++i) desc = (desc ^ (unsigned)((f >> (8 * i)) & 0xff)) * 16777619u;
    cudaError_t e = launch_check(c->d_ranks, c->nlocal, c->layout.bar_off + 16384, ++c->call_seq, desc,
                                 c->timeout_ns, stream);
    if (e != cudaSuccess) return cuda_fail(e, "header check launch");
  }
  if (route == kRouteCast) {
    cudaError_t e = launch_castscale(bufs[0], count, dtype, wire, stream);
    return e == cudaSuccess ? TORUS_OK : cuda_fail(e, "castscale launch");
  }
  const unsigned long long R = round_elems(c, wire);
  const unsigned long long sw = wire_size(wire);
  if (route == kRoutePull) {
    int rc = switch_data_kernel(c, kDataPull, stream);
    if (rc) return rc;
    return launch_pull_rounds(c, bufs, count, dtype, wire, op, aligned, stream);
  }
  if (route == kRouteLL128) return launch_ll128_rounds(c, bufs, count, dtype, wire, op, aligned, stream, segs, nseg);
  LaunchArgs a;
  memset(&a, 0, sizeof a);
  a.ranks = c->d_ranks;
  for (int l = 0; l < c->nlocal; ++l) a.buf[l] = bufs[l];
  a.nlocal = c->nlocal;
  a.q = (int)(kVecBytes / sw);
  a.op = op;
  a.inv_n = 1.0f / (float)(c->X * c->Y);
  a.aligned = aligned ? 1 : 0;
  a.timeout_ns = c->timeout_ns;
  if (route == kRouteLL || route == kRouteLL2) {
    // small message: one-shot broadcast + local fold in the torus order, or mid-size:
    // two-shot LL (scatter to the torus owners, fold, broadcast back) -- NEXT-2
    a.n = count;
    a.buf_off = 0;
    a.ll_off = c->layout.ll_off;
    a.ll_slot = route == kRouteLL ? c->layout.ll_slot : ll2_slot(c, count, sw);
    a.ll_half = c->layout.ll_region / 2;
    a.ll_two_shot = route == kRouteLL2 ? 1 : 0;
    const unsigned long long nvec = (count * sw + kVecBytes - 1) / kVecBytes;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    // every CTA waits on peers' CTAs: keep the grid co-resident (2 per SM always fits)
    const int cap = std::max(1, (int)env_size("TORUS_LL_CTAS", 2 * sms) / c->nlocal);
    a.G = (int)std::min<unsigned long long>(cap, (nvec + kLLThreadsHost - 1) / kLLThreadsHost);
    cudaError_t e = launch_ll(a, dtype, wire, c->virt, stream);
    return e == cudaSuccess ? TORUS_OK : cuda_fail(e, route == kRouteLL ? "one-shot kernel launch"
                                                                         : "two-shot kernel launch");
  }
  // the push kernel (default; TORUS_KERNEL=tma: its TMA-staged variant)
  int rc = switch_data_kernel(c, kDataPush, stream);
  if (rc) return rc;
  a.segs = segs;  // NEXT-1 fused multi-tensor call: the buffer is a concatenation of tensors
  a.nseg = nseg;
  a.G = c->G;
  a.fence_early = c->fence_early;
  a.poll_sleep = c->poll_sleep;
  a.tile_vecs = c->tile_vecs;
  if (a.tile_vecs <= 0) {
    // auto: about kAutoTiles tiles per CTA slice of the largest sub-chunk (measured best
    // at 2 and 4 GPUs); small calls get one tile (latency mode)
    constexpr unsigned long long kAutoTiles = 3;
    unsigned long long o, l0, s0;
    qpart(std::min<unsigned long long>(R, count), c->X, (int)(kVecBytes / sw), 0, &o, &l0);
    qpart(l0, c->Y, (int)(kVecBytes / sw), 0, &o, &s0);
    const unsigned long long nv = (s0 * sw + kVecBytes - 1) / kVecBytes;
    const unsigned long long slice = (nv + c->G - 1) / c->G;
    // up to one_tile_max vectors per CTA slice the call is one tile (stage distance 1):
    // five latency-bound iterations beat ~11 pipelined ones (measured, r01_single_tile_sizes)
    if (slice <= c->one_tile_max) {
      a.tile_vecs = (int)std::max<unsigned long long>(1, (slice + c->mid_tiles - 1) / c->mid_tiles);
      a.sd1 = 1;
    } else {
      a.tile_vecs = (int)std::max<unsigned long long>(256, (slice + kAutoTiles - 1) / kAutoTiles);
    }
  }
  a.trace = c->d_trace;
  a.nbufs = 0;
  a.done_local = c->d_done_local;
  a.sig_ack = c->d_sig_ack;
  a.nsig = c->tma ? (c->nlocal * c->G + kThreads - 1) / kThreads : 0;
  if (c->tma && nseg) return fail(TORUS_ERR_UNSUPPORTED, "fused multi-tensor call on the TMA variant");
  if (c->tma) {
    // ring buffers of one chunk each (tile pieces stream through in chunks): the largest
    // job holds max(X,Y)+3 buffers at once -- keep room for a few so the producer runs
    // ahead; shrink the chunk until that fits
    const int ratio = (int)(wire_size(dtype) / sw);
    const int need = 3 * (std::max(c->X, c->Y) + 3) + 4;
    int cv = std::min(a.tile_vecs, 1024);
    while (cv > 32 && kTmaSmemMax / (tma_buf_bytes(cv, ratio) + 24) < need) cv /= 2;
    a.chunk_vecs = cv;
    a.nbufs = std::min(64, kTmaSmemMax / (tma_buf_bytes(cv, ratio) + 24));
    if (a.nbufs < need) return fail(TORUS_ERR_UNSUPPORTED, "grid %dx%d too large for the TMA ring", c->X, c->Y);
  }
  const unsigned long long Lc = R / c->X, Lcs = R / ((unsigned long long)c->X * c->Y);
  a.hin_off = c->layout.data_off;
  a.hin_stride = Lc * sw;
  a.vin_off = a.hin_off + (c->X > 1 ? (unsigned long long)c->X * a.hin_stride : 0);
  a.vin_stride = Lcs * sw;
  a.chunk_off = a.vin_off + (unsigned long long)c->Y * a.vin_stride;
  if (a.chunk_off + Lc * sw > c->slab_size) return fail(TORUS_ERR_INVALID_ARG, "layout overflow");
  for (unsigned long long r0 = 0; r0 < count; r0 += R) {
    a.n = std::min<unsigned long long>(R, count - r0);
    a.buf_off = r0;
    tile_geometry(a.n, c->X, c->Y, a.q, a.G, a.tile_vecs, &a.T);
    cudaError_t e = launch_torus(a, dtype, wire, c->virt, stream);
    if (e != cudaSuccess) return cuda_fail(e, "torus kernel launch");
  }
  return TORUS_OK;
}

}  // namespace

extern "C" {

int torus_allreduce_ex(torus_comm_t c, void* buf, size_t count, torus_dtype_t dtype,
                       torus_dtype_t wire, torus_op_t op, torus_stream_t stream) {
  if (c && c->virt) return fail(TORUS_ERR_INVALID_ARG, "virtual comm: use torus_vallreduce");
  void* bufs[1] = {buf};
  return allreduce_impl(c, bufs, count, dtype, wire, op, static_cast<cudaStream_t>(stream));
}

int torus_allreduce(torus_comm_t c, void* buf, size_t count, torus_dtype_t dtype, torus_op_t op,
                    torus_stream_t stream) {
  return torus_allreduce_ex(c, buf, count, dtype, dtype, op, stream);
}

int torus_allreduce_host(torus_comm_t c, void* host, void* dev, size_t count, size_t piece,
                         torus_dtype_t dtype, torus_dtype_t wire, torus_op_t op, torus_stream_t stream_) {
  if (!c || !host || !dev) return fail(TORUS_ERR_INVALID_ARG, "null argument");
  if (c->virt) return fail(TORUS_ERR_INVALID_ARG, "virtual comm: not supported by torus_allreduce_host");
  if (!valid_dtype(dtype)) return fail(TORUS_ERR_INVALID_ARG, "bad dtype code");
  if (count == 0) return TORUS_OK;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (!c->s_h2d) {  // lazily: two copy streams and the fork / join events
    cudaError_t e = cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking);
    for (cudaEvent_t* ev : {&c->ev_fork, &c->ev_h2d, &c->ev_red, &c->ev_d2h})
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, "torus_allreduce_host setup");
  }
  const size_t esz = wire_size(dtype);
  const size_t P = piece == 0 || piece > count ? count : piece;
  char* h = static_cast<char*>(host);
  char* d = static_cast<char*>(dev);
  // fork: both copy streams start after the work already queued on `stream`
  cudaError_t e = cudaEventRecord(c->ev_fork, stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(c->s_h2d, c->ev_fork, 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(c->s_d2h, c->ev_fork, 0);
  if (e != cudaSuccess) return cuda_fail(e, "torus_allreduce_host fork");
  // piece k: H2D on s_h2d -> all-reduce on `stream` -> D2H on s_d2h.  An event is re-recorded
  // every piece: a wait binds to the record that precedes it, so two events suffice.
  for (size_t off = 0; off < count; off += P) {
    const size_t n = std::min(P, count - off);
    e = cudaMemcpyAsync(d + off * esz, h + off * esz, n * esz, cudaMemcpyHostToDevice, c->s_h2d);
    if (e == cudaSuccess) e = cudaEventRecord(c->ev_h2d, c->s_h2d);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, c->ev_h2d, 0);
    if (e != cudaSuccess) return cuda_fail(e, "torus_allreduce_host H2D");
    void* bufs[1] = {d + off * esz};
    const int rc = allreduce_impl(c, bufs, n, dtype, wire, op, stream);
    if (rc) return rc;
    e = cudaEventRecord(c->ev_red, stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->s_d2h, c->ev_red, 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h + off * esz, d + off * esz, n * esz, cudaMemcpyDeviceToHost, c->s_d2h);
    if (e != cudaSuccess) return cuda_fail(e, "torus_allreduce_host D2H");
  }
  // join: `stream` continues after the last D2H (and the H2D stream has nothing left)
  e = cudaEventRecord(c->ev_d2h, c->s_d2h);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, c->ev_d2h, 0);
  return e == cudaSuccess ? TORUS_OK : cuda_fail(e, "torus_allreduce_host join");
}

int torus_vallreduce(torus_comm_t c, void* const* bufs, size_t count, torus_dtype_t dtype,
                     torus_dtype_t wire, torus_op_t op, torus_stream_t stream) {
  if (!c || !bufs) return fail(TORUS_ERR_INVALID_ARG, "null argument");
  if (!c->virt) return fail(TORUS_ERR_INVALID_ARG, "not a virtual comm");
  return allreduce_impl(c, bufs, count, dtype, wire, op, static_cast<cudaStream_t>(stream));
}

}  // extern "C"

namespace {

int baseline_impl(torus_comm* c, void* const* bufs, size_t count, int dtype, int wire, int op,
                  cudaStream_t stream, bool hier) {
  if (!c) return fail(TORUS_ERR_INVALID_ARG, "comm is NULL");
  if (!valid_pair(dtype, wire))
    return valid_dtype(dtype) && valid_dtype(wire)
               ? fail(TORUS_ERR_UNSUPPORTED, "dtype %d with wire %d", dtype, wire)
               : fail(TORUS_ERR_INVALID_ARG, "bad dtype/wire code");
  if (op != TORUS_SUM && op != TORUS_MEAN) return fail(TORUS_ERR_INVALID_ARG, "bad op %d", op);
  if (c->poisoned || *reinterpret_cast<volatile int*>(c->h_err)) {
    c->poisoned = true;
    return fail(TORUS_ERR_TIMEOUT, "communicator has an async error; destroy it");
  }
  if (count == 0) return TORUS_OK;
  const size_t esz = wire_size(dtype);
  bool aligned = true;
  for (int l = 0; l < c->nlocal; ++l) {
    if (!bufs[l]) return fail(TORUS_ERR_INVALID_ARG, "buffer %d is NULL", l);
    const uintptr_t p = reinterpret_cast<uintptr_t>(bufs[l]);
    if (p % esz) return fail(TORUS_ERR_INVALID_ARG, "buffer %d not element-aligned", l);
    if (p % kVecBytes) aligned = false;
  }
  if (c->world == 1) {
    if (dtype == wire) return TORUS_OK;
    cudaError_t e = launch_castscale(bufs[0], count, dtype, wire, stream);
    return e == cudaSuccess ? TORUS_OK : cuda_fail(e, "castscale launch");
  }
  const unsigned long long R = hier ? hier_round_elems(c, wire) : ring_round_elems(c, wire);
  const unsigned long long sw = wire_size(wire);
  if (R == 0) return fail(TORUS_ERR_INVALID_ARG, "workspace too small for the baseline");
  LaunchArgs a;
  memset(&a, 0, sizeof a);
  a.ranks = c->d_ranks;
  for (int l = 0; l < c->nlocal; ++l) a.buf[l] = bufs[l];
  a.nlocal = c->nlocal;
  a.G = c->G;
  a.q = (int)(kVecBytes / sw);
  a.op = op;
  a.inv_n = 1.0f / (float)c->world;
  a.aligned = aligned ? 1 : 0;
  a.timeout_ns = c->timeout_ns;
  a.hin_off = c->layout.data_off;
  if (hier) {
    a.hin_stride = R * sw;                                 // chain / broadcast slot
    a.vin_stride = (R / (unsigned long long)c->Y) * sw;     // leader-ring slot
  } else {
    a.hin_stride = (R / (unsigned long long)c->world) * sw;  // one ring chunk slot
  }
  int rc = switch_data_kernel(c, hier ? kDataHier : kDataRing, stream);
  if (rc) return rc;
  for (unsigned long long r0 = 0; r0 < count; r0 += R) {
    a.n = std::min<unsigned long long>(R, count - r0);
    a.buf_off = r0;
    cudaError_t e = hier ? launch_hier(a, dtype, wire, c->virt, stream)
                         : launch_ring(a, dtype, wire, c->virt, stream);
    if (e != cudaSuccess) return cuda_fail(e, "baseline kernel launch");
  }
  return TORUS_OK;
}

}  // namespace

extern "C" {

int torus_ring_allreduce(torus_comm_t c, void* buf, size_t count, torus_dtype_t dtype,
                         torus_dtype_t wire, torus_op_t op, torus_stream_t stream) {
  if (c && c->virt) return fail(TORUS_ERR_INVALID_ARG, "virtual comm: use torus_vring_allreduce");
  void* bufs[1] = {buf};
  return baseline_impl(c, bufs, count, dtype, wire, op, static_cast<cudaStream_t>(stream), false);
}

int torus_vring_allreduce(torus_comm_t c, void* const* bufs, size_t count, torus_dtype_t dtype,
                          torus_dtype_t wire, torus_op_t op, torus_stream_t stream) {
  if (!c || !bufs) return fail(TORUS_ERR_INVALID_ARG, "null argument");
  if (!c->virt) return fail(TORUS_ERR_INVALID_ARG, "not a virtual comm");
  return baseline_impl(c, bufs, count, dtype, wire, op, static_cast<cudaStream_t>(stream), false);
}

int torus_hier_allreduce(torus_comm_t c, void* buf, size_t count, torus_dtype_t dtype,
                         torus_dtype_t wire, torus_op_t op, torus_stream_t stream) {
  if (c && c->virt) return fail(TORUS_ERR_INVALID_ARG, "virtual comm: use torus_vhier_allreduce");
  void* bufs[1] = {buf};
  return baseline_impl(c, bufs, count, dtype, wire, op, static_cast<cudaStream_t>(stream), true);
}

int torus_vhier_allreduce(torus_comm_t c, void* const* bufs, size_t count, torus_dtype_t dtype,
                          torus_dtype_t wire, torus_op_t op, torus_stream_t stream) {
  if (!c || !bufs) return fail(TORUS_ERR_INVALID_ARG, "null argument");
  if (!c->virt) return fail(TORUS_ERR_INVALID_ARG, "not a virtual comm");
  return baseline_impl(c, bufs, count, dtype, wire, op, static_cast<cudaStream_t>(stream), true);
}

size_t torus_comm_hier_round_elems(torus_comm_t c, torus_dtype_t wire) {
  if (!c || !valid_dtype(wire)) return 0;
  return (size_t)hier_round_elems(c, wire);
}

size_t torus_comm_ring_round_elems(torus_comm_t c, torus_dtype_t wire) {
  if (!c || !valid_dtype(wire)) return 0;
  return (size_t)ring_round_elems(c, wire);
}

}  // extern "C"

namespace {

// Device table of a bucket's tensors (all local ranks), cached per bucket: the first call
// with a new bucket allocates and uploads it (synchronously); later calls reuse it, so
// they stay CUDA-graph capturable.
int seg_table(torus_comm* c, void* const* ptrs, const size_t* counts, int ntensors, const MultiSeg** out) {
  std::vector<MultiSeg> h((size_t)c->nlocal * ntensors);
  for (int l = 0; l < c->nlocal; ++l) {
    unsigned long long off = 0;
    for (int i = 0; i < ntensors; ++i) {
      MultiSeg& m = h[(size_t)l * ntensors + i];
      m.ptr = ptrs[(size_t)l * ntensors + i];
      m.count = counts[i];
      m.offset = off;
      off += counts[i];
    }
  }
  for (auto& t : c->seg_tables)
    if (t.host.size() == h.size() &&
        std::equal(h.begin(), h.end(), t.host.begin(), [](const MultiSeg& x, const MultiSeg& y) {
          return x.ptr == y.ptr && x.count == y.count && x.offset == y.offset;
        })) {
      *out = t.dev;
      return TORUS_OK;
    }
  torus_comm::SegTable t;
  t.host = h;
  CU(cudaSetDevice(c->device));
  CU(cudaMalloc(&t.dev, h.size() * sizeof(MultiSeg)));
  cudaError_t e = cudaMemcpy(t.dev, h.data(), h.size() * sizeof(MultiSeg), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(t.dev);
    return cuda_fail(e, "multi-tensor table upload");
  }
  c->seg_tables.push_back(t);
  *out = t.dev;
  return TORUS_OK;
}

}  // namespace

extern "C" {

int torus_vallreduce_multi(torus_comm_t c, void* const* ptrs, const size_t* counts, int ntensors,
                           torus_dtype_t dtype, torus_dtype_t wire, torus_op_t op, torus_stream_t stream) {
  if (!c || !c->virt) return fail(TORUS_ERR_INVALID_ARG, "not a virtual comm");
  if (ntensors <= 0 || !ptrs || !counts) return fail(TORUS_ERR_INVALID_ARG, "multi args");
  if (!valid_pair(dtype, wire)) return fail(TORUS_ERR_UNSUPPORTED, "dtype %d with wire %d", dtype, wire);
  size_t total = 0;
  for (int i = 0; i < ntensors; ++i) total += counts[i];
  for (size_t i = 0; i < (size_t)c->nlocal * ntensors; ++i)
    if (counts[i % ntensors] && !ptrs[i]) return fail(TORUS_ERR_INVALID_ARG, "tensor %zu is NULL", i);
  if (total == 0) return TORUS_OK;
  const int mroute = plan_route(c, total, dtype, wire);
  if (mroute != kRoutePush && mroute != kRouteLL128)
    return fail(TORUS_ERR_UNSUPPORTED, "virtual multi-tensor calls take the multi-phase kernel only");
  const MultiSeg* d = nullptr;
  int rc = seg_table(c, ptrs, counts, ntensors, &d);
  if (rc) return rc;
  std::vector<void*> bufs(c->nlocal);
  for (int l = 0; l < c->nlocal; ++l) bufs[l] = ptrs[(size_t)l * ntensors];
  return allreduce_impl(c, bufs.data(), total, dtype, wire, op, static_cast<cudaStream_t>(stream), d, ntensors);
}

int torus_comm_reserve(torus_comm_t c, size_t staging_bytes) {
  if (!c) return fail(TORUS_ERR_INVALID_ARG, "comm is NULL");
  if (staging_bytes <= c->staging_bytes) return TORUS_OK;
  CU(cudaSetDevice(c->device));
  if (c->d_staging) {
    CU(cudaDeviceSynchronize());
    cudaFree(c->d_staging);
    c->d_staging = nullptr;
    c->staging_bytes = 0;
  }
  const size_t b = (staging_bytes + 65535) & ~(size_t)65535;
  CU(cudaMalloc(&c->d_staging, b));
  c->staging_bytes = b;
  return TORUS_OK;
}

int torus_allreduce_multi(torus_comm_t c, void* const* ptrs, const size_t* counts, int ntensors,
                          torus_dtype_t dtype, torus_dtype_t wire, torus_op_t op,
                          torus_stream_t stream) {
  if (!c || (ntensors > 0 && (!ptrs || !counts))) return fail(TORUS_ERR_INVALID_ARG, "null argument");
  if (c->virt) return fail(TORUS_ERR_INVALID_ARG, "virtual comm: not supported for multi");
  if (ntensors < 0) return fail(TORUS_ERR_INVALID_ARG, "ntensors < 0");
  if (!valid_pair(dtype, wire)) return fail(TORUS_ERR_UNSUPPORTED, "dtype %d with wire %d", dtype, wire);
  size_t total = 0;
  const size_t esz = wire_size(dtype);
  for (int i = 0; i < ntensors; ++i) {
    if (counts[i] && !ptrs[i]) return fail(TORUS_ERR_INVALID_ARG, "tensor %d is NULL", i);
    if (reinterpret_cast<uintptr_t>(ptrs[i]) % esz) return fail(TORUS_ERR_INVALID_ARG, "tensor %d misaligned", i);
    total += counts[i];
  }
  if (total == 0) return TORUS_OK;
  cudaStream_t s0 = static_cast<cudaStream_t>(stream);
  const int mroute = plan_route(c, total, dtype, wire);
  if (mroute == kRoutePush || mroute == kRouteLL128) {
    // fused: the multi-phase kernel reads the tensors with the cast
    // fused and writes them back with the up-cast fused -- no staging, no pack / unpack
    const MultiSeg* d = nullptr;
    int rc = seg_table(c, ptrs, counts, ntensors, &d);
    if (rc) return rc;
    void* bufs[1] = {ptrs[0]};
    return allreduce_impl(c, bufs, total, dtype, wire, op, s0, d, ntensors);
  }
  const size_t need = total * wire_size(wire) + 256;
  if (need > c->staging_bytes) {
    int rc = torus_comm_reserve(c, need);  // first use of a larger bucket allocates
    if (rc) return rc;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  MultiTable tab;
  size_t off = 0;
  for (int i0 = 0; i0 < ntensors; i0 += kMultiMax) {  // pack: dtype -> wire (RNE)
    const int n = std::min(kMultiMax, ntensors - i0);
    for (int i = 0; i < n; ++i) {
      tab.ptr[i] = ptrs[i0 + i];
      tab.count[i] = counts[i0 + i];
      tab.offset[i] = off;
      off += counts[i0 + i];
    }
    cudaError_t e = launch_multi_copy(tab, n, dtype, wire, c->d_staging, true, s);
    if (e != cudaSuccess) return cuda_fail(e, "multi pack");
  }
  int rc = torus_allreduce_ex(c, c->d_staging, total, wire, wire, op, stream);
  if (rc) return rc;
  off = 0;
  for (int i0 = 0; i0 < ntensors; i0 += kMultiMax) {  // unpack: wire -> dtype (exact)
    const int n = std::min(kMultiMax, ntensors - i0);
    for (int i = 0; i < n; ++i) {
      tab.ptr[i] = ptrs[i0 + i];
      tab.count[i] = counts[i0 + i];
      tab.offset[i] = off;
      off += counts[i0 + i];
    }
    cudaError_t e = launch_multi_copy(tab, n, dtype, wire, c->d_staging, false, s);
    if (e != cudaSuccess) return cuda_fail(e, "multi unpack");
  }
  return TORUS_OK;
}

}  // extern "C"

extern "C" {

int torus_nvls_prepare(torus_comm_t c, size_t bytes, long long* blob) {
  if (!c || !blob || c->virt || c->world < 2) return fail(TORUS_ERR_INVALID_ARG, "nvls_prepare args");
  if (c->nvls.mem) return fail(TORUS_ERR_INVALID_ARG, "NVLS already prepared");
  CU(cudaSetDevice(c->device));
  const int rc = nvls_prepare(c->device, c->rank, bytes, c->world, &c->nvls, blob);
  if (rc) {
    nvls_release(&c->nvls);
    return fail(rc, "NVLS prepare (multicast object / physical memory)");
  }
  return TORUS_OK;
}

int torus_nvls_attach(torus_comm_t c, const long long* blob0) {
  if (!c || !blob0 || !c->nvls.mem) return fail(TORUS_ERR_INVALID_ARG, "nvls_attach before prepare");
  CU(cudaSetDevice(c->device));
  const int rc = nvls_attach(&c->nvls, blob0);
  return rc ? fail(rc, "NVLS attach (pidfd_getfd / import / add device)") : TORUS_OK;
}

int torus_nvls_bind(torus_comm_t c) {
  if (!c || !c->nvls.have_mc) return fail(TORUS_ERR_INVALID_ARG, "nvls_bind before attach");
  CU(cudaSetDevice(c->device));
  const int rc = nvls_bind(&c->nvls);
  return rc ? fail(rc, "NVLS bind / map") : TORUS_OK;
}

int torus_nvls_allreduce(torus_comm_t c, void* buf, size_t count, torus_dtype_t dtype,
                         torus_dtype_t wire, torus_op_t op, torus_stream_t stream) {
  if (!c) return fail(TORUS_ERR_INVALID_ARG, "comm is NULL");
  if (!c->nvls.ready) return fail(TORUS_ERR_INVALID_ARG, "NVLS not initialised");
  if (!valid_pair(dtype, wire) || wire == TORUS_I32)
    return fail(TORUS_ERR_UNSUPPORTED, "NVLS: dtype %d with wire %d", dtype, wire);
  if (op != TORUS_SUM && op != TORUS_MEAN) return fail(TORUS_ERR_INVALID_ARG, "bad op %d", op);
  if (c->poisoned || *reinterpret_cast<volatile int*>(c->h_err)) {
    c->poisoned = true;
    return fail(TORUS_ERR_TIMEOUT, "communicator has an async error; destroy it");
  }
  if (count == 0) return TORUS_OK;
  if (!buf || reinterpret_cast<uintptr_t>(buf) % wire_size(dtype))
    return fail(TORUS_ERR_INVALID_ARG, "buffer NULL or misaligned");
  const unsigned long long sw = wire_size(wire), q = kVecBytes / sw, N = (unsigned long long)c->world;
  const unsigned long long R = (c->nvls.size / sw) / (q * N) * (q * N);
  for (unsigned long long r0 = 0; r0 < count; r0 += R) {
    const unsigned long long n = std::min<unsigned long long>(R, count - r0);
    cudaError_t e = launch_nvls(c->d_ranks, &c->nvls, buf, n, r0, dtype, wire, op, 1.0f / (float)N, c->G,
                                c->timeout_ns, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "nvls kernel launch");
  }
  return TORUS_OK;
}

}  // extern "C"

extern "C" {

const char* torus_comm_route(torus_comm_t c, size_t count, torus_dtype_t dtype, torus_dtype_t wire) {
  if (!c || !valid_pair(dtype, wire)) return "invalid";
  return route_name(plan_route(c, count, dtype, wire));
}

int torus_comm_config(torus_comm_t c, unsigned long long* words, int n) {
  if (!c || !words || n < 1) return -fail(TORUS_ERR_INVALID_ARG, "config args");
  // Everything that decides which bytes and flags a call touches on a PEER: the grid,
  // the slab layout, the routing thresholds and every tiling knob of every kernel.
  int tv16 = 0, ns16 = 0, tv32 = 0, ns32 = 0;
  pull_ring(c, 1, &tv16, &ns16);
  pull_ring(c, 2, &tv32, &ns32);
  const unsigned long long v[] = {
      (unsigned long long)c->world, (unsigned long long)c->X, (unsigned long long)c->Y,
      (unsigned long long)c->G, c->slab_size, c->layout.data_off, c->layout.ll_off,
      c->layout.ll_slot, c->layout.ll_region, c->layout.pull_flag_off, c->ll2_max,
      (unsigned long long)c->mode, (unsigned long long)c->tile_vecs, c->one_tile_max, c->mid_tiles,
      (unsigned long long)tv16, (unsigned long long)tv32, c->timeout_ns, (unsigned long long)c->ll128_lane};
  const int m = (int)(sizeof v / sizeof v[0]);
  for (int i = 0; i < n; ++i) words[i] = i < m ? v[i] : 0;
  return m;
}

}  // extern "C"

namespace {

typedef CUresult (*PFN_getAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);

// base and size of the allocation that contains p (driver API through the runtime's
// entry-point query, so the library does not link libcuda)
bool alloc_range(const void* p, char** base, size_t* size) {
  static PFN_getAddressRange fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !f)
      return false;
    fn = reinterpret_cast<PFN_getAddressRange>(f);
  }
  CUdeviceptr b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS) return false;
  *base = reinterpret_cast<char*>(b);
  *size = sz;
  return true;
}

}  // namespace

extern "C" {

int torus_buffer_export(const void* ptr, size_t bytes, torus_ipc_handle_t* out) {
  if (!ptr || !out || !bytes) return fail(TORUS_ERR_INVALID_ARG, "buffer_export args");
  char* base = nullptr;
  size_t size = 0;
  if (!alloc_range(ptr, &base, &size)) return fail(TORUS_ERR_INVALID_ARG, "not a device allocation");
  const size_t off = static_cast<const char*>(ptr) - base;
  if (off + bytes > size) return fail(TORUS_ERR_INVALID_ARG, "buffer exceeds its allocation");
  cudaIpcMemHandle_t h;
  CU(cudaIpcGetMemHandle(&h, base));
  memset(out, 0, sizeof *out);
  memcpy(out->bytes, &h, 64);
  out->offset = off;
  out->size = bytes;
  return TORUS_OK;
}

int torus_register_buffer(torus_comm_t c, void* ptr, size_t bytes, const torus_ipc_handle_t* handles) {
  if (!c || !ptr || !handles || !bytes) return fail(TORUS_ERR_INVALID_ARG, "register args");
  if (c->virt) return fail(TORUS_ERR_INVALID_ARG, "virtual comm: buffers are local already");
  for (int r = 0; r < c->world; ++r)
    if (handles[r].size != bytes) return fail(TORUS_ERR_MISMATCH, "registered sizes differ across ranks");
  CU(cudaSetDevice(c->device));
  torus_comm::Reg g;
  g.ptr = static_cast<char*>(ptr);
  g.bytes = bytes;
  g.aligned = true;
  g.peer.assign(c->world, nullptr);
  for (int r = 0; r < c->world; ++r) {
    if ((handles[r].offset & 15) != 0 || (r == c->rank && (reinterpret_cast<uintptr_t>(ptr) & 15) != 0))
      g.aligned = false;  // every rank sees the same handles: the same decision everywhere
    if (r == c->rank) {
      g.peer[r] = g.ptr;
      continue;
    }
    const std::string key(reinterpret_cast<const char*>(handles[r].bytes), 64);
    void* base = nullptr;
    for (auto& h : c->ipc_opened)
      if (h.first == key) base = h.second;
    if (!base) {
      cudaIpcMemHandle_t h;
      memcpy(&h, handles[r].bytes, 64);
      cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) return fail(TORUS_ERR_PEER, "cudaIpcOpenMemHandle(buffer of rank %d): %s", r,
                                        cudaGetErrorString(e));
      c->ipc_opened.emplace_back(key, base);
    }
    g.peer[r] = static_cast<char*>(base) + handles[r].offset;
  }
  for (auto& old : c->regs)
    if (old.ptr == g.ptr) {
      old = g;
      return TORUS_OK;
    }
  c->regs.push_back(g);
  return TORUS_OK;
}

int torus_deregister_buffer(torus_comm_t c, void* ptr) {
  if (!c) return fail(TORUS_ERR_INVALID_ARG, "comm is NULL");
  for (size_t i = 0; i < c->regs.size(); ++i)
    if (c->regs[i].ptr == ptr) {
      c->regs.erase(c->regs.begin() + i);
      return TORUS_OK;  // the peer mappings stay open until destroy (others may share them)
    }
  return fail(TORUS_ERR_INVALID_ARG, "buffer is not registered");
}

}  // extern "C"
