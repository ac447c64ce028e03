// torus_pull.cu -- the default large-message 2D-Torus all-reduce kernel (Sec. 2.2):
// a tile-granular DATAFLOW pipeline in which every byte crosses NVLink as a TMA bulk LOAD
// (cp.async.bulk, peer -> shared memory) and every store is local.
//
//   "Firstly, reduce-scatter is performed horizontally. Then, all-reduce is performed
//    vertically. Finally, all-gather is performed horizontally."
//
// Rank (rho, c) of the X-by-Y grid runs five kinds of CTA, each a loop over its own tiles
// ("jobs") that meets the others only through per-tile flags:
//
//   S0  (a2 pre-pass)  cast/copy my buffer's tiles that peers will read into my slab's
//                      `win` region (wire type; the fp16 cast of PAPER.md:121 fused)
//   R   (a2, H-RS)     pull the X row peers' `win` tiles of MY chunk c, fold them in ring
//                      order c+1, ..., c, round once to the wire: my P1 tile
//                      (Y == 1: this is the last reduce phase -> mean, final)
//   VR  (a3, V-RS)     pull the Y column peers' P1 tiles of MY sub-chunk (c, rho), fold in
//                      ring order rho+1, ..., rho, mean (C8), round once: final values into
//                      my buffer and my `chunk` region
//   VA  (a4, V-AG)     pull the column peers' reduced sub-chunks of chunk c (a copy)
//   H   (a5, H-AG)     pull the row peers' completed chunks into my buffer (up-cast fused)
//
// Why pull: a store over NVLink is complete only when the peer acknowledges it, so the
// system-scope fence that must precede a flag waits for every in-flight remote store of
// the SM (5-22 us measured) -- the latency that bounded the round-1
// push kernel.  Here every flag covers LOCAL stores only (sub-us fence), and the reader
// pulls after it sees the flag.  Why dataflow: the round-1 kernel moved all five stages
// in lock-step iterations, so every hand-off latency was paid once per iteration; here a
// stage starts tile k the moment its inputs for tile k are flagged, and the fill/drain of
// the pipeline is paid once per call.
//
// Slab regions are double-buffered by call parity (epoch & 1).  A rank writes parity p in
// call e + 2 only after its call e + 1 observed a flag of call e + 1 from every row and
// column peer, i.e. after each of them finished call e (stream order) and with it every
// read of this rank's parity-p regions -- so no entry or exit barrier is needed.
//
// Fold order, partition, rounding points and the mean placement are the oracle's
// (SURVEY C3-C10), so every dtype is bit-exact against the CPU oracle.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "torus_device.cuh"
#include "torus_pull.h"

namespace torus {
namespace {

#ifndef TORUS_PULL_CW
#define TORUS_PULL_CW 4
#endif
#ifndef TORUS_PULL_U
#define TORUS_PULL_U 4
#endif
constexpr int kConsumerWarps = TORUS_PULL_CW;           // warps 2.. : consumers
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kPullThreads = 64 + kConsumers;           // warp 0 producer, warp 1 storer

// ------------------------------------------------------------------------------------
// tile geometry (identical on every rank: host and device derive it from n, X, Y, q, TV)
// ------------------------------------------------------------------------------------
struct Tile {
  bool ok;                       // the tile exists (k < tiles of its sub-chunk)
  unsigned long long co;         // chunk offset in the round (elements)
  unsigned long long cs;         // sub-chunk offset inside the chunk (elements)
  unsigned long long e0;         // first element of the tile, relative to the chunk
  unsigned long long nel;        // elements in the tile (the round's last one may be ragged)
  int nvec;                      // 16-byte wire vectors (last one possibly partial)
};

__device__ __forceinline__ Tile tile_of(const PullArgs& a, int X, int Y, int j, int s, int k) {
  Tile t;
  const int js = j * Y + s;
  const unsigned long long per = (unsigned long long)a.TV * a.q;
  const unsigned long long st = (unsigned long long)k * per;
  const unsigned long long sl = a.g_sl[js];
  t.ok = k < a.g_K[js];
  t.co = a.g_co[j];
  t.cs = a.g_cs[js];
  t.e0 = t.cs + st;
  t.nel = t.ok ? min(per, sl - st) : 0;
  t.nvec = ((int)t.nel + a.q - 1) / a.q;  // nel <= TV * q fits 32 bits
  return t;
}

// Flag word index inside the pull flag region (u32 epochs, value = call epoch + 1).
//   WIN[src][s][k]  src's win tile (s, k) of my chunk is ready   (src = column j, or row i if X == 1)
//   P1 [i][k]       row i's P1 tile k of my sub-chunk is ready    (column peers)
//   V  [i][k]       row i's reduced sub-chunk tile k is ready     (column peers)
//   C  [j][s][k]    column j's chunk tile (s, k) is complete       (row peers)
__device__ __forceinline__ size_t fl_win(const PullArgs& a, int Y, int src, int s, int k) {
  return a.fl_win + ((size_t)src * Y + s) * a.Kmax + k;
}
__device__ __forceinline__ size_t fl_p1(const PullArgs& a, int i, int k) { return a.fl_p1 + (size_t)i * a.Kmax + k; }
__device__ __forceinline__ size_t fl_v(const PullArgs& a, int i, int k) { return a.fl_v + (size_t)i * a.Kmax + k; }
__device__ __forceinline__ size_t fl_c(const PullArgs& a, int Y, int j, int s, int k) {
  return a.fl_c + ((size_t)j * Y + s) * a.Kmax + k;
}

enum PullKind { kS0 = 0, kR = 1, kVR = 2, kVA = 3, kH = 4, kSig = 5, kKinds = 6 };

// One job of a CTA: the tile, where its operands come from, where it waits.
struct Job {
  bool ok;
  int j, s, k, i;                // chunk column, sub-chunk row, tile, source row (VA)
  Tile t;
};

// Number of job slots of each kind (jobs J = 0 .. count-1; CTA b of the kind takes
// J = b, b + g, ...).  k-major order so that every rank produces tile k before k + 1.
__device__ __forceinline__ int job_count(const PullArgs& a, int kind, int X, int Y) {
  switch (kind) {
    case kS0: return (a.zc ? 1 : a.Kmax) * (X > 1 ? X * Y : Y);
    case kR: return a.Kmax * Y;
    case kVR: return a.Kmax;
    case kVA: return a.Kmax * (Y - 1);
    case kH: return a.Kmax * (X - 1) * Y;
    default: return 0;
  }
}

template <int DT, int W>
__device__ __forceinline__ Job job_of(const PullArgs& a, int kind, int J, int X, int Y, int rho, int c) {
  Job jb;
  jb.i = -1;
  switch (kind) {
    case kS0:
      if (X > 1) {
        jb.k = J / (X * Y);
        jb.j = (J / Y) % X;
        jb.s = J % Y;
      } else {
        jb.k = J / Y;
        jb.j = 0;
        jb.s = J % Y;
      }
      // zero-copy: S0 only copies ragged tails, i.e. each sub-chunk's last tile
      if (a.zc) jb.k = max(0, a.g_K[jb.j * Y + jb.s] - 1);
      break;
    case kR:
      jb.k = J / Y;
      jb.j = c;
      jb.s = J % Y;
      break;
    case kVR:
      jb.k = J;
      jb.j = c;
      jb.s = rho;
      break;
    case kVA:
      jb.k = J / (Y - 1);
      jb.i = (rho + 1 + J % (Y - 1)) % Y;
      jb.j = c;
      jb.s = jb.i;
      break;
    default: {
      const int jj = 1 + (J / Y) % (X - 1);
      jb.k = J / ((X - 1) * Y);
      jb.j = (c + jj) % X;
      jb.s = J % Y;
    }
  }
  jb.t = tile_of(a, X, Y, jb.j, jb.s, jb.k);
  jb.ok = jb.t.ok;
  return jb;
}

// operands of a job, in fold order (o = 0 .. nops-1)
__device__ __forceinline__ int job_nops(int kind, int X, int Y) {
  return kind == kR ? X : (kind == kVR ? Y : 1);
}

// ------------------------------------------------------------------------------------
// waits with the device watchdog and the CTA abort flag
// ------------------------------------------------------------------------------------
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_wait_abortable(uint64_t* bar, uint32_t phase, volatile int* abort) {
  while (!mbar_try(bar, phase))
    if (*abort) return false;
  return true;
}
__device__ __forceinline__ void mbar_arrive1(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// generic-proxy shared-memory writes -> visible to a later async-proxy (TMA) read
__device__ __forceinline__ void fence_view_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void consumer_bar() {  // named barrier 1 over the consumer warps
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ bool ragged(const PullArgs& a, const Tile& t) {
  return (t.nel % (unsigned long long)a.q) != 0;
}

// Where a reduce reads the first-phase input tile of rank `src`: its user buffer (own
// buffer, or a peer's registered buffer in zero-copy mode) or its slab's `win` copy.
template <int DT, int W>
__device__ __forceinline__ bool input_from_buf(const PullArgs& a, const Tile& t, bool own) {
  if (ragged(a, t)) return false;  // a TMA read of the last partial vector would overrun
  return own ? (DT == W && a.aligned) : (a.zc != 0);
}

// the final values of a tile go to the user buffer by a TMA bulk store when they are
// wire-typed, aligned and whole vectors; otherwise the consumers store them (cast fused)
template <int DT, int W>
__device__ __forceinline__ bool buf_bulk(const PullArgs& a, const Tile& t) {
  return DT == W && a.aligned && !ragged(a, t);
}

// S0 jobs: copy the tiles some reduce reads from `win` (see input_from_buf)
template <int DT, int W>
__device__ __forceinline__ Job job_of_checked(const PullArgs& a, int kind, int J, int X, int Y, int rho, int c) {
  Job jb = job_of<DT, W>(a, kind, J, X, Y, rho, c);
  if (jb.ok && kind == kS0) {
    const bool own = X > 1 ? (jb.j == c) : (jb.s == rho);
    if (input_from_buf<DT, W>(a, jb.t, own)) jb.ok = false;
  }
  return jb;
}

__device__ __forceinline__ void st_release_gpu64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_gpu64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Raise the flags that announce job `jg` of a CTA of `kind` to the ranks that consume it
// (called after a fence that orders the job's stores before the flags).
__device__ __forceinline__ void raise_flags(const PullArgs& a, const RankDev* R, int kind, const Job& jg,
                                            uint32_t v) {
  const int X = R->X, Y = R->Y, rho = R->rho, c = R->c;
  auto flag_at = [&](int rank, size_t idx) -> uint32_t* {
    return reinterpret_cast<uint32_t*>(R->ws[rank] + a.flag_off) + idx;
  };
  if (kind == kS0) {
    if (X > 1) st_relaxed_sys(flag_at(rho * X + jg.j, fl_win(a, Y, c, jg.s, jg.k)), v);
    else st_relaxed_sys(flag_at(jg.s * X, fl_win(a, Y, rho, 0, jg.k)), v);
  } else if (kind == kR) {
    if (Y > 1) {
      st_relaxed_sys(flag_at(jg.s * X + c, fl_p1(a, rho, jg.k)), v);
    } else {
      for (int jj = 1; jj < X; ++jj) st_relaxed_sys(flag_at(rho * X + (c + jj) % X, fl_c(a, Y, c, 0, jg.k)), v);
    }
  } else if (kind == kVR) {
    for (int ii = 1; ii < Y; ++ii) st_relaxed_sys(flag_at(((rho + ii) % Y) * X + c, fl_v(a, rho, jg.k)), v);
    for (int jj = 1; jj < X; ++jj) st_relaxed_sys(flag_at(rho * X + (c + jj) % X, fl_c(a, Y, c, rho, jg.k)), v);
  } else if (kind == kVA) {
    for (int jj = 1; jj < X; ++jj) st_relaxed_sys(flag_at(rho * X + (c + jj) % X, fl_c(a, Y, c, jg.i, jg.k)), v);
  }
}

// Trace (TORUS_TRACE=1): per CTA, per job n < 63 globaltimer stamps -- 0 producer saw the
// inputs' flags, 1 consumers saw the operands land, 2 consumers done, 3 flags raised,
// 4 bulk stores issued, 5 stores read (slots freed); slot 63 = the CTA's start and end.
__device__ __forceinline__ void pstamp(const PullArgs& a, int cta, int n, int ev) {
  if (a.trace && n < kPullTraceJobs - 1 && cta < kMaxLocal * 512)
    a.trace[((size_t)cta * kPullTraceJobs + n) * kPullTraceEv + ev] = gtimer();
}

// ------------------------------------------------------------------------------------
// the kernel
// ------------------------------------------------------------------------------------
//   warp 0 (lane 0)  producer: per job, wait for the input tiles' flags, then TMA-load the
//                    operands (fold order) into consecutive ring slots
//   warps 2..5       consumers: fold the operands (f32 / u32) into slot 0 of the job in
//                    shared memory, or cast (S0); ILP: each thread holds 4 vectors
//   warp 1 (lane 0)  storer + signaler: TMA bulk-stores every finished job's result from
//                    shared memory to its LOCAL destinations (win / P1 / chunk / user
//                    buffer), frees the slots once read, waits for the writes, then ONE
//                    fence publishes all jobs stored so far and their flags are raised.
// No generic global store sits on the hot path (consumers store only for a cast or a
// ragged/unaligned user buffer), so the publishing fence is not stuck behind a backlog
// of st.global.
template <int DT, int W>
__global__ void __launch_bounds__(kPullThreads) torus_pull_kernel(const PullArgs a) {
  using Acc = typename Wire<W>::Acc;
  constexpr int VE = Wire<W>::VE;
  constexpr int SW = kVecBytes / VE;           // bytes per wire element
  constexpr int DB = sizeof(typename Elem<DT>::T);
  constexpr int U = TORUS_PULL_U;              // vectors in flight per consumer thread

  // ---- which rank, which kind, which CTA of the kind ----
  const int lr = blockIdx.x / a.gsum;
  int b = blockIdx.x - lr * a.gsum;
  int kind = 0;
  while (kind < kKinds - 1 && b >= a.g[kind]) b -= a.g[kind++];
  const int G = a.g[kind];
  const RankDev* __restrict__ R = a.ranks + lr;
  const int X = R->X, Y = R->Y, N = R->N, rho = R->rho, c = R->c, me = R->rank;
  void* const buf = a.buf[lr];

  extern __shared__ __align__(128) unsigned char smem[];
  const int NS = a.nslots;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NS * a.slot_bytes);
  uint64_t* empty = full + NS;
  __shared__ uint32_t s_epoch;
  __shared__ int s_abort;
  __shared__ int s_done;      // consumer-warp job completions (storer polls)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    s_epoch = ld_acquire_gpu(R->pull_ctr);
    s_abort = 0;
    s_done = 0;
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0 && a.trace && blockIdx.x < kMaxLocal * 512)
    a.trace[((size_t)blockIdx.x * kPullTraceJobs + kPullTraceJobs - 1) * kPullTraceEv] = gtimer();
  const uint32_t epoch = s_epoch;
  const uint32_t v = epoch + 1u;               // flag value of this call
  if (a.delay_ns) {  // robustness runs: start every CTA after a pseudo-random delay
    uint32_t h = (uint32_t)(me * 7919 + blockIdx.x * 104729) ^ (epoch * 2654435761u);
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    h ^= h >> 15;
    const unsigned long long until = gtimer() + (h % a.delay_ns);
    while (gtimer() < until) __nanosleep(256);
  }
  const int par = (int)(epoch & 1u);
  char* const myws = R->ws[me];
  uint32_t* const myflags = reinterpret_cast<uint32_t*>(myws + a.flag_off);
  auto flag_at = [&](int rank, size_t idx) -> uint32_t* {
    return reinterpret_cast<uint32_t*>(R->ws[rank] + a.flag_off) + idx;
  };
  auto bufp = [&](int rank, const Tile& t) -> char* {  // a rank's user buffer at a tile
    char* base = (rank == me) ? reinterpret_cast<char*>(buf) : a.peer_buf[rank];
    return base + (a.buf_off + t.co + t.e0) * DB;
  };
  const int njobs = job_count(a, kind, X, Y);
  const int nops = job_nops(kind, X, Y);

  if (kind == kSig) {
    // ================================ SIG CTA ======================================
    // Every thread watches up to 4 data CTAs of this rank: when one publishes (gpu-scope
    // release of its job count), acquire it, fence at system scope -- on this SM, which
    // moves no bulk data -- and raise the flags of the newly published jobs.
    const int ndata = a.gsum - a.g[kSig];
    const unsigned long long deadline = gtimer() + a.timeout_ns;
    constexpr int M = 4;
    int dk[M], db[M], dJ[M], dn[M], dtot[M], dcta[M];
    for (int m = 0; m < M; ++m) {
      const int d = (b + m * G) * kPullThreads + tid;
      dk[m] = -1;
      if (d >= ndata) continue;
      int k2 = 0, b2 = d;
      while (k2 < kSig - 1 && b2 >= a.g[k2]) b2 -= a.g[k2++];
      if (k2 == kH) continue;  // H raises no flags
      const int nj2 = job_count(a, k2, X, Y);
      int tot = 0;
      for (int J = b2; J < nj2; J += a.g[k2])
        if (job_of_checked<DT, W>(a, k2, J, X, Y, rho, c).ok) ++tot;
      if (tot == 0) continue;
      dk[m] = k2;
      db[m] = b2;
      dcta[m] = d;
      dJ[m] = b2;
      dn[m] = 0;
      dtot[m] = tot;
    }
    const unsigned long long* pub = a.pub + (size_t)lr * a.gsum;
    unsigned spin = 0;
    while (true) {
      bool live = false, work = false;
      int cnt[M];
      for (int m = 0; m < M; ++m) {
        cnt[m] = 0;
        if (dk[m] < 0) continue;
        live = true;
        const unsigned long long w = ld_relaxed_gpu64(pub + dcta[m]);
        if ((uint32_t)(w >> 32) == epoch && (int)(uint32_t)w > dn[m]) {
          cnt[m] = (int)(uint32_t)w;
          work = true;
        }
      }
      if (!live) break;
      if (!work) {
        __nanosleep(64);
        if ((++spin & 255u) == 0 && (gtimer() > deadline || *(volatile int*)&s_abort || *(volatile int*)R->err)) {
          atomicCAS_system(R->err, 0, kErrTimeout);
          break;
        }
        continue;
      }
      // acquire what was published, then one system-scope fence for all of it
      for (int m = 0; m < M; ++m) {
        if (cnt[m] == 0) continue;
        (void)ld_acquire_gpu64(pub + dcta[m]);
      }
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      for (int m = 0; m < M; ++m) {
        if (cnt[m] == 0) continue;
        const int k2 = dk[m], g2 = a.g[k2], nj2 = job_count(a, k2, X, Y);
        while (dn[m] < cnt[m] && dJ[m] < nj2) {
          const Job jg = job_of_checked<DT, W>(a, k2, dJ[m], X, Y, rho, c);
          dJ[m] += g2;
          if (!jg.ok) continue;
          raise_flags(a, R, k2, jg, v);
          ++dn[m];
        }
        if (dn[m] >= dtot[m]) dk[m] = -1;
      }
    }
  } else if (warp == 0) {
    // =============================== producer =====================================
    if (lane == 0) {
      const unsigned long long deadline = gtimer() + a.timeout_ns;
      // Presence: CTA 0 of S0 tells every row and column peer that this rank has entered
      // the call (so its user buffer holds this call's input), and does not finish before
      // all of them have -- so every call observes every peer, which the parity double-
      // buffering relies on even when a short round leaves some tiles (and flags) empty.
      const bool presence = (kind == kS0 && b == 0);
      if (presence) {
        for (int jj = 1; jj < X; ++jj) st_relaxed_sys(flag_at(rho * X + (c + jj) % X, a.fl_pres + me), v);
        for (int ii = 1; ii < Y; ++ii) st_relaxed_sys(flag_at(((rho + ii) % Y) * X + c, a.fl_pres + me), v);
      }
      bool ok = true;
      auto need = [&](size_t idx) {
        if (!ok) return;
        const uint32_t* f = myflags + idx;
        unsigned spin = 0;
        while ((int32_t)(ld_relaxed_sys(f) - v) < 0) {
          __nanosleep(32);
          if ((++spin & 255u) == 0 &&
              (gtimer() > deadline || *(volatile int*)&s_abort || *(volatile int*)R->err)) {
            ok = false;
            return;
          }
        }
        (void)ld_acquire_sys(f);  // synchronizes with the peer's fence + flag store
      };
      uint32_t ps = 0;  // operand loads issued (ring position)
      int nj = 0;       // valid jobs so far (trace index)
      for (int J = b; J < njobs && ok; J += G) {
        const Job jb = job_of_checked<DT, W>(a, kind, J, X, Y, rho, c);
        if (!jb.ok) continue;
        // -- wait for this job's inputs --
        if (kind == kR) {
          for (int j = 0; j < X; ++j) {
            if (input_from_buf<DT, W>(a, jb.t, j == c)) {
              if (j != c) need(a.fl_pres + rho * X + j);
            } else {
              need(fl_win(a, Y, j, jb.s, jb.k));
            }
          }
        } else if (kind == kVR) {
          const bool skip = (a.fault == 2 && me == 0 && b == 0 && nj == 0);  // negative control
          for (int i = 0; i < Y; ++i) {
            if (X > 1) { if (!skip) need(fl_p1(a, i, jb.k)); }
            else if (input_from_buf<DT, W>(a, jb.t, i == rho)) { if (i != rho) need(a.fl_pres + i * X); }
            else need(fl_win(a, Y, i, 0, jb.k));
          }
        } else if (kind == kVA) {
          need(fl_v(a, jb.i, jb.k));
        } else if (kind == kH) {
          need(fl_c(a, Y, jb.j, jb.s, jb.k));
        }
        if (!ok) break;
        fence_proxy_async();  // generic-proxy acquire before the async-proxy (TMA) reads
        pstamp(a, blockIdx.x, nj++, 0);
        // -- issue the operand loads (fold order) --
        const bool direct = (kind == kS0) && !(a.aligned && !ragged(a, jb.t));
        for (int o = 0; o < nops && ok; ++o) {
          const uint32_t slot = ps % NS, use = ps / NS;
          ++ps;
          if (use > 0 && !mbar_wait_abortable(&empty[slot], (use - 1) & 1u, &s_abort)) { ok = false; break; }
          const char* src = nullptr;
          uint32_t bytes = (uint32_t)jb.t.nvec * kVecBytes;
          if (kind == kS0) {
            bytes = (uint32_t)jb.t.nvec * VE * DB;  // my buffer's tile (dtype bytes)
            src = bufp(me, jb.t);
          } else if (kind == kR) {
            const int j = (c + 1 + o) % X;  // fold order: columns c+1, ..., c
            src = input_from_buf<DT, W>(a, jb.t, j == c) ? bufp(rho * X + j, jb.t)
                                                        : R->ws[rho * X + j] + a.win_off[par] + (jb.t.co + jb.t.e0) * SW;
          } else if (kind == kVR) {
            const int i = (rho + 1 + o) % Y;  // fold order: rows rho+1, ..., rho
            if (X > 1) src = R->ws[i * X + c] + a.p1_off[par] + jb.t.e0 * SW;
            else src = input_from_buf<DT, W>(a, jb.t, i == rho) ? bufp(i * X, jb.t)
                                                               : R->ws[i * X] + a.win_off[par] + (jb.t.co + jb.t.e0) * SW;
          } else if (kind == kVA) {
            src = R->ws[jb.i * X + c] + a.chunk_off[par] + jb.t.e0 * SW;
          } else {
            src = R->ws[rho * X + jb.j] + a.chunk_off[par] + jb.t.e0 * SW;
          }
          if (direct) {
            mbar_arrive1(&full[slot]);  // consumers read the user buffer themselves
          } else {
            mbar_expect_tx(&full[slot], bytes);
            tma_load(smem + (size_t)slot * a.slot_bytes, src, bytes, &full[slot]);
          }
        }
      }
      if (!ok) {
        atomicCAS_system(R->err, 0, kErrTimeout);  // keep an earlier MISMATCH
        s_abort = 1;
      }
      if (presence && ok) {
        auto seen = [&](int peer) {
          const uint32_t* f = myflags + a.fl_pres + peer;
          unsigned spin = 0;
          while (ok && (int32_t)(ld_relaxed_sys(f) - v) < 0) {
            __nanosleep(64);
            if ((++spin & 255u) == 0 && (gtimer() > deadline || *(volatile int*)R->err)) ok = false;
          }
        };
        for (int jj = 1; jj < X; ++jj) seen(rho * X + (c + jj) % X);
        for (int ii = 1; ii < Y; ++ii) seen(((rho + ii) % Y) * X + c);
        if (!ok) atomicCAS_system(R->err, 0, kErrTimeout);
      }
    }
  } else if (warp == 1) {
    // ========================== storer + signaler ==================================
    // Stores are issued one bulk group per batch of finished jobs; a batch's flags are
    // raised once the NEXT batch has been issued (wait_group 1) or, when no new job has
    // finished, after waiting for it alone (wait_group 0) -- so waiting for write
    // completion never holds up slot recycling.
    if (lane == 0) {
      int Js = b, Jg = b;          // cursors: next job to store / to signal
      int nst = 0, nsig = 0;       // jobs stored / signaled
      int older = 0;               // stored jobs of the older unsignaled batch (rest: newest)
      uint32_t rs = 0;             // ring position of the next job to release
      auto next_valid = [&](int& J, Job& jb) -> bool {
        for (; J < njobs; J += G) {
          jb = job_of_checked<DT, W>(a, kind, J, X, Y, rho, c);
          if (jb.ok) return true;
        }
        return false;
      };
      Job js, jg;
      bool more_s = next_valid(Js, js);
      bool more_g = next_valid(Jg, jg);
      auto publish = [&](int upto) {  // raise the flags of jobs [nsig, upto)
        fence_proxy_async();
        if (a.fence == 3) {
          // hand the jobs to a SIG CTA: gpu-scope release here, the system-scope fence
          // and the remote flag stores happen on an SM without bulk traffic
          st_release_gpu64(a.pub + blockIdx.x, ((unsigned long long)epoch << 32) | (unsigned)upto);
          for (; nsig < upto; ++nsig) pstamp(a, blockIdx.x, nsig, 3);
          return;
        }
        if (a.fence == 0) asm volatile("fence.acq_rel.sys;" ::: "memory");
        else if (a.fence == 1) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        while (nsig < upto && more_g) {
          raise_flags(a, R, kind, jg, v);
          pstamp(a, blockIdx.x, nsig, 3);
          ++nsig;
          Jg += G;
          more_g = next_valid(Jg, jg);
        }
      };
      while (more_s || nsig < nst) {
        if (*(volatile int*)&s_abort) break;
        const int done = ld_acquire_cta(&s_done) / kConsumerWarps;  // consumers finished [0, done)
        if (done > nst && more_s) {
          // ---- one bulk group: every finished job, from its slot 0 ----
          const uint32_t rs0 = rs;
          const int nst0 = nst;
          while (nst < done && more_s) {
            const Tile& t = js.t;
            const unsigned char* src = smem + (size_t)(rs % NS) * a.slot_bytes;
            const uint32_t bytes = (uint32_t)t.nvec * kVecBytes;
            if (kind == kS0) {
              tma_store(myws + a.win_off[par] + (t.co + t.e0) * SW, src, bytes);
            } else if (kind == kR && Y > 1) {
              tma_store(myws + a.p1_off[par] + t.e0 * SW, src, bytes);
            } else {  // final values: my chunk region (read by peers) and my buffer
              const bool chunk_out = (kind == kVR) || (kind == kR) || (kind == kVA && X > 1);
              if (chunk_out) tma_store(myws + a.chunk_off[par] + t.e0 * SW, src, bytes);
              if (buf_bulk<DT, W>(a, t)) tma_store(bufp(me, t), src, bytes);
            }
            pstamp(a, blockIdx.x, nst, 4);
            rs += (uint32_t)nops;
            ++nst;
            Js += G;
            more_s = next_valid(Js, js);
          }
          tma_commit();
          // ---- free the slots once the bulk stores have read them ----
          tma_wait_read<0>();
          for (uint32_t p = rs0; p < rs; ++p) mbar_arrive1(&empty[p % NS]);
          for (int n = nst0; n < nst; ++n) pstamp(a, blockIdx.x, n, 5);
          if (kind == kH) continue;
          if (older > 0) {  // the previous batch is complete once only this one may pend
            tma_wait_all<1>();
            publish(nsig + older);
          }
          older = nst - nsig;
        } else if (nsig < nst && kind != kH) {
          tma_wait_all<0>();  // nothing new finished: publish what is stored
          publish(nst);
          older = 0;
        } else if (!more_s) {
          break;
        } else {
          __nanosleep(20);
        }
      }
      tma_wait_all<0>();
    }
  } else {
    // =============================== consumers ====================================
    const int ct = tid - 64;  // 0 .. kConsumers-1
    uint32_t cs = 0;          // operands consumed (ring position)
    int nj = 0;               // valid jobs so far (trace index)
    for (int J = b; J < njobs; J += G) {
      const Job jb = job_of_checked<DT, W>(a, kind, J, X, Y, rho, c);
      if (!jb.ok) continue;
      const uint32_t slot0 = cs;
      bool ok = true;
      for (int o = 0; o < nops && ok; ++o)
        ok = mbar_wait_abortable(&full[(slot0 + o) % NS], ((slot0 + o) / NS) & 1u, &s_abort);
      if (!ok) break;
      if (ct == 0) pstamp(a, blockIdx.x, nj, 1);
      const Tile& t = jb.t;
      const unsigned long long cbase = t.co;                  // chunk offset in the round
      const uint32_t sbase = smem_u32(smem);
      const uint32_t out = sbase + (slot0 % NS) * (uint32_t)a.slot_bytes;  // slot 0 = result
      auto slota = [&](int o) -> uint32_t { return sbase + ((slot0 + o) % NS) * (uint32_t)a.slot_bytes; };
      const bool bb = buf_bulk<DT, W>(a, t);
      if (kind == kS0) {
        // C1: w = to_wire(in) into the slot (then the storer bulk-stores it to win)
        const bool direct = !(a.aligned && !ragged(a, t));
        if (direct || DT != W) {
          for (int base = 0; base < t.nvec; base += kConsumers * U) {  // uniform trip count
            const int v0 = base + ct;
            uint4 w[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int vv = v0 + u * kConsumers;
              if (vv >= t.nvec) continue;
              const unsigned long long el = t.e0 + (unsigned long long)vv * VE;
              const int nrem = (int)min((unsigned long long)VE, t.nel - (unsigned long long)vv * VE);
              if (direct) {
                w[u] = load_user<DT, W>(buf, a.buf_off + cbase + el, nrem, a.aligned != 0);
              } else if constexpr (DT != W) {
                const uint4 f0 = lds128(slota(0) + vv * 32), f1 = lds128(slota(0) + vv * 32 + 16);
                const float ff[8] = {__uint_as_float(f0.x), __uint_as_float(f0.y), __uint_as_float(f0.z),
                                     __uint_as_float(f0.w), __uint_as_float(f1.x), __uint_as_float(f1.y),
                                     __uint_as_float(f1.z), __uint_as_float(f1.w)};
                w[u] = pack<W>(ff);
              }
            }
            if (!direct && DT != W) consumer_bar();  // in-place f32 -> wire: all reads first
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int vv = v0 + u * kConsumers;
              if (vv < t.nvec) sts128(out + vv * 16, w[u]);
            }
            if (!direct && DT != W) consumer_bar();
          }
        }
      } else if (kind == kR || kind == kVR) {
        // fold the operands in ring order (loaded in that order), f32 / u32 accumulation
        const bool last_reduce = (kind == kVR) || (Y == 1);
        for (int v0 = ct; v0 < t.nvec; v0 += kConsumers * U) {  // vectors v0 + u * kConsumers
          Acc acc[U][VE];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int vv = v0 + u * kConsumers;
            if (vv < t.nvec) unpack<W>(lds128(out + vv * 16), acc[u]);
          }
          for (int o = 1; o < nops; ++o) {
            uint4 r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int vv = v0 + u * kConsumers;
              if (vv < t.nvec) r[u] = lds128(slota(o) + vv * 16);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int vv = v0 + u * kConsumers;
              if (vv < t.nvec) {
                Acc tmp[VE];
                unpack<W>(r[u], tmp);
                acc_add<W>(acc[u], tmp);
              }
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int vv = v0 + u * kConsumers;
            if (vv >= t.nvec) continue;
            if (last_reduce && a.op == 1) acc_mean<W>(acc[u], a.inv_n, N);
            uint4 o4 = pack<W>(acc[u]);
            if (a.fault == 1 && me == 0 && b == 0 && nj == 0 && vv == 0) o4.x ^= 1u;  // negative control
            sts128(out + vv * 16, o4);
            if (last_reduce && !bb) {
              const unsigned long long el = t.e0 + (unsigned long long)vv * VE;
              const int nrem = (int)min((unsigned long long)VE, t.nel - (unsigned long long)vv * VE);
              store_user<DT, W>(buf, a.buf_off + cbase + el, nrem, o4, a.aligned != 0);
            }
          }
        }
      } else if (!bb) {
        // VA / H into a buffer the bulk store cannot take (cast, unaligned, ragged)
        for (int vv = ct; vv < t.nvec; vv += kConsumers) {
          const uint4 w = lds128(out + vv * 16);
          const unsigned long long el = t.e0 + (unsigned long long)vv * VE;
          const int nrem = (int)min((unsigned long long)VE, t.nel - (unsigned long long)vv * VE);
          store_user<DT, W>(buf, a.buf_off + cbase + el, nrem, w, a.aligned != 0);
        }
      }
      cs += nops;
      if (kind == kR || kind == kVR || (kind == kS0 && (DT != W || !(a.aligned && !ragged(a, t)))))
        fence_view_async_smem();  // my shared-memory writes -> the storer's TMA reads
      __syncwarp();
      if (lane == 0) atomicAdd(&s_done, 1);
      if (ct == 0) pstamp(a, blockIdx.x, nj, 2);
      ++nj;
    }
  }
  __syncthreads();
  if (tid == 0 && a.trace && blockIdx.x < kMaxLocal * 512)
    a.trace[((size_t)blockIdx.x * kPullTraceJobs + kPullTraceJobs - 1) * kPullTraceEv + 1] = gtimer();
  // the last CTA of this rank to finish advances the call epoch (device-resident, so the
  // call can be captured in a CUDA graph)
  if (tid == 0) {
    __threadfence();
    const uint32_t prev = atomicAdd(R->pull_ctr + 1, 1u);
    if (prev + 1 == (uint32_t)a.gsum) {
      R->pull_ctr[1] = 0;
      if (!s_abort) {
        __threadfence();
        st_release_gpu(R->pull_ctr, epoch + 1u);
      }
    }
  }
}

// Per-call header check: slot [parity][src] of u64 (seq << 32 | desc) in every rank's
// barrier region.  Double-buffered by call parity: a rank writes slot seq & 1 of call seq + 2
// only after it saw every peer's header of call seq + 1, i.e. after they read seq's.
__global__ void check_kernel(const RankDev* ranks, unsigned long long hdr_off, unsigned seq, unsigned desc,
                             unsigned long long timeout_ns) {
  const RankDev* R = ranks + blockIdx.x;
  const int t = threadIdx.x, N = R->N, me = R->rank, par = (int)(seq & 1u);
  const unsigned long long word = ((unsigned long long)seq << 32) | desc;
  auto slot = [&](int rank, int src) -> unsigned long long* {
    return reinterpret_cast<unsigned long long*>(R->ws[rank] + hdr_off) + par * kMaxRanks + src;
  };
  if (t < N && t != me) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(slot(t, me)), "l"(word) : "memory");
    const unsigned long long* f = slot(me, t);
    const unsigned long long deadline = gtimer() + timeout_ns;
    unsigned it = 0;
    while (true) {
      unsigned long long w;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(w) : "l"(f) : "memory");
      if ((unsigned)(w >> 32) == seq) {
        if ((unsigned)w != desc) atomicExch_system(R->err, 7 /* TORUS_ERR_MISMATCH */);
        break;
      }
      if ((++it & 255u) == 0 && gtimer() > deadline) {
        atomicCAS_system(R->err, 0, kErrTimeout);
        break;
      }
    }
  }
}

template <int DT, int W>
cudaError_t launch_pull_typed(const PullArgs& a, bool cooperative, cudaStream_t stream) {
  const dim3 grid(a.nlocal * a.gsum), block(kPullThreads);
  const size_t smem = pull_smem_bytes(a.nslots, a.slot_bytes);
  static int attr_done = 0;
  if (attr_done < (int)smem) {
    cudaError_t e = cudaFuncSetAttribute(torus_pull_kernel<DT, W>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_done = (int)smem;
  }
  if (cooperative) {
    void* args[] = {const_cast<PullArgs*>(&a)};
    return cudaLaunchCooperativeKernel((const void*)torus_pull_kernel<DT, W>, grid, block, args, smem,
                                       stream);
  }
  torus_pull_kernel<DT, W><<<grid, block, smem, stream>>>(a);
  return cudaGetLastError();
}

template <int DT, int W>
int pull_occupancy_typed(size_t smem) {
  int nb = 0;
  if (cudaFuncSetAttribute(torus_pull_kernel<DT, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, torus_pull_kernel<DT, W>, kPullThreads, smem) !=
      cudaSuccess)
    return 0;
  return nb;
}

}  // namespace

cudaError_t launch_pull(const PullArgs& a, int dtype, int wire, bool cooperative, cudaStream_t stream) {
  if (dtype == wire) {
    switch (dtype) {
      case DT_F32: return launch_pull_typed<DT_F32, DT_F32>(a, cooperative, stream);
      case DT_F16: return launch_pull_typed<DT_F16, DT_F16>(a, cooperative, stream);
      case DT_BF16: return launch_pull_typed<DT_BF16, DT_BF16>(a, cooperative, stream);
      case DT_I32: return launch_pull_typed<DT_I32, DT_I32>(a, cooperative, stream);
    }
  } else if (dtype == DT_F32 && wire == DT_F16) {
    return launch_pull_typed<DT_F32, DT_F16>(a, cooperative, stream);
  } else if (dtype == DT_F32 && wire == DT_BF16) {
    return launch_pull_typed<DT_F32, DT_BF16>(a, cooperative, stream);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_check(const RankDev* ranks, int nlocal, unsigned long long hdr_off, unsigned seq,
                         unsigned desc, unsigned long long timeout_ns, cudaStream_t stream) {
  if (nlocal > 1) {
    void* args[] = {const_cast<RankDev**>(&ranks), &hdr_off, &seq, &desc, &timeout_ns};
    return cudaLaunchCooperativeKernel((const void*)check_kernel, dim3(nlocal), dim3(kMaxRanks), args, 0, stream);
  }
  check_kernel<<<1, kMaxRanks, 0, stream>>>(ranks, hdr_off, seq, desc, timeout_ns);
  return cudaGetLastError();
}

int pull_ctas_per_sm(size_t smem) {
  int m = pull_occupancy_typed<DT_F32, DT_F16>(smem);
  m = std::min(m, pull_occupancy_typed<DT_F16, DT_F16>(smem));
  m = std::min(m, pull_occupancy_typed<DT_F32, DT_F32>(smem));
  m = std::min(m, pull_occupancy_typed<DT_BF16, DT_BF16>(smem));
  m = std::min(m, pull_occupancy_typed<DT_I32, DT_I32>(smem));
  m = std::min(m, pull_occupancy_typed<DT_F32, DT_BF16>(smem));
  return m;
}

}  // namespace torus
