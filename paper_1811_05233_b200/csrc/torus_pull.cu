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
// (SURVEY C3-C10), so every dtype is bit-exact against oracle/torus_oracle.c.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "torus_device.cuh"

namespace torus {
namespace {

constexpr int kPullThreads = 192;   // warp 0 producer, warp 1 signaler, warps 2..5 consumers
constexpr int kConsumerWarps = 4;
constexpr int kConsumers = kConsumerWarps * 32;

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
  unsigned long long cl, sl;
  qpart(a.n, X, a.q, j, &t.co, &cl);
  qpart(cl, Y, a.q, s, &t.cs, &sl);
  const unsigned long long per = (unsigned long long)a.TV * a.q;
  const unsigned long long st = (unsigned long long)k * per;
  t.ok = st < sl;
  t.e0 = t.cs + st;
  t.nel = t.ok ? min(per, sl - st) : 0;
  t.nvec = (int)((t.nel + a.q - 1) / a.q);
  return t;
}

// the own operand of a reduce can be read straight from the user buffer (no S0 copy)
// when the buffer holds wire values, is 16-byte aligned and the tile has no ragged tail
template <int DT, int W>
__device__ __forceinline__ bool own_from_buf(const PullArgs& a, const Tile& t) {
  return DT == W && a.aligned && (t.nel % (unsigned long long)a.q) == 0;
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

enum PullKind { kS0 = 0, kR = 1, kVR = 2, kVA = 3, kH = 4, kKinds = 5 };

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
    case kS0: return a.Kmax * (X > 1 ? X * Y : Y);
    case kR: return a.Kmax * Y;
    case kVR: return a.Kmax;
    case kVA: return a.Kmax * (Y - 1);
    default: return a.Kmax * (X - 1) * Y;
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
  if (jb.ok && kind == kS0) {
    // S0 copies what a peer reads in the first reduce phase: the chunks of my row peers
    // (X > 1) or the sub-chunks of my column peers (X == 1), plus my own tiles the
    // reduce cannot take from the user buffer directly
    const bool own = X > 1 ? (jb.j == c) : (jb.s == rho);
    if (own && own_from_buf<DT, W>(a, jb.t)) jb.ok = false;
  }
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

// ------------------------------------------------------------------------------------
// the kernel
// ------------------------------------------------------------------------------------
template <int DT, int W>
__global__ void __launch_bounds__(kPullThreads) torus_pull_kernel(const PullArgs a) {
  using Acc = typename Wire<W>::Acc;
  constexpr int VE = Wire<W>::VE;
  constexpr int SW = kVecBytes / VE;           // bytes per wire element
  constexpr int DB = sizeof(typename Elem<DT>::T);

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
  __shared__ int s_done;      // consumer-warp job completions (signaler polls)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    s_epoch = ld_acquire_gpu(R->pull_ctr);
    s_abort = 0;
    s_done = 0;
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint32_t epoch = s_epoch;
  const uint32_t v = epoch + 1u;               // flag value of this call
  const int par = (int)(epoch & 1u);
  char* const myws = R->ws[me];
  uint32_t* const myflags = reinterpret_cast<uint32_t*>(myws + a.flag_off);
  auto flag_at = [&](int rank, size_t idx) -> uint32_t* {
    return reinterpret_cast<uint32_t*>(R->ws[rank] + a.flag_off) + idx;
  };
  const int njobs = job_count(a, kind, X, Y);
  const int nops = job_nops(kind, X, Y);

  if (warp == 0) {
    // =============================== producer =====================================
    if (lane == 0) {
      const unsigned long long deadline = gtimer() + a.timeout_ns;
      // Presence: CTA 0 of S0 tells every row and column peer that this rank has entered
      // the call, and does not finish before all of them have -- so every call observes
      // every peer, which the parity double-buffering relies on even when a short round
      // leaves some sub-chunks (and their flags) empty.
      const bool presence = (kind == kS0 && b == 0);
      if (presence) {
        for (int jj = 1; jj < X; ++jj) st_relaxed_sys(flag_at(rho * X + (c + jj) % X, a.fl_pres + me), v);
        for (int ii = 1; ii < Y; ++ii) st_relaxed_sys(flag_at(((rho + ii) % Y) * X + c, a.fl_pres + me), v);
      }
      uint32_t ps = 0;  // operand loads issued (ring position)
      for (int J = b; J < njobs; J += G) {
        const Job jb = job_of<DT, W>(a, kind, J, X, Y, rho, c);
        if (!jb.ok) continue;
        // -- wait for this job's inputs --
        bool ok = true;
        auto need = [&](size_t idx) {
          if (!ok) return;
          const uint32_t* f = myflags + idx;
          unsigned spin = 0;
          while ((int32_t)(ld_relaxed_sys(f) - v) < 0) {
            __nanosleep(32);
            if ((++spin & 255u) == 0 && (gtimer() > deadline || *(volatile int*)&s_abort)) {
              ok = false;
              return;
            }
          }
          (void)ld_acquire_sys(f);  // synchronizes with the peer's fence + flag store
        };
        const bool ownbuf = own_from_buf<DT, W>(a, jb.t);
        if (kind == kR) {
          for (int j = 0; j < X; ++j)
            if (j != c || !ownbuf) need(fl_win(a, Y, j, jb.s, jb.k));
        } else if (kind == kVR) {
          for (int i = 0; i < Y; ++i) {
            if (X > 1) need(fl_p1(a, i, jb.k));
            else if (i != rho || !ownbuf) need(fl_win(a, Y, i, 0, jb.k));
          }
        } else if (kind == kVA) {
          need(fl_v(a, jb.i, jb.k));
        } else if (kind == kH) {
          need(fl_c(a, Y, jb.j, jb.s, jb.k));
        }
        if (!ok) {
          atomicExch_system(R->err, kErrTimeout);
          s_abort = 1;
          break;
        }
        fence_proxy_async();  // generic-proxy acquire before the async-proxy (TMA) reads
        // -- issue the operand loads (fold order) --
        const bool direct = (kind == kS0) && !(a.aligned && (jb.t.nel % a.q) == 0);
        for (int o = 0; o < nops; ++o) {
          const uint32_t slot = ps % NS, use = ps / NS;
          ++ps;
          if (use > 0 && !mbar_wait_abortable(&empty[slot], (use - 1) & 1u, &s_abort)) { ok = false; break; }
          const char* src = nullptr;
          uint32_t bytes = (uint32_t)jb.t.nvec * kVecBytes;
          if (kind == kS0) {
            // my buffer's tile (dtype bytes)
            bytes = (uint32_t)jb.t.nvec * VE * DB;
            src = reinterpret_cast<const char*>(buf) + (a.buf_off + jb.t.co + jb.t.e0) * DB;
          } else if (kind == kR) {
            const int j = (c + 1 + o) % X;  // fold order: columns c+1, ..., c
            if (j == c && ownbuf)
              src = reinterpret_cast<const char*>(buf) + (a.buf_off + jb.t.co + jb.t.e0) * DB;
            else
              src = R->ws[rho * X + j] + a.win_off[par] + (jb.t.co + jb.t.e0) * SW;
          } else if (kind == kVR) {
            const int i = (rho + 1 + o) % Y;  // fold order: rows rho+1, ..., rho
            if (X > 1)
              src = R->ws[i * X + c] + a.p1_off[par] + jb.t.e0 * SW;
            else if (i == rho && ownbuf)
              src = reinterpret_cast<const char*>(buf) + (a.buf_off + jb.t.co + jb.t.e0) * DB;
            else
              src = R->ws[i * X + c] + a.win_off[par] + (jb.t.co + jb.t.e0) * SW;
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
        if (!ok) {
          s_abort = 1;
          break;
        }
      }
      if (presence && !*(volatile int*)&s_abort) {
        bool ok = true;
        auto seen = [&](int peer) {
          const uint32_t* f = myflags + a.fl_pres + peer;
          unsigned spin = 0;
          while (ok && (int32_t)(ld_relaxed_sys(f) - v) < 0) {
            __nanosleep(64);
            if ((++spin & 255u) == 0 && gtimer() > deadline) ok = false;
          }
        };
        for (int jj = 1; jj < X; ++jj) seen(rho * X + (c + jj) % X);
        for (int ii = 1; ii < Y; ++ii) seen(((rho + ii) % Y) * X + c);
        if (!ok) atomicExch_system(R->err, kErrTimeout);
      }
    }
  } else if (warp == 1) {
    // =============================== signaler =====================================
    // After the consumers finish job J (all its stores issued, local), one system-scope
    // fence publishes every completed job, then the flag stores tell the consumers of
    // each tile that it may be pulled.  Jobs complete in order; one fence covers all
    // jobs completed so far.
    if (lane == 0 && kind != kH) {
      int signaled = 0;  // jobs of this CTA signaled so far (valid jobs only)
      int J = b;
      while (true) {
        // next valid job
        Job jb;
        jb.ok = false;
        for (; J < njobs; J += G) {
          jb = job_of<DT, W>(a, kind, J, X, Y, rho, c);
          if (jb.ok) break;
        }
        if (J >= njobs) break;
        bool aborted = false;
        while (ld_acquire_cta(&s_done) < kConsumerWarps * (signaled + 1)) {
          if (*(volatile int*)&s_abort) { aborted = true; break; }
          __nanosleep(20);
        }
        if (aborted) break;
        fence_proxy_async();
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        // signal every job completed so far (at least this one)
        const int done = ld_acquire_cta(&s_done) / kConsumerWarps;
        while (true) {
          // ---- raise the flags of job jb ----
          if (kind == kS0) {
            if (X > 1) st_relaxed_sys(flag_at(rho * X + jb.j, fl_win(a, Y, c, jb.s, jb.k)), v);
            else st_relaxed_sys(flag_at(jb.s * X, fl_win(a, Y, rho, 0, jb.k)), v);
          } else if (kind == kR) {
            if (Y > 1) {
              st_relaxed_sys(flag_at(jb.s * X + c, fl_p1(a, rho, jb.k)), v);
            } else {
              for (int jj = 1; jj < X; ++jj)
                st_relaxed_sys(flag_at(rho * X + (c + jj) % X, fl_c(a, Y, c, 0, jb.k)), v);
            }
          } else if (kind == kVR) {
            for (int ii = 1; ii < Y; ++ii)
              st_relaxed_sys(flag_at(((rho + ii) % Y) * X + c, fl_v(a, rho, jb.k)), v);
            for (int jj = 1; jj < X; ++jj)
              st_relaxed_sys(flag_at(rho * X + (c + jj) % X, fl_c(a, Y, c, rho, jb.k)), v);
          } else if (kind == kVA) {
            for (int jj = 1; jj < X; ++jj)
              st_relaxed_sys(flag_at(rho * X + (c + jj) % X, fl_c(a, Y, c, jb.i, jb.k)), v);
          }
          ++signaled;
          J += G;
          if (signaled >= done) break;
          jb.ok = false;
          for (; J < njobs; J += G) {
            jb = job_of<DT, W>(a, kind, J, X, Y, rho, c);
            if (jb.ok) break;
          }
          if (J >= njobs) break;
        }
      }
    }
  } else {
    // =============================== consumers ====================================
    const int ct = tid - 64;  // 0 .. kConsumers-1
    uint32_t cs = 0;          // operands consumed (ring position)
    for (int J = b; J < njobs; J += G) {
      const Job jb = job_of<DT, W>(a, kind, J, X, Y, rho, c);
      if (!jb.ok) continue;
      const uint32_t slot0 = cs;
      bool ok = true;
      for (int o = 0; o < nops && ok; ++o)
        ok = mbar_wait_abortable(&full[(slot0 + o) % NS], ((slot0 + o) / NS) & 1u, &s_abort);
      if (!ok) break;
      const Tile& t = jb.t;
      const unsigned long long cbase = t.co;                  // chunk offset in the round
      auto slotp = [&](int o) -> const unsigned char* {
        return smem + (size_t)((slot0 + o) % NS) * a.slot_bytes;
      };
      if (kind == kS0) {
        // cast/copy my buffer's tile into win (C1: w = to_wire(in))
        const bool direct = !(a.aligned && (t.nel % a.q) == 0);
        char* dst = myws + a.win_off[par] + (cbase + t.e0) * SW;
        for (int vv = ct; vv < t.nvec; vv += kConsumers) {
          uint4 w;
          if (direct) {
            const unsigned long long el = t.e0 + (unsigned long long)vv * VE;
            const int nrem = (int)min((unsigned long long)VE, t.nel - (unsigned long long)vv * VE);
            w = load_user<DT, W>(buf, a.buf_off + cbase + el, nrem, a.aligned != 0);
          } else if constexpr (DT == W) {
            w = *reinterpret_cast<const uint4*>(slotp(0) + (size_t)vv * 16);
          } else {
            const float4* f = reinterpret_cast<const float4*>(slotp(0) + (size_t)vv * 32);
            const float4 f0 = f[0], f1 = f[1];
            const float ff[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
            w = pack<W>(ff);
          }
          st_ws(dst + (size_t)vv * 16, w);
        }
      } else if (kind == kR || kind == kVR) {
        // fold the operands in ring order (loaded in that order), f32 / u32 accumulation
        const bool last_reduce = (kind == kVR) || (Y == 1);
        for (int vv = ct; vv < t.nvec; vv += kConsumers) {
          Acc acc[VE];
          {
            Acc tmp[VE];
            unpack<W>(*reinterpret_cast<const uint4*>(slotp(0) + (size_t)vv * 16), acc);
            for (int o = 1; o < nops; ++o) {
              unpack<W>(*reinterpret_cast<const uint4*>(slotp(o) + (size_t)vv * 16), tmp);
              acc_add<W>(acc, tmp);
            }
          }
          const unsigned long long el = t.e0 + (unsigned long long)vv * VE;  // in chunk
          if (!last_reduce) {
            st_ws(myws + a.p1_off[par] + el * SW, pack<W>(acc));
          } else {
            if (a.op == 1) acc_mean<W>(acc, a.inv_n, N);
            const uint4 out = pack<W>(acc);
            if (X > 1 || Y > 1) st_ws(myws + a.chunk_off[par] + el * SW, out);
            const int nrem = (int)min((unsigned long long)VE, t.nel - (unsigned long long)vv * VE);
            store_user<DT, W>(buf, a.buf_off + cbase + el, nrem, out, a.aligned != 0);
          }
        }
      } else {
        // VA / H: copy a peer's final tile into my buffer (and my chunk region for VA,
        // which my row peers pull next)
        for (int vv = ct; vv < t.nvec; vv += kConsumers) {
          const uint4 w = *reinterpret_cast<const uint4*>(slotp(0) + (size_t)vv * 16);
          const unsigned long long el = t.e0 + (unsigned long long)vv * VE;
          if (kind == kVA && X > 1) st_ws(myws + a.chunk_off[par] + el * SW, w);
          const int nrem = (int)min((unsigned long long)VE, t.nel - (unsigned long long)vv * VE);
          store_user<DT, W>(buf, a.buf_off + cbase + el, nrem, w, a.aligned != 0);
        }
      }
      cs += nops;
      __syncwarp();
      if (lane == 0) {
        for (int o = 0; o < nops; ++o) mbar_arrive1(&empty[(slot0 + o) % NS]);
        __threadfence_block();
        atomicAdd(&s_done, 1);
      }
    }
  }
  __syncthreads();
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
