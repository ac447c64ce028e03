// torus_kernels.cu -- sm_100a kernels of the 2D-Torus all-reduce (Sec. 2.2).
//
//   torus_kernel      (TORUS_KERNEL=push; the round-1 default) one fused launch per round: the paper's three steps as a
//                     5-stage tile wavefront (A push / B row fold / C column fold + mean /
//                     D column all-gather / E row all-gather), control warp + 15 data
//                     warps, 128-bit LDG/STG over NVLink, one system fence per iteration
//   torus_tma_kernel  (TORUS_KERNEL=tma) the same protocol with TMA bulk copies, a
//                     producer / consumer / storer / poller / publisher split and a signal
//                     CTA that fences from a quiet SM (parity-green, latency-bound today)
//   castscale_kernel  the N = 1 degenerate case (fused cast round trip)
//   barrier_kernel    init / destroy / algorithm-switch barrier
// (the pull kernel, the default, is torus_pull.cu; baselines and probes are in
// torus_baselines.cu; the small-message kernels in torus_ll.cu)
// Phases in the paper's words: "Firstly, reduce-scatter is performed horizontally. Then,
// all-reduce is performed vertically. Finally, all-gather is performed horizontally."
// Fold order, partition and rounding points follow the oracle, so every
// dtype is bit-exact.  No tensor cores: a bandwidth-bound reduction, not a contraction.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "torus_device.cuh"

namespace torus {
namespace {


// ------------------------------------------------------------------------------------
// pipeline geometry: CTA b owns slice b of every sub-chunk; tile t of that slice is the
// vector range [p0, p1) below.  Host and every rank compute the same T (tile_geometry).
// ------------------------------------------------------------------------------------
struct Piece {
  unsigned long long co, cl;  // chunk j: offset / length in the round (elements)
  unsigned long long so;      // sub-chunk s: offset inside chunk j (elements)
  unsigned long long p0, p1;  // vectors of the sub-chunk handled in this tile
};

__device__ __forceinline__ Piece make_piece(unsigned long long n, int X, int Y, int q, int G,
                                            int b, int TV, int j, int s, int t) {
  Piece p;
  unsigned long long sl;
  qpart(n, X, q, j, &p.co, &p.cl);
  qpart(p.cl, Y, q, s, &p.so, &sl);
  const unsigned long long nv = (sl + q - 1) / q;
  const unsigned long long va = nv * (unsigned long long)b / (unsigned long long)G;
  const unsigned long long vz = nv * (unsigned long long)(b + 1) / (unsigned long long)G;
  const unsigned long long a0 = va + (unsigned long long)t * (unsigned long long)TV;
  p.p0 = a0 < vz ? a0 : vz;
  p.p1 = (a0 + TV) < vz ? (a0 + TV) : vz;
  return p;
}

constexpr int kCtrlThreads = 32;                     // warp 0: flags, fences, signals
#ifndef TORUS_LDG_THREADS
#define TORUS_LDG_THREADS 512
#endif
constexpr int kLdgThreads = TORUS_LDG_THREADS;       // threads per CTA of torus_kernel
constexpr int kLdgCtasPerSm = 512 / TORUS_LDG_THREADS;
constexpr int kWorkers = kLdgThreads - kCtrlThreads; // warps 1..: data movement
#ifndef TORUS_UNROLL
#define TORUS_UNROLL 2
#endif
#ifndef TORUS_UNROLL_FOLD
#define TORUS_UNROLL_FOLD 2
#endif
constexpr int kUnroll = TORUS_UNROLL;                // vectors per worker per pass (copies)
constexpr int kUnrollFold = TORUS_UNROLL_FOLD;       // vectors per worker per pass (folds)

// Stages of the wavefront (iteration `it` runs A on tile it, B on it-1, ... E on it-4).
enum Stage { kA = 0, kB = 1, kC = 2, kD = 3, kE = 4, kStages = 5 };
// Trace events per iteration (TORUS_TRACE=1): control lane 0 stamps 0 poll start,
// 1 poll done, 2 DONE(it-1) synced, 3 READY(it) arrived, 4 raise(it-1) done; worker
// warp 1 lane 0 stamps 5 READY passed, 6 work done.
__device__ __forceinline__ void stamp(unsigned long long* tr, int b, int it, int ev) {
  if (tr && it < kTraceIters) tr[((size_t)b * kTraceIters + it) * kTraceEvents + ev] = gtimer();
}

// named barriers between the control warp and the workers (0 is __syncthreads)
constexpr int kBarReady = 1;  // control -> workers: inputs of iteration it are visible
constexpr int kBarDone = 2;   // workers -> control: iteration it's data is written
__device__ __forceinline__ void bar_sync(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kLdgThreads) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(kLdgThreads) : "memory");
}

// ------------------------------------------------------------------------------------
// the fused, tile-pipelined torus kernel
// ------------------------------------------------------------------------------------
//   stage A (tile t)   phase 1 push: cast my buffer's share of every row peer's chunk
//                      and store it into that peer's h_in[c]                -> flag H
//   stage B (t-1)      phase 1 fold: wait H; fold the X shares of my chunk in ring order;
//                      Y > 1: push the rounded P1 into v_in[rho] of the column owner
//                      of each sub-chunk (-> flag V); Y == 1: mean, round, write my chunk
//                      slot and my buffer
//   stage C (t-2)      phase 2 reduce-scatter: wait V; fold the Y rows' P1 in ring order,
//                      mean, round once; write my chunk slot + my buffer      -> flag AG
//   stage D (t-3)      phase 2 all-gather: wait AG; pull the column peers' reduced
//                      sub-chunks into my buffer (+ my chunk slot when X > 1) -> flag R
//   stage E (t-4)      phase 3 all-gather: wait R; pull the row peers' completed chunks
//                      into my buffer (wire -> dtype cast fused)
// Every wait is on flags peers raise one iteration earlier, so in steady state no stage
// stalls on a cross-GPU round trip; the control warp polls the next stage's flags and
// fences/raises the previous stage's flags while the workers move data.
template <int DT, int W, bool MULTI>
__global__ void __launch_bounds__(kLdgThreads, kLdgCtasPerSm) torus_kernel(const LaunchArgs a) {
  using Acc = typename Wire<W>::Acc;
  constexpr int VE = Wire<W>::VE;
  constexpr int SW = kVecBytes / VE;  // bytes per wire element

  const int lr = blockIdx.x / a.G;
  const int b = blockIdx.x - lr * a.G;
  const RankDev* __restrict__ R = a.ranks + lr;
  const int X = R->X, Y = R->Y, N = R->N, rho = R->rho, c = R->c, me = R->rank;
  const int G = a.G, q = a.q, T = a.T, TV = a.tile_vecs;
  const int tid = threadIdx.x;
  const unsigned long long n = a.n;
  const bool aligned = a.aligned != 0;
  void* const buf = a.buf[lr];
  char* const myws = R->ws[me];
  char* const hin = myws + a.hin_off;
  char* const vin = myws + a.vin_off;
  char* const chunk = myws + a.chunk_off;
  const MultiSeg* const segs = MULTI ? a.segs + (size_t)lr * a.nseg : nullptr;
  // the user buffer: one flat buffer, or (MULTI, NEXT-1) the concatenation of a bucket's
  // tensors -- a separate instantiation, so the flat path keeps its register budget
  int seg_hint = 0;  // MULTI: this thread's last segment
  auto uload = [&](unsigned long long e, int nrem) -> uint4 {
    if constexpr (MULTI) return load_user_seg<DT, W>(segs, a.nseg, e, nrem, seg_hint);
    else return load_user<DT, W>(buf, e, nrem, aligned);
  };
  auto ustore = [&](unsigned long long e, int nrem, uint4 v) {
    if constexpr (MULTI) store_user_seg<DT, W>(segs, a.nseg, e, nrem, v, seg_hint);
    else store_user<DT, W>(buf, e, nrem, v, aligned);
  };

  __shared__ uint32_t s_seq;
  __shared__ int s_abort;
  if (tid == 0) {
    s_seq = R->epoch[b];
    s_abort = 0;
  }
  __syncthreads();
  const uint32_t seq = s_seq;

  // Active stages of this grid in pipeline order.  Stage p works on tile it - 2p in
  // iteration it, so every flag it consumes was raised by its peers one full iteration
  // earlier: the ~3 us cross-GPU flag latency hides behind an iteration of data movement.
  int kinds[kStages];
  int P = 0;
  if (X > 1) kinds[P++] = kA;
  kinds[P++] = kB;
  if (Y > 1) {
    kinds[P++] = kC;
    kinds[P++] = kD;
  }
  if (X > 1) kinds[P++] = kE;
  // Stage distance: 2 (flags hide behind an iteration of data) when the call has several
  // tiles; 1 for single-tile (small) calls, where latency is all there is -- each stage
  // then waits on the previous one directly and the control warp raises before it polls.
  const int SD = (T == 1 || a.sd1) ? 1 : 2;
  const int iters = T + SD * (P - 1);

  if (tid < kCtrlThreads) {
    // =============================== control warp ===============================
    const int lane = tid;
    const unsigned long long deadline = gtimer() + a.timeout_ns;
    auto flagp = [&](char* ws, int kind, int src) -> uint32_t* {
      return reinterpret_cast<uint32_t*>(ws) + ((size_t)(kind * kMaxDim + src) * G + b);
    };
    // Visit the flags stage k at tile t consumes (in) or produces (!in).
    auto for_flags = [&](int k, int t, bool in, auto visit) {
      int kind = -1, cnt = 0;
      bool row = true;
      switch (k) {
        case kA:
          if (!in) { kind = kFlagH; cnt = X - 1; row = true; }
          break;
        case kB:
          if (in) {
            if (X > 1) { kind = kFlagH; cnt = X - 1; row = true; }
          } else if (Y > 1) {
            kind = kFlagV; cnt = Y - 1; row = false;
          } else if (X > 1) {
            kind = kFlagR; cnt = X - 1; row = true;  // Y == 1: B wrote the final chunk
          }
          break;
        case kC:
          kind = in ? kFlagV : kFlagAG; cnt = Y - 1; row = false;
          break;
        case kD:
          if (in) { kind = kFlagAG; cnt = Y - 1; row = false; }
          else if (X > 1) { kind = kFlagR; cnt = X - 1; row = true; }
          break;
        default:
          if (in) { kind = kFlagR; cnt = X - 1; row = true; }
          break;
      }
      const uint32_t v = seq + (uint32_t)t + 1u;
      for (int l = 0; l < cnt; ++l) {
        const int other = row ? (c + 1 + l) % X : (rho + 1 + l) % Y;
        const int peer = row ? rho * X + other : other * X + c;
        visit(in ? flagp(myws, kind, other) : flagp(R->ws[peer], kind, row ? c : rho), v);
      }
    };
    auto poll_iter = [&](int it) -> bool {
      bool ok = true;
      int e = 0;
      for (int p = 0; p < P; ++p) {
        const int t = it - SD * p;
        if (t < 0 || t >= T) continue;
        for_flags(kinds[p], t, true, [&](uint32_t* f, uint32_t v) {
          if ((e++ & 31) == lane && ok) ok = wait_flag_ge(f, v, deadline, a.poll_sleep, R->err);
        });
      }
      return __all_sync(0xffffffffu, ok);
    };
    // one system-scope fence for all the flags an iteration raises
    auto raise_iter = [&](int it, bool fence = true) {
      if (fence) asm volatile("fence.acq_rel.sys;" ::: "memory");
      int e = 0;
      for (int p = 0; p < P; ++p) {
        const int t = it - SD * p;
        if (t < 0 || t >= T) continue;
        for_flags(kinds[p], t, false, [&](uint32_t* f, uint32_t v) {
          if ((e++ & 31) == lane) st_relaxed_sys(f, v);
        });
      }
    };
    unsigned long long* const tr = (lane == 0 && lr == 0) ? a.trace : nullptr;
    for (int it = 0; it < iters; ++it) {
      stamp(tr, b, it, 0);
      if (SD == 1 && it > 0) {            // latency mode: publish it-1 before waiting on it
        bar_sync(kBarDone);
        raise_iter(it - 1);
      }
      const bool ok = poll_iter(it);      // inputs: raised by peers in iteration <= it-1
      stamp(tr, b, it, 1);
      if (SD == 2 && it > 0) bar_sync(kBarDone);  // workers finished iteration it-1
      stamp(tr, b, it, 2);
      if (!ok) {
        if (lane == 0) {
          atomicCAS_system(R->err, 0, kErrTimeout);
          s_abort = 1;
        }
        __syncwarp();
        bar_arrive(kBarReady);
        return;
      }
      if (SD == 2 && it > 0 && a.fence_early) {  // fence on it-1's stores only, then go
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        bar_arrive(kBarReady);
        stamp(tr, b, it, 3);
        raise_iter(it - 1, false);
      } else {
        bar_arrive(kBarReady);              // workers start iteration it ...
        stamp(tr, b, it, 3);
        if (SD == 2 && it > 0) raise_iter(it - 1);  // ... while the fence for it-1 drains
      }
      stamp(tr, b, it, 4);
    }
    bar_sync(kBarDone);
    raise_iter(iters - 1);
  } else {
    // =============================== worker warps ===============================
    const int w = tid - kCtrlThreads;
    unsigned long long* const tr = (w == 0 && lr == 0) ? a.trace : nullptr;
    for (int it = 0; it < iters; ++it) {
      bar_sync(kBarReady);
      stamp(tr, b, it, 5);
      if (*(volatile int*)&s_abort) return;
      for (int p = 0; p < P; ++p) {
        const int t = it - SD * p;
        if (t < 0 || t >= T) continue;
        const int k = kinds[p];
        if (k == kA) {
          // ---- phase 1 push ----
          for (int jj = 1; jj < X; ++jj) {
            const int j = (c + jj) % X;
            char* const dst = R->ws[rho * X + j] + a.hin_off + (size_t)c * a.hin_stride;
            for (int s = 0; s < Y; ++s) {
              const Piece p = make_piece(n, X, Y, q, G, b, TV, j, s, t);
              for (unsigned long long v0 = p.p0 + w; v0 < p.p1; v0 += kUnroll * kWorkers) {
                uint4 r[kUnroll];
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                  const unsigned long long v = v0 + (unsigned long long)u * kWorkers;
                  if (v < p.p1) {
                    const unsigned long long el = p.so + v * VE;
                    const int nrem = (int)min((unsigned long long)VE, p.cl - el);
                    r[u] = uload(a.buf_off + p.co + el, nrem);
                  }
                }
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                  const unsigned long long v = v0 + (unsigned long long)u * kWorkers;
                  if (v < p.p1) st_ws(dst + (p.so + v * VE) * SW, r[u]);
                }
              }
            }
          }
        } else if (k == kB) {
          // ---- phase 1 fold: columns c+1, ..., c ----
          for (int s = 0; s < Y; ++s) {
            const Piece p = make_piece(n, X, Y, q, G, b, TV, c, s, t);
            char* const dst = R->ws[s * X + c] + a.vin_off + (size_t)rho * a.vin_stride;
            for (unsigned long long v0 = p.p0 + w; v0 < p.p1; v0 += kUnrollFold * kWorkers) {
              Acc acc[kUnrollFold][VE];
              for (int kk = 1; kk <= X; ++kk) {
                const int j = (c + kk) % X;
                uint4 r[kUnrollFold];
#pragma unroll
                for (int u = 0; u < kUnrollFold; ++u) {
                  const unsigned long long v = v0 + (unsigned long long)u * kWorkers;
                  if (v < p.p1) {
                    const unsigned long long el = p.so + v * VE;
                    if (j == c) {
                      const int nrem = (int)min((unsigned long long)VE, p.cl - el);
                      r[u] = uload(a.buf_off + p.co + el, nrem);
                    } else {
                      r[u] = ld_ws(hin + (size_t)j * a.hin_stride + el * SW);
                    }
                  } else {
                    r[u] = make_uint4(0, 0, 0, 0);
                  }
                }
#pragma unroll
                for (int u = 0; u < kUnrollFold; ++u) {
                  Acc tmp[VE];
                  unpack<W>(r[u], tmp);
                  if (kk == 1) {
#pragma unroll
                    for (int i = 0; i < VE; ++i) acc[u][i] = tmp[i];
                  } else {
                    acc_add<W>(acc[u], tmp);
                  }
                }
              }
#pragma unroll
              for (int u = 0; u < kUnrollFold; ++u) {
                const unsigned long long v = v0 + (unsigned long long)u * kWorkers;
                if (v >= p.p1) continue;
                const unsigned long long el = p.so + v * VE;
                if (Y > 1) {
                  st_ws(dst + v * VE * SW, pack<W>(acc[u]));
                } else {  // last reduce phase: mean, round once, final
                  if (a.op == 1) acc_mean<W>(acc[u], a.inv_n, N);
                  const uint4 out = pack<W>(acc[u]);
                  if (X > 1) st_ws(chunk + el * SW, out);
                  const int nrem = (int)min((unsigned long long)VE, p.cl - el);
                  ustore(a.buf_off + p.co + el, nrem, out);
                }
              }
            }
          }
        } else if (k == kC) {
          // ---- phase 2 reduce-scatter: rows rho+1, ..., rho, mean, round ----
          const Piece p = make_piece(n, X, Y, q, G, b, TV, c, rho, t);
          for (unsigned long long v0 = p.p0 + w; v0 < p.p1; v0 += kUnrollFold * kWorkers) {
            Acc acc[kUnrollFold][VE];
            for (int kk = 1; kk <= Y; ++kk) {
              const int i = (rho + kk) % Y;
              uint4 r[kUnrollFold];
#pragma unroll
              for (int u = 0; u < kUnrollFold; ++u) {
                const unsigned long long v = v0 + (unsigned long long)u * kWorkers;
                r[u] = (v < p.p1) ? ld_ws(vin + (size_t)i * a.vin_stride + v * VE * SW)
                                  : make_uint4(0, 0, 0, 0);
              }
#pragma unroll
              for (int u = 0; u < kUnrollFold; ++u) {
                Acc tmp[VE];
                unpack<W>(r[u], tmp);
                if (kk == 1) {
#pragma unroll
                  for (int i2 = 0; i2 < VE; ++i2) acc[u][i2] = tmp[i2];
                } else {
                  acc_add<W>(acc[u], tmp);
                }
              }
            }
#pragma unroll
            for (int u = 0; u < kUnrollFold; ++u) {
              const unsigned long long v = v0 + (unsigned long long)u * kWorkers;
              if (v >= p.p1) continue;
              if (a.op == 1) acc_mean<W>(acc[u], a.inv_n, N);
              const uint4 out = pack<W>(acc[u]);
              const unsigned long long el = p.so + v * VE;
              st_ws(chunk + el * SW, out);
              const int nrem = (int)min((unsigned long long)VE, p.cl - el);
              ustore(a.buf_off + p.co + el, nrem, out);
            }
          }
        } else if (k == kD) {
          // ---- phase 2 all-gather: pull the column peers' reduced sub-chunks ----
          for (int ii = 1; ii < Y; ++ii) {
            const int i = (rho + ii) % Y;
            const char* const src = R->ws[i * X + c] + a.chunk_off;
            const Piece p = make_piece(n, X, Y, q, G, b, TV, c, i, t);
            for (unsigned long long v0 = p.p0 + w; v0 < p.p1; v0 += kUnroll * kWorkers) {
              uint4 r[kUnroll];
#pragma unroll
              for (int u = 0; u < kUnroll; ++u) {
                const unsigned long long v = v0 + (unsigned long long)u * kWorkers;
                if (v < p.p1) r[u] = ld_ws(src + (p.so + v * VE) * SW);
              }
#pragma unroll
              for (int u = 0; u < kUnroll; ++u) {
                const unsigned long long v = v0 + (unsigned long long)u * kWorkers;
                if (v >= p.p1) continue;
                const unsigned long long el = p.so + v * VE;
                if (X > 1) st_ws(chunk + el * SW, r[u]);
                const int nrem = (int)min((unsigned long long)VE, p.cl - el);
                ustore(a.buf_off + p.co + el, nrem, r[u]);
              }
            }
          }
        } else {
          // ---- phase 3 all-gather: pull the row peers' completed chunks ----
          for (int jj = 1; jj < X; ++jj) {
            const int j = (c + jj) % X;
            const char* const src = R->ws[rho * X + j] + a.chunk_off;
            for (int s = 0; s < Y; ++s) {
              const Piece p = make_piece(n, X, Y, q, G, b, TV, j, s, t);
              for (unsigned long long v0 = p.p0 + w; v0 < p.p1; v0 += kUnroll * kWorkers) {
                uint4 r[kUnroll];
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                  const unsigned long long v = v0 + (unsigned long long)u * kWorkers;
                  if (v < p.p1) r[u] = ld_ws(src + (p.so + v * VE) * SW);
                }
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                  const unsigned long long v = v0 + (unsigned long long)u * kWorkers;
                  if (v >= p.p1) continue;
                  const unsigned long long el = p.so + v * VE;
                  const int nrem = (int)min((unsigned long long)VE, p.cl - el);
                  ustore(a.buf_off + p.co + el, nrem, r[u]);
                }
              }
            }
          }
        }
      }
      stamp(tr, b, it, 6);
      bar_arrive(kBarDone);
    }
  }
  __syncthreads();
  if (tid == 0 && !s_abort) R->epoch[b] = seq + (uint32_t)T;
}

// ------------------------------------------------------------------------------------
// the TMA-staged torus kernel (product path)
// ------------------------------------------------------------------------------------
// Same wavefront and flag protocol as torus_kernel (stage p of iteration it works on
// tile it - 2p), with every bulk transfer -- reads AND writes of the user buffer, the
// workspace slots and the peers' slots over NVLink -- done by TMA (cp.async.bulk)
// through a ring of shared-memory buffers.  Keeping ordinary st.global traffic out of
// the CTA keeps the system-scope fence behind every flag at ~1.3 us (measured; with
// thousands of in-flight st.global it took 5-9 us).  Roles, meeting only at mbarriers
// (full[b] / consumed[b] / empty[b] per buffer) and two shared-memory counters:
//   warp 0      poller: waits for the iteration's input flags (ld.acquire.sys) and for my
//               own stores of iteration it-2 (stage C reads the v_in slot my stage B
//               filled), then posts s_ready; never waits on a fence
//   warp 1      producer (lane 0): TMA-loads every job's operands into ring buffers
//   warps 2-5   storers (lane 0 each, jobs dealt round-robin): after the consumers sign
//               off a job, TMA-store its results and free its buffers as soon as the
//               stores have read them; at each iteration end drain the warp's bulk groups
//               and post s_done[storer] (one warp each: a lane blocked in wait_group
//               stalls its whole warp)
//   warp 6      publisher: once every storer has drained iteration it, post each stage's
//               completed tile to global memory (st.release.gpu; no system fence here)
//   signal CTA  (appended after the data CTAs, on its own quiet SM) one lane per data
//               CTA: when a posted tile advances, one fence.acq_rel.sys and the flag
//               stores to the peers.  A system-scope fence issued from an SM that is
//               streaming bulk traffic took ~8 us (traced); from a quiet SM ~1 us.
//   warps 7-15  consumers: folds (ring order, f32 accumulation, mean, one rounding) and
//               dtype<->wire casts from shared memory into shared memory; scalar
//               st/ld.global only for a ragged last vector or an unaligned user buffer
constexpr int kStorers = 4;                     // storer warps 2..5
constexpr int kRaiserWarp = 2 + kStorers;       // warp 6
constexpr int kConsWarp0 = kRaiserWarp + 1;     // consumers: warps 7..15
constexpr int kConsWarps = kThreads / 32 - kConsWarp0;
constexpr int kCons = kConsWarps * 32;

struct Job {
  int kind;
  int j, s;            // chunk (column) and sub-chunk (row) of the piece
  Piece p;
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int DT, int W>
__global__ void __launch_bounds__(kThreads, 1) torus_tma_kernel(const LaunchArgs a) {
  using Acc = typename Wire<W>::Acc;
  using UT = typename Elem<DT>::T;
  constexpr int VE = Wire<W>::VE;
  constexpr int SW = kVecBytes / VE;
  constexpr int ST = (int)sizeof(UT);
  constexpr bool kCast = DT != W;

  if (blockIdx.x >= a.nlocal * a.G) {
    // ================================ signal CTA ================================
    const int gidx = (blockIdx.x - a.nlocal * a.G) * blockDim.x + threadIdx.x;
    if (gidx >= a.nlocal * a.G) return;
    const int lr = gidx / a.G, b = gidx - (gidx / a.G) * a.G, G = a.G;
    const RankDev* __restrict__ R = a.ranks + lr;
    const int X = R->X, Y = R->Y, rho = R->rho, c = R->c;
    const uint32_t seq = R->epoch[b];
    const uint32_t target = seq + (uint32_t)a.T;
    // output flag of each stage: A -> H, B -> V (Y > 1) or R, C -> AG, D -> R
    const int okind[kStages] = {X > 1 ? kFlagH : -1, Y > 1 ? kFlagV : (X > 1 ? kFlagR : -1),
                                Y > 1 ? kFlagAG : -1, (Y > 1 && X > 1) ? kFlagR : -1, -1};
    uint32_t raised[kStages];
    for (int k2 = 0; k2 < kStages; ++k2) raised[k2] = seq;
    const uint32_t* const dl = a.done_local + (size_t)gidx * 8;
    const unsigned long long deadline = gtimer() + a.timeout_ns;
    bool ok = true;
    while (true) {
      bool all = true, fresh = false;
      uint32_t v[kStages];
      for (int k2 = 0; k2 < kStages; ++k2) {
        if (okind[k2] < 0) continue;
        v[k2] = ld_acquire_gpu(dl + k2);
        if ((int32_t)(v[k2] - raised[k2]) > 0) fresh = true;
        if (v[k2] != target) all = false;
      }
      if (fresh) {
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        for (int k2 = 0; k2 < kStages; ++k2) {
          if (okind[k2] < 0 || (int32_t)(v[k2] - raised[k2]) <= 0) continue;
          const int kind = okind[k2];
          const bool row = (kind == kFlagH || kind == kFlagR);
          const int cnt = row ? X - 1 : Y - 1;
          for (int l = 0; l < cnt; ++l) {
            const int other = row ? (c + 1 + l) % X : (rho + 1 + l) % Y;
            const int peer = row ? rho * X + other : other * X + c;
            uint32_t* f = reinterpret_cast<uint32_t*>(R->ws[peer]) +
                          ((size_t)(kind * kMaxDim + (row ? c : rho)) * G + b);
            st_relaxed_sys(f, v[k2]);
          }
          raised[k2] = v[k2];
        }
      }
      if (all) break;
      if (!fresh) {
        __nanosleep(64);
        if (gtimer() > deadline) {
          atomicCAS_system(R->err, 0, kErrTimeout);
          ok = false;
          break;
        }
      }
    }
    if (ok) st_release_gpu(a.sig_ack + gidx, target);
    return;
  }

  extern __shared__ __align__(1024) unsigned char smem[];
  const int NB = a.nbufs;
  const int TV = a.tile_vecs;
  const int CV = a.chunk_vecs;  // a tile piece moves through the ring in chunks of CV vectors
  const unsigned PB = (unsigned)CV * VE * (ST > SW ? ST : SW);  // one chunk, user or wire
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NB * PB);
  uint64_t* empty = full + NB;
  uint64_t* consumed = empty + NB;

  const int lr = blockIdx.x / a.G;
  const int b = blockIdx.x - lr * a.G;
  const RankDev* __restrict__ R = a.ranks + lr;
  const int X = R->X, Y = R->Y, N = R->N, rho = R->rho, c = R->c, me = R->rank;
  const int G = a.G, q = a.q, T = a.T;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const unsigned long long n = a.n;
  const bool aligned = a.aligned != 0;
  void* const buf = a.buf[lr];
  char* const myws = R->ws[me];

  __shared__ uint32_t s_seq;
  __shared__ int s_abort;
  __shared__ int s_ready;    // control -> producer: iterations whose inputs are visible
  __shared__ int s_done[kStorers];  // storer lane -> raiser: iterations it has drained
  if (tid == 0) {
    s_seq = R->epoch[b];
    s_abort = 0;
    s_ready = 0;
    for (int i = 0; i < kStorers; ++i) s_done[i] = 0;
    for (int i = 0; i < NB; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
      mbar_init(&consumed[i], kConsWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint32_t seq = s_seq;

  int kinds[kStages];
  int P = 0;
  if (X > 1) kinds[P++] = kA;
  kinds[P++] = kB;
  if (Y > 1) {
    kinds[P++] = kC;
    kinds[P++] = kD;
  }
  if (X > 1) kinds[P++] = kE;
  const int iters = T + 2 * (P - 1);

  // Jobs of iteration `it` in a fixed order (identical in every role): each tile piece
  // is cut into chunks of CV vectors, one job per chunk.
  auto for_jobs = [&](int it, auto visit0) {
    auto visit = [&](Job& jb) {
      const unsigned long long p0 = jb.p.p0, p1 = jb.p.p1;
      for (unsigned long long c0 = p0; c0 < p1; c0 += CV) {
        jb.p.p0 = c0;
        jb.p.p1 = (c0 + CV < p1) ? c0 + CV : p1;
        visit0(jb);
      }
      jb.p.p0 = p0;
      jb.p.p1 = p1;
    };
    for (int pp = 0; pp < P; ++pp) {
      const int t = it - 2 * pp;
      if (t < 0 || t >= T) continue;
      Job jb;
      jb.kind = kinds[pp];
      if (jb.kind == kA || jb.kind == kE) {
        for (int jj = 1; jj < X; ++jj)
          for (int s = 0; s < Y; ++s) {
            jb.j = (c + jj) % X;
            jb.s = s;
            jb.p = make_piece(n, X, Y, q, G, b, TV, jb.j, s, t);
            if (jb.p.p1 > jb.p.p0) visit(jb);
          }
      } else if (jb.kind == kB) {
        for (int s = 0; s < Y; ++s) {
          jb.j = c;
          jb.s = s;
          jb.p = make_piece(n, X, Y, q, G, b, TV, c, s, t);
          if (jb.p.p1 > jb.p.p0) visit(jb);
        }
      } else if (jb.kind == kC) {
        jb.j = c;
        jb.s = rho;
        jb.p = make_piece(n, X, Y, q, G, b, TV, c, rho, t);
        if (jb.p.p1 > jb.p.p0) visit(jb);
      } else {
        for (int ii = 1; ii < Y; ++ii) {
          jb.j = c;
          jb.s = (rho + ii) % Y;
          jb.p = make_piece(n, X, Y, q, G, b, TV, c, jb.s, t);
          if (jb.p.p1 > jb.p.p0) visit(jb);
        }
      }
    }
  };
  // Leading vectors of a piece whose user-buffer side moves by TMA (full 16-byte-aligned
  // vectors); a ragged last vector, or all of an unaligned buffer, goes through registers.
  auto nut_of = [&](const Job& jb) -> unsigned long long {
    if (!aligned) return 0;
    const unsigned long long last_el = jb.p.so + (jb.p.p1 - 1) * VE;
    return (last_el + VE > jb.p.cl) ? jb.p.p1 - jb.p.p0 - 1 : jb.p.p1 - jb.p.p0;
  };
  // Buffer plan: [wire loads (nw)][user load?][scratch (wire result)?][ustage (f32)?]
  struct Plan {
    int nw, ul, sc, us, nb;
    bool cons;  // consumers have work
  };
  auto plan_of = [&](const Job& jb) -> Plan {
    Plan pl;
    const unsigned long long nv = jb.p.p1 - jb.p.p0, nut = nut_of(jb);
    const bool ragged = nut < nv;
    const bool reads_user = jb.kind == kA || jb.kind == kB;
    const bool writes_user = jb.kind == kC || jb.kind == kD || jb.kind == kE || (jb.kind == kB && Y == 1);
    pl.nw = jb.kind == kB ? X - 1 : jb.kind == kC ? Y : (jb.kind == kA ? 0 : 1);
    pl.ul = (reads_user && nut > 0) ? 1 : 0;
    pl.sc = (jb.kind == kB || jb.kind == kC || (jb.kind == kA && (kCast || ragged))) ? 1 : 0;
    pl.us = (kCast && writes_user && nut > 0) ? 1 : 0;
    pl.nb = pl.nw + pl.ul + pl.sc + pl.us;
    pl.cons = jb.kind == kB || jb.kind == kC || kCast || ragged;
    return pl;
  };
  auto user_ptr = [&](const Job& jb) -> char* {
    return reinterpret_cast<char*>(buf) + (a.buf_off + jb.p.co + jb.p.so + jb.p.p0 * VE) * ST;
  };

  if (warp == 0 || warp == kRaiserWarp) {
    // ========================== poller (0) and raiser (6) ==========================
    const unsigned long long deadline = gtimer() + a.timeout_ns;
    auto flagp = [&](char* ws, int kind, int src) -> uint32_t* {
      return reinterpret_cast<uint32_t*>(ws) + ((size_t)(kind * kMaxDim + src) * G + b);
    };
    auto for_flags = [&](int k, int t, bool in, auto visit) {
      int kind = -1, cnt = 0;
      bool row = true;
      switch (k) {
        case kA:
          if (!in) { kind = kFlagH; cnt = X - 1; row = true; }
          break;
        case kB:
          if (in) {
            if (X > 1) { kind = kFlagH; cnt = X - 1; row = true; }
          } else if (Y > 1) {
            kind = kFlagV; cnt = Y - 1; row = false;
          } else if (X > 1) {
            kind = kFlagR; cnt = X - 1; row = true;
          }
          break;
        case kC:
          kind = in ? kFlagV : kFlagAG; cnt = Y - 1; row = false;
          break;
        case kD:
          if (in) { kind = kFlagAG; cnt = Y - 1; row = false; }
          else if (X > 1) { kind = kFlagR; cnt = X - 1; row = true; }
          break;
        default:
          if (in) { kind = kFlagR; cnt = X - 1; row = true; }
          break;
      }
      const uint32_t v = seq + (uint32_t)t + 1u;
      for (int l = 0; l < cnt; ++l) {
        const int other = row ? (c + 1 + l) % X : (rho + 1 + l) % Y;
        const int peer = row ? rho * X + other : other * X + c;
        visit(in ? flagp(myws, kind, other) : flagp(R->ws[peer], kind, row ? c : rho), v);
      }
    };
    auto poll_iter = [&](int it) -> bool {
      bool ok = true;
      int e = 0;
      for (int pp = 0; pp < P; ++pp) {
        const int t = it - 2 * pp;
        if (t < 0 || t >= T) continue;
        for_flags(kinds[pp], t, true, [&](uint32_t* f, uint32_t v) {
          if ((e++ & 31) == lane && ok) ok = wait_flag_ge(f, v, deadline, 64, R->err);
        });
      }
      return __all_sync(0xffffffffu, ok);
    };
    auto raise_iter = [&](int it) {
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      stamp((lane == 0 && lr == 0) ? a.trace : nullptr, b, it, 3);
      int e = 0;
      for (int pp = 0; pp < P; ++pp) {
        const int t = it - 2 * pp;
        if (t < 0 || t >= T) continue;
        for_flags(kinds[pp], t, false, [&](uint32_t* f, uint32_t v) {
          if ((e++ & 31) == lane) st_relaxed_sys(f, v);
        });
      }
    };
    auto wait_done = [&](int it) -> bool {  // every storer lane drained iteration it
      bool ok = true;
      if (lane < kStorers) {
        unsigned spin = 0;
        while (ld_acquire_cta(&s_done[lane]) <= it) {
          if ((++spin & 255u) == 0 && gtimer() > deadline) {
            ok = false;
            break;
          }
        }
      }
      return __all_sync(0xffffffffu, ok);
    };
    unsigned long long* const tr = (lane == 0 && lr == 0) ? a.trace : nullptr;
    if (warp == 0) {
      for (int it = 0; it < iters; ++it) {
        stamp(tr, b, it, 0);
        if (!poll_iter(it)) {  // watchdog: poison; the producer walks the rest without loads
          if (lane == 0) {
            atomicCAS_system(R->err, 0, kErrTimeout);
            s_abort = 1;
            st_release_cta(&s_ready, iters);
          }
          __syncwarp();
          break;
        }
        // my own stores of iteration it-2 (stage B's local v_in slot, read by stage C)
        if (it >= 2 && !wait_done(it - 2)) {
          if (lane == 0) {
            atomicCAS_system(R->err, 0, kErrTimeout);
            s_abort = 1;
            st_release_cta(&s_ready, iters);
          }
          __syncwarp();
          break;
        }
        stamp(tr, b, it, 1);
        if (lane == 0) st_release_cta(&s_ready, it + 1);  // producer may load iteration it
        __syncwarp();
      }
    } else {
      // publisher: each stage's newest completed tile -> global (gpu scope) for the
      // signal CTA, which fences on a quiet SM and forwards it to the peers' flags
      uint32_t* const dl = a.done_local + (size_t)(lr * G + b) * 8;
      for (int it = 0; it < iters; ++it) {
        if (!wait_done(it)) {
          if (lane == 0) {
            atomicCAS_system(R->err, 0, kErrTimeout);
            s_abort = 1;
          }
          __syncwarp();
          break;
        }
        if (*(volatile int*)&s_abort) break;
        stamp(tr, b, it, 2);
        if (lane == 0)
          for (int pp = 0; pp < P; ++pp) {
            const int t = it - 2 * pp;
            if (t >= 0 && t < T) st_release_gpu(dl + kinds[pp], seq + (uint32_t)t + 1u);
          }
        __syncwarp();
        stamp(tr, b, it, 4);
      }
    }
  } else if (warp == 1) {
    // =============================== producer warp ==============================
    if (lane == 0) {
      int slot = 0;
      bool aborted = false;
      for (int it = 0; it < iters; ++it) {
        if (!aborted) {
          while (ld_acquire_cta(&s_ready) <= it) {}
          aborted = *(volatile int*)&s_abort != 0;
        }
        fence_proxy_async();  // data the control warp acquired -> async-proxy loads
        for_jobs(it, [&](const Job& jb) {
          const Plan pl = plan_of(jb);
          const unsigned wbytes = (unsigned)((jb.p.p1 - jb.p.p0) * kVecBytes);
          for (int o = 0; o < pl.nb; ++o, ++slot) {
            const int bi = slot % NB;
            mbar_wait(&empty[bi], ((slot / NB) & 1) ^ 1);
            const bool is_wire = o < pl.nw, is_user = pl.ul && o == pl.nw;
            if (aborted || !(is_wire || is_user)) {  // scratch / staging / poisoned call
              mbar_arrive(&full[bi]);
              continue;
            }
            const char* src;
            unsigned bytes = wbytes;
            if (is_user) {
              bytes = (unsigned)(nut_of(jb) * VE * ST);
              src = user_ptr(jb);
            } else if (jb.kind == kB) {  // h_in slot of source column (c+1+o) % X
              src = myws + a.hin_off + (size_t)((c + 1 + o) % X) * a.hin_stride +
                    (jb.p.so + jb.p.p0 * VE) * SW;
            } else if (jb.kind == kC) {  // v_in slot of row (rho+1+o) % Y
              src = myws + a.vin_off + (size_t)((rho + 1 + o) % Y) * a.vin_stride +
                    jb.p.p0 * VE * SW;
            } else if (jb.kind == kD) {  // column peer (s, c)'s chunk slot
              src = R->ws[jb.s * X + c] + a.chunk_off + (jb.p.so + jb.p.p0 * VE) * SW;
            } else {                     // row peer (rho, j)'s chunk slot
              src = R->ws[rho * X + jb.j] + a.chunk_off + (jb.p.so + jb.p.p0 * VE) * SW;
            }
            mbar_expect_tx(&full[bi], bytes);
            tma_load(smem + (size_t)bi * PB, src, bytes, &full[bi]);
          }
        });
      }
    }
  } else if (warp >= 2 && warp < 2 + kStorers) {
    // =============================== storer warps ===============================
    const int sw_id = warp - 2;
    if (lane == 0) {
      int slot = 0, jobno = 0;
      for (int it = 0; it < iters; ++it) {
        for_jobs(it, [&](const Job& jb) {
          const Plan pl = plan_of(jb);
          const int b0 = slot;
          slot += pl.nb;
          if ((jobno++ % kStorers) != sw_id) return;
          for (int o = 0; o < pl.nb; ++o) mbar_wait(&consumed[(b0 + o) % NB], ((b0 + o) / NB) & 1);
          const bool live = *(volatile int*)&s_abort == 0;
          const unsigned long long nv = jb.p.p1 - jb.p.p0, nut = nut_of(jb);
          const unsigned wbytes = (unsigned)(nv * kVecBytes);
          const unsigned ubytes = (unsigned)(nut * VE * ST);
          // the wire result of the job (the buffer a wire-side store reads)
          const int wbuf = (jb.kind == kA) ? (b0 + (pl.sc ? pl.nw + pl.ul : pl.nw)) % NB
                         : (jb.kind == kB || jb.kind == kC) ? (b0 + pl.nw + pl.ul) % NB
                         : b0 % NB;
          // the user-layout data a user-side store reads
          const int ubuf = pl.us ? (b0 + pl.nb - 1) % NB : wbuf;
          bool stored = false;
          if (live) {
            if (jb.kind == kA) {  // push my share into (rho, j).h_in[c]
              tma_store(R->ws[rho * X + jb.j] + a.hin_off + (size_t)c * a.hin_stride +
                            (jb.p.so + jb.p.p0 * VE) * SW,
                        smem + (size_t)wbuf * PB, wbytes);
              stored = true;
            } else if (jb.kind == kB && Y > 1) {  // P1 -> v_in[rho] of sub-chunk owner (s, c)
              tma_store(R->ws[jb.s * X + c] + a.vin_off + (size_t)rho * a.vin_stride +
                            jb.p.p0 * VE * SW,
                        smem + (size_t)wbuf * PB, wbytes);
              stored = true;
            } else {
              // final values: my chunk slot (pulled by peers) and my user buffer
              if ((jb.kind == kB && X > 1) || jb.kind == kC || (jb.kind == kD && X > 1)) {
                tma_store(myws + a.chunk_off + (jb.p.so + jb.p.p0 * VE) * SW,
                          smem + (size_t)wbuf * PB, wbytes);
                stored = true;
              }
              if (nut > 0) {
                tma_store(user_ptr(jb), smem + (size_t)ubuf * PB, ubytes);
                stored = true;
              }
            }
          }
          if (stored) {
            tma_commit();
            tma_wait_read<0>();  // the stores have read their shared-memory sources
          }
          for (int o = 0; o < pl.nb; ++o) mbar_arrive(&empty[(b0 + o) % NB]);
        });
        // this warp's stores of iteration it are complete before the raiser's fence
        tma_wait_all<0>();
        fence_proxy_async();
        st_release_cta(&s_done[sw_id], it + 1);
        if (sw_id == 0) stamp(lr == 0 ? a.trace : nullptr, b, it, 7);
      }
    }
  } else {
    // =============================== consumer warps =============================
    const int ct = tid - kConsWarp0 * 32;
    int slot = 0;
    unsigned long long* const tr = (ct == 0 && lr == 0) ? a.trace : nullptr;
    for (int it = 0; it < iters; ++it) {
      stamp(tr, b, it, 5);
      for_jobs(it, [&](const Job& jb) {
        const Plan pl = plan_of(jb);
        const int b0 = slot;
        slot += pl.nb;
        // Every buffer's full / consumed / empty barriers advance exactly once per use:
        // the consumers wait for and sign off every buffer of every job, even pure copies.
        for (int o = 0; o < pl.nb; ++o) mbar_wait(&full[(b0 + o) % NB], ((b0 + o) / NB) & 1);
        if (pl.cons) {
          const bool live = *(volatile int*)&s_abort == 0;
          const unsigned long long nv = jb.p.p1 - jb.p.p0, nut = nut_of(jb);
          const unsigned char* const uin = smem + (size_t)((b0 + pl.nw) % NB) * PB;    // user load
          unsigned char* const wout =                                                  // wire result
              smem + (size_t)((jb.kind == kD || jb.kind == kE) ? b0 % NB : (b0 + pl.nw + pl.ul) % NB) * PB;
          unsigned char* const uout = smem + (size_t)((b0 + pl.nb - 1) % NB) * PB;      // f32 staging
          auto user_in = [&](unsigned long long v, unsigned long long el, int nrem) -> uint4 {
            if (v < nut) {
              if constexpr (!kCast) {
                return *reinterpret_cast<const uint4*>(uin + v * kVecBytes);
              } else {
                const float* f = reinterpret_cast<const float*>(uin + v * VE * ST);
                float t[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) t[i] = f[i];
                return pack<W>(t);
              }
            }
            return load_user<DT, W>(buf, a.buf_off + jb.p.co + el, nrem, aligned);
          };
          auto user_out = [&](unsigned long long v, unsigned long long el, int nrem, uint4 w) {
            if (v < nut) {
              if constexpr (kCast) {
                float f[8];
                unpack<W>(w, f);
                float4* d = reinterpret_cast<float4*>(uout + v * VE * ST);
                d[0] = make_float4(f[0], f[1], f[2], f[3]);
                d[1] = make_float4(f[4], f[5], f[6], f[7]);
              }  // same dtype: the TMA store reads the wire result directly
            } else if (live) {
              store_user<DT, W>(buf, a.buf_off + jb.p.co + el, nrem, w, aligned);
            }
          };
          for (unsigned long long v = ct; v < nv; v += kCons) {
            const unsigned long long el = jb.p.so + (jb.p.p0 + v) * VE;
            const int nrem = (int)min((unsigned long long)VE, jb.p.cl - el);
            if (jb.kind == kA) {
              *reinterpret_cast<uint4*>(wout + v * kVecBytes) = user_in(v, el, nrem);
            } else if (jb.kind == kB || jb.kind == kC) {
              const int nops = (jb.kind == kB) ? X : Y;
              Acc acc[VE];
              for (int k = 0; k < nops; ++k) {  // ring order; my own contribution last in B
                const uint4 w = (jb.kind == kB && k == X - 1)
                                    ? user_in(v, el, nrem)
                                    : *reinterpret_cast<const uint4*>(smem + (size_t)((b0 + k) % NB) * PB +
                                                                      v * kVecBytes);
                Acc t[VE];
                unpack<W>(w, t);
                if (k == 0) {
#pragma unroll
                  for (int i = 0; i < VE; ++i) acc[i] = t[i];
                } else {
                  acc_add<W>(acc, t);
                }
              }
              const bool last_reduce = (jb.kind == kC) || (Y == 1);
              if (last_reduce && a.op == 1) acc_mean<W>(acc, a.inv_n, N);
              const uint4 o = pack<W>(acc);
              *reinterpret_cast<uint4*>(wout + v * kVecBytes) = o;
              if (last_reduce) user_out(v, el, nrem, o);
            } else {  // D / E: pulled wire data -> my user buffer
              user_out(v, el, nrem, *reinterpret_cast<const uint4*>(wout + v * kVecBytes));
            }
          }
          fence_proxy_async_smem();  // staged results -> the storers' async-proxy reads
        }
        __syncwarp();
        if (lane == 0)
          for (int o = 0; o < pl.nb; ++o) mbar_arrive(&consumed[(b0 + o) % NB]);
      });
      stamp(tr, b, it, 6);
    }
  }
  __syncthreads();
  if (tid == 0 && !s_abort) {
    // the signal lane has read this call's epoch and forwarded every flag
    const unsigned long long deadline = gtimer() + a.timeout_ns;
    const uint32_t* ack = a.sig_ack + (size_t)(lr * G + b);
    bool ok = true;
    while ((int32_t)(ld_acquire_gpu(ack) - (seq + (uint32_t)T)) < 0) {
      __nanosleep(64);
      if (gtimer() > deadline) {
        atomicCAS_system(R->err, 0, kErrTimeout);
        ok = false;
        break;
      }
    }
    if (ok) R->epoch[b] = seq + (uint32_t)T;
  }
}

// N = 1: buf = from_wire(to_wire(buf)); the mean scale is x * 1.0 (identity).
// HBM-bound: 8 B per element.  Each thread keeps U 32-byte vectors in flight (2U x
// LDG.E.128 before the first store); the grid is CPS CTAs per SM of BLK threads.
template <int W, int U, int BLK>
__global__ void __launch_bounds__(BLK) castscale_kernel(float* buf, unsigned long long n) {
  const unsigned long long nv = (n + 7) / 8;
  const bool aligned = (reinterpret_cast<uintptr_t>(buf) & 15) == 0;
  const unsigned long long stride = (unsigned long long)gridDim.x * BLK;
  for (unsigned long long v0 = blockIdx.x * (unsigned long long)BLK + threadIdx.x; v0 < nv;
       v0 += stride * U) {
    uint4 w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned long long v = v0 + u * stride;
      if (v < nv) w[u] = load_user<DT_F32, W>(buf, v * 8, (int)min(8ull, n - v * 8), aligned);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned long long v = v0 + u * stride;
      if (v < nv) store_user<DT_F32, W>(buf, v * 8, (int)min(8ull, n - v * 8), w[u], aligned);
    }
  }
}

// Cache-operator variants of the one-shot cast (env TORUS_CS_CACHE = "<load>,<store>"):
// load 0 ld.global.cs, 1 ld.global.nc.L1::no_allocate, 2 ld.global with an L2 evict_first
// policy; store 0 st.global.cs, 1 st.global (write-back), 2 / 3 st.global with an L2
// evict_first / evict_last policy.  One 32-byte vector per thread, 512 threads per CTA.
template <int W, int LC, int SC>
__global__ void __launch_bounds__(512) castscale_cache_kernel(float* buf, unsigned long long n) {
  const unsigned long long nv = n / 8;  // whole vectors (the caller handles n % 8 == 0 only)
  const unsigned long long v = blockIdx.x * 512ull + threadIdx.x;
  if (v >= nv) return;
  float* p = buf + v * 8;
  uint64_t pol_first = 0, pol_last = 0;
  if constexpr (LC == 2 || SC == 2)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
  if constexpr (SC == 3)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
  float f[8];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float* q = p + 4 * h;
    if constexpr (LC == 0)
      asm volatile("ld.global.cs.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(f[4 * h]), "=f"(f[4 * h + 1]), "=f"(f[4 * h + 2]), "=f"(f[4 * h + 3]) : "l"(q));
    else if constexpr (LC == 1)
      asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(f[4 * h]), "=f"(f[4 * h + 1]), "=f"(f[4 * h + 2]), "=f"(f[4 * h + 3]) : "l"(q));
    else
      asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                   : "=f"(f[4 * h]), "=f"(f[4 * h + 1]), "=f"(f[4 * h + 2]), "=f"(f[4 * h + 3])
                   : "l"(q), "l"(pol_first));
  }
  float y[8];
  unpack<W>(pack<W>(f), y);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float* q = p + 4 * h;
    if constexpr (SC == 0)
      asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(q), "f"(y[4 * h]), "f"(y[4 * h + 1]),
                   "f"(y[4 * h + 2]), "f"(y[4 * h + 3]) : "memory");
    else if constexpr (SC == 1)
      asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(q), "f"(y[4 * h]), "f"(y[4 * h + 1]),
                   "f"(y[4 * h + 2]), "f"(y[4 * h + 3]) : "memory");
    else
      asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(q), "f"(y[4 * h]),
                   "f"(y[4 * h + 1]), "f"(y[4 * h + 2]), "f"(y[4 * h + 3]), "l"(SC == 2 ? pol_first : pol_last)
                   : "memory");
  }
}

template <int W>
cudaError_t launch_cs_cache(float* buf, unsigned long long n, int lc, int sc, cudaStream_t stream) {
  const unsigned long long blocks = (n / 8 + 511) / 512;
  const int k = lc * 4 + sc;
#define CSC(L, S) \
  case L * 4 + S: castscale_cache_kernel<W, L, S><<<(unsigned)blocks, 512, 0, stream>>>(buf, n); break;
  switch (k) {
    CSC(0, 0) CSC(0, 1) CSC(0, 2) CSC(0, 3) CSC(1, 0) CSC(1, 1) CSC(1, 2) CSC(1, 3)
    CSC(2, 0) CSC(2, 1) CSC(2, 2) CSC(2, 3)
    default: return cudaErrorInvalidValue;
  }
#undef CSC
  return cudaGetLastError();
}

// Device barrier among all ranks (init/destroy): every rank stores its epoch into every
// peer's barrier slot, then waits for all peers' slots.
__global__ void barrier_kernel(const RankDev* ranks, unsigned long long bar_off,
                               unsigned long long timeout_ns) {
  const RankDev* R = ranks + blockIdx.x;
  __shared__ uint32_t s_e;
  if (threadIdx.x == 0) s_e = *R->bar_epoch + 1u;
  __syncthreads();
  const uint32_t e = s_e;
  const int t = threadIdx.x;
  if (t < R->N && t != R->rank)
    st_release_sys(reinterpret_cast<uint32_t*>(R->ws[t] + bar_off) + R->rank, e);
  if (t < R->N && t != R->rank) {
    const uint32_t* f = reinterpret_cast<const uint32_t*>(R->ws[R->rank] + bar_off) + t;
    const unsigned long long deadline = gtimer() + timeout_ns;
    unsigned it = 0;
    while ((int32_t)(ld_acquire_sys(f) - e) < 0) {
      if ((++it & 255u) == 0 && gtimer() > deadline) {
        atomicCAS_system(R->err, 0, kErrTimeout);
        break;
      }
    }
  }
  __syncthreads();
  if (t == 0) *R->bar_epoch = e;
}

template <int DT, int W>
cudaError_t launch_typed(const LaunchArgs& a, bool cooperative, cudaStream_t stream) {
  const dim3 grid(a.nlocal * a.G), block(kThreads);
  if (a.nbufs > 0) {  // TMA-staged kernel: data CTAs + signal CTAs
    const dim3 grid(a.nlocal * a.G + a.nsig), block(kThreads);
    const int smem = tma_smem_bytes(a.nbufs, a.chunk_vecs, (int)(sizeof(typename Elem<DT>::T) * Wire<W>::VE / 16));
    static bool attr_set = false;
    if (!attr_set) {
      cudaError_t e = cudaFuncSetAttribute(torus_tma_kernel<DT, W>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmemMax);
      if (e != cudaSuccess) return e;
      attr_set = true;
    }
    if (cooperative) {
      void* args[] = {const_cast<LaunchArgs*>(&a)};
      return cudaLaunchCooperativeKernel((const void*)torus_tma_kernel<DT, W>, grid, block, args, smem,
                                         stream);
    }
    torus_tma_kernel<DT, W><<<grid, block, smem, stream>>>(a);
    return cudaGetLastError();
  }
  const dim3 lblock(kLdgThreads);
  const void* fn = (const void*)torus_kernel<DT, W, false>;
  if constexpr (DT != DT_I32) {
    if (a.nseg) fn = (const void*)torus_kernel<DT, W, true>;
  }
  if (a.nseg && DT == DT_I32) return cudaErrorNotSupported;
  if (cooperative) {
    void* args[] = {const_cast<LaunchArgs*>(&a)};
    return cudaLaunchCooperativeKernel(fn, grid, lblock, args, 0, stream);
  }
  void* args[] = {const_cast<LaunchArgs*>(&a)};
  return cudaLaunchKernel(fn, grid, lblock, args, 0, stream);
}

template <int DT, int W>
int max_ctas_typed() {
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, torus_kernel<DT, W, false>, kLdgThreads, 0) !=
      cudaSuccess)
    return 0;
  return nb;
}

}  // namespace

cudaError_t launch_torus(const LaunchArgs& a, int dtype, int wire, bool cooperative,
                         cudaStream_t stream) {
  if (dtype == wire) {
    switch (dtype) {
      case DT_F32: return launch_typed<DT_F32, DT_F32>(a, cooperative, stream);
      case DT_F16: return launch_typed<DT_F16, DT_F16>(a, cooperative, stream);
      case DT_BF16: return launch_typed<DT_BF16, DT_BF16>(a, cooperative, stream);
      case DT_I32: return launch_typed<DT_I32, DT_I32>(a, cooperative, stream);
    }
  } else if (dtype == DT_F32 && wire == DT_F16) {
    return launch_typed<DT_F32, DT_F16>(a, cooperative, stream);
  } else if (dtype == DT_F32 && wire == DT_BF16) {
    return launch_typed<DT_F32, DT_BF16>(a, cooperative, stream);
  }
  return cudaErrorInvalidValue;
}

int torus_kernel_max_ctas_per_sm(int dtype, int wire) {
  if (dtype == wire) {
    switch (dtype) {
      case DT_F32: return max_ctas_typed<DT_F32, DT_F32>();
      case DT_F16: return max_ctas_typed<DT_F16, DT_F16>();
      case DT_BF16: return max_ctas_typed<DT_BF16, DT_BF16>();
      case DT_I32: return max_ctas_typed<DT_I32, DT_I32>();
    }
  } else if (dtype == DT_F32 && wire == DT_F16) {
    return max_ctas_typed<DT_F32, DT_F16>();
  } else if (dtype == DT_F32 && wire == DT_BF16) {
    return max_ctas_typed<DT_F32, DT_BF16>();
  }
  return 0;
}

// castscale variant (env TORUS_CS = "<unroll>x<block>x<ctas per SM>", default 1x512x0: one
// 32-byte vector per thread, a one-shot grid covering the buffer, no CTA cap (0)).  Measured
// in the steady state of back-to-back calls on cold buffers (profiles/r02_cast_probe*.jsonl:
// 36.0 us for the 102 MB buffer, vs 38.5 for the best TMA ring and 36.5 for torch's own
// in-place elementwise kernel on the same bytes).
template <int W, int U, int BLK>
cudaError_t launch_cs(float* buf, unsigned long long n, int cps, cudaStream_t stream) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const unsigned long long nv = (n + 7) / 8;
  const unsigned long long want = (nv + (unsigned long long)BLK * U - 1) / ((unsigned long long)BLK * U);
  const unsigned long long cap = cps > 0 ? (unsigned long long)sms * cps : want;
  const int blocks = (int)(want < 1 ? 1 : (want < cap ? want : cap));
  castscale_kernel<W, U, BLK><<<blocks, BLK, 0, stream>>>(buf, n);
  return cudaGetLastError();
}

template <int W>
cudaError_t launch_cs_variant(float* buf, unsigned long long n, cudaStream_t stream) {
  int u = 1, blk = 512, cps = 0;
  if (const char* v = getenv("TORUS_CS")) sscanf(v, "%dx%dx%d", &u, &blk, &cps);
  if (u == 8 && blk == 256) return launch_cs<W, 8, 256>(buf, n, cps, stream);
  if (u == 2 && blk == 256) return launch_cs<W, 2, 256>(buf, n, cps, stream);
  if (u == 4 && blk == 512) return launch_cs<W, 4, 512>(buf, n, cps, stream);
  if (u == 8 && blk == 512) return launch_cs<W, 8, 512>(buf, n, cps, stream);
  if (u == 4 && blk == 128) return launch_cs<W, 4, 128>(buf, n, cps, stream);
  if (u == 2 && blk == 128) return launch_cs<W, 2, 128>(buf, n, cps, stream);
  if (u == 1 && blk == 128) return launch_cs<W, 1, 128>(buf, n, cps, stream);
  if (u == 1 && blk == 256) return launch_cs<W, 1, 256>(buf, n, cps, stream);
  if (u == 1 && blk == 512) return launch_cs<W, 1, 512>(buf, n, cps, stream);
  if (u == 4 && blk == 256) return launch_cs<W, 4, 256>(buf, n, cps, stream);
  return launch_cs<W, 1, 512>(buf, n, cps, stream);
}

bool castscale_use_tma() {
  const char* kv = getenv("TORUS_CS_KERNEL");
  return kv && strcmp(kv, "tma") == 0;
}

cudaError_t launch_castscale(void* buf, unsigned long long n, int dtype, int wire,
                             cudaStream_t stream) {
  if (dtype != DT_F32) return cudaErrorInvalidValue;
  // the TMA-streamed ring (torus_cast.cu) for aligned buffers with TORUS_CS_KERNEL=tma
  if (const char* cc = getenv("TORUS_CS_CACHE")) {  // cache-operator experiment (aligned, n % 8 == 0)
    int lc = 0, sc = 0;
    sscanf(cc, "%d,%d", &lc, &sc);
    if ((reinterpret_cast<uintptr_t>(buf) & 15) == 0 && n % 8 == 0) {
      if (wire == DT_F16) return launch_cs_cache<DT_F16>(reinterpret_cast<float*>(buf), n, lc, sc, stream);
      if (wire == DT_BF16) return launch_cs_cache<DT_BF16>(reinterpret_cast<float*>(buf), n, lc, sc, stream);
    }
  }
  if (castscale_use_tma() && (reinterpret_cast<uintptr_t>(buf) & 15) == 0 && n >= 8)
    return launch_castscale_tma(buf, n, wire, stream);
  if (wire == DT_F16) return launch_cs_variant<DT_F16>(reinterpret_cast<float*>(buf), n, stream);
  if (wire == DT_BF16) return launch_cs_variant<DT_BF16>(reinterpret_cast<float*>(buf), n, stream);
  return cudaErrorInvalidValue;
}

cudaError_t launch_barrier(const RankDev* ranks, int nlocal, unsigned long long bar_off,
                           unsigned long long timeout_ns, cudaStream_t stream) {
  if (nlocal > 1) {
    void* args[] = {const_cast<RankDev**>(&ranks), &bar_off, &timeout_ns};
    return cudaLaunchCooperativeKernel((const void*)barrier_kernel, dim3(nlocal), dim3(kMaxRanks),
                                       args, 0, stream);
  }
  barrier_kernel<<<1, kMaxRanks, 0, stream>>>(ranks, bar_off, timeout_ns);
  return cudaGetLastError();
}

}  // namespace torus
