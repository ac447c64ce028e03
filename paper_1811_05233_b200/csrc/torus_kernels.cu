// torus_kernels.cu -- sm_100a kernels of the 2D-Torus all-reduce (Sec. 2.2).
//
//   torus_kernel      (default) one fused launch per round: the paper's three steps as a
//                     5-stage tile wavefront (A push / B row fold / C column fold + mean /
//                     D column all-gather / E row all-gather), control warp + 15 data
//                     warps, 128-bit LDG/STG over NVLink, one system fence per iteration
//   torus_tma_kernel  (TORUS_KERNEL=tma) the same protocol with TMA bulk copies, a
//                     producer / consumer / storer / poller / publisher split and a signal
//                     CTA that fences from a quiet SM (parity-green, latency-bound today)
//   castscale_kernel  the N = 1 degenerate case (fused cast round trip)
//   ring_kernel, hier_kernel   the flat-ring and hierarchical baselines
//   probe kernels     NVLink / fence calibration (torus_probe)
//   multi_copy_kernel bucketed pack / unpack (NEXT-1)
// Phases in the paper's words: "Firstly, reduce-scatter is performed horizontally. Then,
// all-reduce is performed vertically. Finally, all-gather is performed horizontally."
// Fold order, partition and rounding points follow the oracle, so every
// dtype is bit-exact.  No tensor cores: a bandwidth-bound reduction, not a contraction.
#include <cstdio>
#include <cstdlib>

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
template <int DT, int W>
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
          if ((e++ & 31) == lane && ok) ok = wait_flag_ge(f, v, deadline, a.poll_sleep);
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
          atomicExch_system(R->err, kErrTimeout);
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
                    r[u] = load_user<DT, W>(buf, a.buf_off + p.co + el, nrem, aligned);
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
                      r[u] = load_user<DT, W>(buf, a.buf_off + p.co + el, nrem, aligned);
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
                  store_user<DT, W>(buf, a.buf_off + p.co + el, nrem, out, aligned);
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
              store_user<DT, W>(buf, a.buf_off + p.co + el, nrem, out, aligned);
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
                store_user<DT, W>(buf, a.buf_off + p.co + el, nrem, r[u], aligned);
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
                  store_user<DT, W>(buf, a.buf_off + p.co + el, nrem, r[u], aligned);
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
          atomicExch_system(R->err, kErrTimeout);
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
          if ((e++ & 31) == lane && ok) ok = wait_flag_ge(f, v, deadline);
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
            atomicExch_system(R->err, kErrTimeout);
            s_abort = 1;
            st_release_cta(&s_ready, iters);
          }
          __syncwarp();
          break;
        }
        // my own stores of iteration it-2 (stage B's local v_in slot, read by stage C)
        if (it >= 2 && !wait_done(it - 2)) {
          if (lane == 0) {
            atomicExch_system(R->err, kErrTimeout);
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
            atomicExch_system(R->err, kErrTimeout);
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
        atomicExch_system(R->err, kErrTimeout);
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
        atomicExch_system(R->err, kErrTimeout);
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
  if (cooperative) {
    void* args[] = {const_cast<LaunchArgs*>(&a)};
    return cudaLaunchCooperativeKernel((const void*)torus_kernel<DT, W>, grid, lblock, args, 0,
                                       stream);
  }
  torus_kernel<DT, W><<<grid, lblock, 0, stream>>>(a);
  return cudaGetLastError();
}

template <int DT, int W>
int max_ctas_typed() {
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, torus_kernel<DT, W>, kLdgThreads, 0) !=
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

// castscale variant (env TORUS_CS = "<unroll>x<block>x<ctas per SM>", default 4x256x4)
template <int W, int U, int BLK>
cudaError_t launch_cs(float* buf, unsigned long long n, int cps, cudaStream_t stream) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const unsigned long long nv = (n + 7) / 8;
  const unsigned long long want = (nv + (unsigned long long)BLK * U - 1) / ((unsigned long long)BLK * U);
  const unsigned long long cap = (unsigned long long)sms * cps;
  const int blocks = (int)(want < 1 ? 1 : (want < cap ? want : cap));
  castscale_kernel<W, U, BLK><<<blocks, BLK, 0, stream>>>(buf, n);
  return cudaGetLastError();
}

template <int W>
cudaError_t launch_cs_variant(float* buf, unsigned long long n, cudaStream_t stream) {
  int u = 4, blk = 256, cps = 4;
  if (const char* v = getenv("TORUS_CS")) sscanf(v, "%dx%dx%d", &u, &blk, &cps);
  if (u == 8 && blk == 256) return launch_cs<W, 8, 256>(buf, n, cps, stream);
  if (u == 2 && blk == 256) return launch_cs<W, 2, 256>(buf, n, cps, stream);
  if (u == 4 && blk == 512) return launch_cs<W, 4, 512>(buf, n, cps, stream);
  if (u == 8 && blk == 512) return launch_cs<W, 8, 512>(buf, n, cps, stream);
  if (u == 4 && blk == 128) return launch_cs<W, 4, 128>(buf, n, cps, stream);
  return launch_cs<W, 4, 256>(buf, n, cps, stream);
}

cudaError_t launch_castscale(void* buf, unsigned long long n, int dtype, int wire,
                             cudaStream_t stream) {
  if (dtype != DT_F32) return cudaErrorInvalidValue;
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

// ------------------------------------------------------------------------------------
// Calibration probes (SURVEY.md 8(d) "Calibration"; not on the all-reduce path):
//   mode 0  push: each rank stores `bytes` split evenly over its N-1 peers' data regions
//   mode 1  pull: each rank loads `bytes` split evenly from its N-1 peers' data regions
//   mode 2  ping-pong: rank 0 and rank 1 bounce a flag `iters` times (alpha)
//   mode 3  local copy: bytes from the slab's first half to its second half (HBM)
// ------------------------------------------------------------------------------------
namespace torus {
namespace {

__global__ void __launch_bounds__(512) probe_kernel(const RankDev* ranks, unsigned long long data_off,
                                                    unsigned long long bytes, int mode, int iters,
                                                    unsigned long long* out) {
  const RankDev* R = ranks;
  const int N = R->N, me = R->rank, tid = threadIdx.x, G = gridDim.x, b = blockIdx.x;
  if (mode == 2) {
    // flag words live in the barrier area (bar region + 4 KiB), never touched by data
    if (b != 0 || tid != 0 || me > 1 || N < 2) return;
    uint32_t* mine = reinterpret_cast<uint32_t*>(R->ws[me] + data_off);
    uint32_t* theirs = reinterpret_cast<uint32_t*>(R->ws[1 - me] + data_off);
    const uint32_t base = ld_acquire_sys(mine);
    const unsigned long long t0 = gtimer();
    const unsigned long long deadline = t0 + 5000000000ull;
    bool ok = true;
    for (int i = 1; i <= iters && ok; ++i) {
      if (me == 0) st_release_sys(theirs, base + i);
      unsigned spin = 0;
      while ((int32_t)(ld_acquire_sys(mine) - (base + i)) < 0) {
        if ((++spin & 1023u) == 0 && gtimer() > deadline) { ok = false; break; }
      }
      if (me == 1 && ok) st_release_sys(theirs, base + i);
    }
    if (!ok) atomicExch_system(R->err, kErrTimeout);
    if (out) out[0] = ok ? gtimer() - t0 : 0;
    return;
  }
  const unsigned long long nvec = bytes / 16;
  if (mode == 3) {
    const uint4* src = reinterpret_cast<const uint4*>(R->ws[me] + data_off);
    uint4* dst = reinterpret_cast<uint4*>(R->ws[me] + data_off + nvec * 16);
    for (unsigned long long v = (unsigned long long)b * blockDim.x + tid; v < nvec;
         v += (unsigned long long)G * blockDim.x)
      st_ws(dst + v, ld_ws(src + v));
    return;
  }
  const unsigned long long per = nvec / (N - 1);
  for (int pp = 1; pp < N; ++pp) {
    const int p = (me + pp) % N;
    if (mode == 0) {
      uint4* dst = reinterpret_cast<uint4*>(R->ws[p] + data_off) + (unsigned long long)me * per;
      const uint4* src = reinterpret_cast<const uint4*>(R->ws[me] + data_off) + (unsigned long long)(N + pp) * per;
      for (unsigned long long v = (unsigned long long)b * blockDim.x + tid; v < per;
           v += (unsigned long long)G * blockDim.x)
        st_ws(dst + v, ld_ws(src + v));
    } else {
      const uint4* src = reinterpret_cast<const uint4*>(R->ws[p] + data_off) + (unsigned long long)p * per;
      uint4* dst = reinterpret_cast<uint4*>(R->ws[me] + data_off) + (unsigned long long)(N + pp) * per;
      for (unsigned long long v0 = (unsigned long long)b * blockDim.x + tid; v0 < per;
           v0 += 4ull * G * blockDim.x) {
        uint4 r[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const unsigned long long v = v0 + (unsigned long long)u * G * blockDim.x;
          if (v < per) r[u] = ld_ws(src + v);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const unsigned long long v = v0 + (unsigned long long)u * G * blockDim.x;
          if (v < per) st_ws(dst + v, r[u]);
        }
      }
    }
  }
}


// TMA probe (modes 4 push / 5 pull): one elected thread per CTA streams 16 KiB bulk
// copies through a ring of kTmaStages shared-memory buffers.
constexpr int kTmaChunk = 16384;
constexpr int kTmaStages = 8;

__global__ void __launch_bounds__(64) tma_probe_kernel(const RankDev* ranks, unsigned long long data_off,
                                                      unsigned long long bytes, int mode) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kTmaStages * kTmaChunk);
  const RankDev* R = ranks;
  const int N = R->N, me = R->rank, G = gridDim.x, b = blockIdx.x;
  if (mode == 8 || mode == 9) {
    // fence latency inside a CTA whose warp 0 streams TMA (8: pushes, 9: pulls):
    // warp 1 lane 0 of CTA 0 times fences while its sibling warp keeps traffic in flight
    if (threadIdx.x == 32) {
      if (b == 0) {
        unsigned long long t = 0;
        for (int i = 0; i < 100; ++i) {
          const unsigned long long t0 = gtimer();
          asm volatile("fence.acq_rel.sys;" ::: "memory");
          t += gtimer() - t0;
          const unsigned long long w0 = gtimer();
          while (gtimer() - w0 < 2000) {}
        }
        *reinterpret_cast<unsigned long long*>(R->ws[me] + data_off - 65536 + 8192) = t / 100;
      }
      return;
    }
    if (threadIdx.x != 0) return;
    mode = mode == 8 ? 4 : 5;
  }
  if (threadIdx.x != 0) return;
  if (mode == 6 || mode == 7) {
    // fence.acq_rel.sys latency: CTA 0 times 200 fences (mode 6: while the other CTAs
    // stream TMA pushes; mode 7: on a quiet GPU); ns/fence -> barrier area + 8 KiB
    // (data_off = bar_off + 64 KiB, see SlabLayout)
    if (b == 0) {
      const unsigned long long t0 = gtimer();
      for (int i = 0; i < 200; ++i) asm volatile("fence.acq_rel.sys;" ::: "memory");
      *reinterpret_cast<unsigned long long*>(R->ws[me] + data_off - 65536 + 8192) = (gtimer() - t0) / 200;
      return;
    }
    if (mode == 7) return;
    mode = 4;
  }
  for (int s = 0; s < kTmaStages; ++s) mbar_init(&bars[s], 1);
  fence_mbar_init();
  const unsigned long long per = (bytes / (N - 1)) / kTmaChunk * kTmaChunk;
  int issued = 0, done = 0;
  for (int pp = 1; pp < N; ++pp) {
    const int p = (me + pp) % N;
    const char* src;
    char* dst;
    if (mode == 4) {  // push: my slab -> peer's slab
      src = R->ws[me] + data_off + (unsigned long long)(N + pp) * per;
      dst = R->ws[p] + data_off + (unsigned long long)me * per;
    } else {          // pull: peer's slab -> my slab
      src = R->ws[p] + data_off + (unsigned long long)p * per;
      dst = R->ws[me] + data_off + (unsigned long long)(N + pp) * per;
    }
    const unsigned long long nchunks = per / kTmaChunk;
    const unsigned long long c0 = nchunks * b / G, c1 = nchunks * (b + 1) / G;
    // software pipeline: keep up to kTmaStages-1 loads ahead of the stores
    unsigned long long next = c0;
    for (; next < c1 && next - c0 < kTmaStages - 1; ++next, ++issued) {
      const int s = issued % kTmaStages;
      mbar_expect_tx(&bars[s], kTmaChunk);
      tma_load(smem + s * kTmaChunk, src + next * kTmaChunk, kTmaChunk, &bars[s]);
    }
    for (unsigned long long ci = c0; ci < c1; ++ci, ++done) {
      const int s = done % kTmaStages;
      mbar_wait(&bars[s], (done / kTmaStages) & 1);
      tma_store(dst + ci * kTmaChunk, smem + s * kTmaChunk, kTmaChunk);
      tma_commit();
      if (next < c1) {
        tma_wait_read<1>();  // the buffer reloaded next was read by the store before this one
        const int s2 = issued % kTmaStages;
        mbar_expect_tx(&bars[s2], kTmaChunk);
        tma_load(smem + s2 * kTmaChunk, src + next * kTmaChunk, kTmaChunk, &bars[s2]);
        ++next;
        ++issued;
      }
    }
    tma_wait_read<0>();
  }
  tma_wait_all<0>();
}

}  // namespace

cudaError_t launch_probe(const RankDev* ranks, unsigned long long data_off, unsigned long long bytes,
                         int mode, int iters, int ctas, unsigned long long* out, cudaStream_t stream) {
  if (mode >= 4 && mode <= 9) {
    const int smem = kTmaStages * kTmaChunk + kTmaStages * 8;
    cudaError_t e = cudaFuncSetAttribute(tma_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    tma_probe_kernel<<<ctas, mode >= 8 ? 64 : 32, smem, stream>>>(ranks, data_off, bytes, mode);
    return cudaGetLastError();
  }
  probe_kernel<<<mode == 2 ? 1 : ctas, 512, 0, stream>>>(ranks, data_off, bytes, mode, iters, out);
  return cudaGetLastError();
}

}  // namespace torus

// ------------------------------------------------------------------------------------
// Flat ring all-reduce (baseline, PAPER.md:66-70 and its ref [14]): N-1
// reduce-scatter steps then N-1 all-gather steps around the rank ring, HOP policy (every
// message rounded to the wire type, as an NCCL ring does).  Not the product path: it
// exists so the torus can be compared against the ring it replaces (config 3).
// Workspace: 2(N-1) slots of one chunk (RS steps, then AG steps), never reused within a
// call; flag kinds H (RS step s) / R (AG step t), source index = step.
// ------------------------------------------------------------------------------------
namespace torus {
namespace {

template <int DT, int W>
__global__ void __launch_bounds__(512, 1) ring_kernel(const LaunchArgs a) {
  using Acc = typename Wire<W>::Acc;
  constexpr int VE = Wire<W>::VE;
  constexpr int SW = kVecBytes / VE;
  const int lr = blockIdx.x / a.G;
  const int b = blockIdx.x - lr * a.G;
  const RankDev* __restrict__ R = a.ranks + lr;
  const int N = R->N, p = R->rank, G = a.G, q = a.q, tid = threadIdx.x;
  const int next = (p + 1) % N;
  const unsigned long long n = a.n;
  const bool aligned = a.aligned != 0;
  void* const buf = a.buf[lr];
  char* const myws = R->ws[p];
  const unsigned long long slot_bytes = a.hin_stride;  // one chunk of wire data

  __shared__ uint32_t s_e;
  __shared__ int s_abort;
  if (tid == 0) {
    s_e = R->epoch[b] + 1u;
    s_abort = 0;
  }
  __syncthreads();
  const uint32_t e = s_e;
  const unsigned long long deadline = gtimer() + a.timeout_ns;
  auto flag = [&](char* ws, int kind, int step) -> uint32_t* {
    return reinterpret_cast<uint32_t*>(ws) + ((size_t)(kind * kMaxDim + step) * G + b);
  };
  auto slot = [&](char* ws, int kind, int step) -> char* {
    return ws + a.hin_off + ((size_t)kind * (N - 1) + step) * slot_bytes;
  };
  auto wait_prev = [&](int kind, int step) -> bool {
    if (tid == 0 && !wait_flag_ge(flag(myws, kind, step), e, deadline)) {
      atomicExch_system(R->err, kErrTimeout);
      s_abort = 1;
    }
    __syncthreads();
    return s_abort == 0;
  };
  auto signal_next = [&](int kind, int step) {
    __syncthreads();
    if (tid == 0) st_release_sys(flag(R->ws[next], kind, step), e);
  };
  auto slice = [&](int k, unsigned long long* co, unsigned long long* cl, unsigned long long* va,
                   unsigned long long* vz) {
    qpart(n, N, q, k, co, cl);
    const unsigned long long nv = (*cl + VE - 1) / VE;
    *va = nv * (unsigned long long)b / G;
    *vz = nv * (unsigned long long)(b + 1) / G;
  };

  // ---- reduce-scatter: at step s send the partial of chunk (p - s - 1) mod N ----
  for (int s = 0; s <= N - 1; ++s) {
    const int k = ((p - s - 1) % N + N) % N;  // s == N-1: k == p, my finished chunk
    unsigned long long co, cl, va, vz;
    slice(k, &co, &cl, &va, &vz);
    if (s > 0 && !wait_prev(0, s - 1)) return;
    const char* in = slot(myws, 0, s - 1 < 0 ? 0 : s - 1);
    for (unsigned long long v = va + tid; v < vz; v += blockDim.x) {
      const unsigned long long el = v * VE;
      const int nrem = (int)min((unsigned long long)VE, cl - el);
      const uint4 own = load_user<DT, W>(buf, a.buf_off + co + el, nrem, aligned);
      Acc acc[VE];
      unpack<W>(own, acc);
      if (s > 0) {  // partial = incoming message + my own contribution
        Acc t[VE];
        unpack<W>(ld_ws(in + el * SW), t);
        acc_add<W>(t, acc);
#pragma unroll
        for (int i = 0; i < VE; ++i) acc[i] = t[i];
      }
      if (s < N - 1) {
        st_ws(slot(R->ws[next], 0, s) + el * SW, pack<W>(acc));  // HOP: the message is rounded
      } else {
        if (a.op == 1) acc_mean<W>(acc, a.inv_n, N);
        const uint4 out = pack<W>(acc);
        store_user<DT, W>(buf, a.buf_off + co + el, nrem, out, aligned);
        if (N > 1) st_ws(slot(R->ws[next], 1, 0) + el * SW, out);  // all-gather step 0
      }
    }
    if (s < N - 1) signal_next(0, s);
  }
  if (N > 1) signal_next(1, 0);
  // ---- all-gather: at step t forward chunk (p - t) mod N, received at step t-1 ----
  for (int t = 1; t <= N - 1; ++t) {
    const int k = ((p - t) % N + N) % N;
    unsigned long long co, cl, va, vz;
    slice(k, &co, &cl, &va, &vz);
    if (!wait_prev(1, t - 1)) return;
    const char* in = slot(myws, 1, t - 1);
    for (unsigned long long v = va + tid; v < vz; v += blockDim.x) {
      const unsigned long long el = v * VE;
      const int nrem = (int)min((unsigned long long)VE, cl - el);
      const uint4 w = ld_ws(in + el * SW);
      store_user<DT, W>(buf, a.buf_off + co + el, nrem, w, aligned);
      if (t < N - 1) st_ws(slot(R->ws[next], 1, t) + el * SW, w);
    }
    if (t < N - 1) signal_next(1, t);
  }
  __syncthreads();
  if (tid == 0) R->epoch[b] = e;
}

template <int DT, int W>
cudaError_t launch_ring_typed(const LaunchArgs& a, bool cooperative, cudaStream_t stream) {
  const dim3 grid(a.nlocal * a.G), block(512);
  if (cooperative) {
    void* args[] = {const_cast<LaunchArgs*>(&a)};
    return cudaLaunchCooperativeKernel((const void*)ring_kernel<DT, W>, grid, block, args, 0, stream);
  }
  ring_kernel<DT, W><<<grid, block, 0, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_ring(const LaunchArgs& a, int dtype, int wire, bool cooperative, cudaStream_t stream) {
  if (dtype == wire) {
    switch (dtype) {
      case DT_F32: return launch_ring_typed<DT_F32, DT_F32>(a, cooperative, stream);
      case DT_F16: return launch_ring_typed<DT_F16, DT_F16>(a, cooperative, stream);
      case DT_BF16: return launch_ring_typed<DT_BF16, DT_BF16>(a, cooperative, stream);
      case DT_I32: return launch_ring_typed<DT_I32, DT_I32>(a, cooperative, stream);
    }
  } else if (dtype == DT_F32 && wire == DT_F16) {
    return launch_ring_typed<DT_F32, DT_F16>(a, cooperative, stream);
  } else if (dtype == DT_F32 && wire == DT_BF16) {
    return launch_ring_typed<DT_F32, DT_BF16>(a, cooperative, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace torus

// ------------------------------------------------------------------------------------
// Multi-tensor pack / unpack (NEXT-1, BASELINE.json config 5): the bucket's tensors are
// concatenated in order into a wire-typed staging buffer (cast fused, round to nearest
// even) and scattered back (up-cast fused) -- exactly the all-reduce of the concatenated
// buffer with dtype -> wire conversion on the first read and back on the last write.
// The tensor table travels in the kernel parameters (no host->device copy per call).
// ------------------------------------------------------------------------------------
namespace torus {
namespace {

template <int DT, int W, bool PACK>
__global__ void __launch_bounds__(256) multi_copy_kernel(const MultiTable tab, void* staging) {
  using UT = typename Elem<DT>::T;
  using WT = typename Elem<W>::T;
  const int t = blockIdx.y;
  const unsigned long long n = tab.count[t];
  UT* user = reinterpret_cast<UT*>(tab.ptr[t]);
  WT* st = reinterpret_cast<WT*>(staging) + tab.offset[t];
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    if constexpr (PACK) {
      if constexpr (DT == W) st[i] = user[i];
      else if constexpr (W == DT_F16) st[i] = __float2half_rn(user[i]);
      else st[i] = __float2bfloat16_rn(user[i]);
    } else {
      if constexpr (DT == W) user[i] = st[i];
      else user[i] = static_cast<float>(st[i]);  // exact
    }
  }
}

template <int DT, int W>
cudaError_t launch_multi_typed(const MultiTable& tab, int n, void* staging, bool pack, cudaStream_t s) {
  unsigned long long mx = 1;
  for (int i = 0; i < n; ++i) mx = tab.count[i] > mx ? tab.count[i] : mx;
  const unsigned gx = (unsigned)((mx + 255) / 256 < 296 ? (mx + 255) / 256 : 296);
  const dim3 grid(gx, n);
  if (pack) multi_copy_kernel<DT, W, true><<<grid, 256, 0, s>>>(tab, staging);
  else multi_copy_kernel<DT, W, false><<<grid, 256, 0, s>>>(tab, staging);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_multi_copy(const MultiTable& tab, int n, int dtype, int wire, void* staging,
                              bool pack, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  if (dtype == wire) {
    switch (dtype) {
      case DT_F32: return launch_multi_typed<DT_F32, DT_F32>(tab, n, staging, pack, stream);
      case DT_F16: return launch_multi_typed<DT_F16, DT_F16>(tab, n, staging, pack, stream);
      case DT_BF16: return launch_multi_typed<DT_BF16, DT_BF16>(tab, n, staging, pack, stream);
      case DT_I32: return launch_multi_typed<DT_I32, DT_I32>(tab, n, staging, pack, stream);
    }
  } else if (dtype == DT_F32 && wire == DT_F16) {
    return launch_multi_typed<DT_F32, DT_F16>(tab, n, staging, pack, stream);
  } else if (dtype == DT_F32 && wire == DT_BF16) {
    return launch_multi_typed<DT_F32, DT_BF16>(tab, n, staging, pack, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace torus

// ------------------------------------------------------------------------------------
// Hierarchical all-reduce (baseline [6]; NEXT-3): per
// row, a chain reduce of the FULL buffer to the column-0 leader; a ring all-reduce of the
// full buffer among the Y leaders; a chain broadcast back along each row.  Every message
// is rounded to the wire type (HOP).  Workspace (wire elements, round of n): chain slot
// [n], broadcast slot [n], leader-ring slots 2(Y-1) x [n/Y].  Flags: H = chain step,
// V / AG = leader-ring RS / AG step, R = broadcast step (source index = step).
// ------------------------------------------------------------------------------------
namespace torus {
namespace {

template <int DT, int W>
__global__ void __launch_bounds__(512, 1) hier_kernel(const LaunchArgs a) {
  using Acc = typename Wire<W>::Acc;
  constexpr int VE = Wire<W>::VE;
  constexpr int SW = kVecBytes / VE;
  const int lr = blockIdx.x / a.G;
  const int b = blockIdx.x - lr * a.G;
  const RankDev* __restrict__ R = a.ranks + lr;
  const int X = R->X, Y = R->Y, N = R->N, rho = R->rho, c = R->c, G = a.G, q = a.q, tid = threadIdx.x;
  const unsigned long long n = a.n;
  const bool aligned = a.aligned != 0;
  void* const buf = a.buf[lr];
  char* const myws = R->ws[R->rank];
  char* const chain_slot = myws + a.hin_off;                 // [n]
  char* const bcast_slot = chain_slot + a.hin_stride;        // [n]
  char* const ring_base = bcast_slot + a.hin_stride;         // 2(Y-1) x [vin_stride]
  const unsigned long long ring_slot = a.vin_stride;
  auto rank_of = [&](int row, int col) { return row * X + col; };

  __shared__ uint32_t s_e;
  __shared__ int s_abort;
  if (tid == 0) {
    s_e = R->epoch[b] + 1u;
    s_abort = 0;
  }
  __syncthreads();
  const uint32_t e = s_e;
  const unsigned long long deadline = gtimer() + a.timeout_ns;
  auto flag = [&](char* ws, int kind, int step) -> uint32_t* {
    return reinterpret_cast<uint32_t*>(ws) + ((size_t)(kind * kMaxDim + step) * G + b);
  };
  auto wait_in = [&](int kind, int step) -> bool {
    if (tid == 0 && !wait_flag_ge(flag(myws, kind, step), e, deadline)) {
      atomicExch_system(R->err, kErrTimeout);
      s_abort = 1;
    }
    __syncthreads();
    return s_abort == 0;
  };
  auto signal_to = [&](int peer, int kind, int step) {
    __syncthreads();
    if (tid == 0) st_release_sys(flag(R->ws[peer], kind, step), e);
  };
  // CTA b's slice of [0, len) in vectors
  auto slice = [&](unsigned long long len, unsigned long long* va, unsigned long long* vz) {
    const unsigned long long nv = (len + VE - 1) / VE;
    *va = nv * (unsigned long long)b / G;
    *vz = nv * (unsigned long long)(b + 1) / G;
  };
  // CTA b owns slice b of each of the Y leader-ring chunks in EVERY phase, so no phase
  // reads another CTA's data (no grid-wide synchronization needed)
  auto for_mine = [&](auto f) {
    for (int k = 0; k < Y; ++k) {
      unsigned long long co, cl, pa, pz;
      qpart(n, Y, q, k, &co, &cl);
      slice(cl, &pa, &pz);
      for (unsigned long long v = pa + tid; v < pz; v += blockDim.x) {
        const unsigned long long el = co + v * VE;
        f(el, (int)min((unsigned long long)VE, co + cl - el));
      }
    }
  };

  // ---- phase 1: chain reduce to the leader (column X-1 -> ... -> 0) ----
  // column c receives at step X-2-c from column c+1 and sends at step X-1-c to c-1
  if (c < X - 1 && !wait_in(kFlagH, X - 2 - c)) return;
  for_mine([&](unsigned long long el, int nrem) {
    Acc acc[VE];
    unpack<W>(load_user<DT, W>(buf, a.buf_off + el, nrem, aligned), acc);
    if (c < X - 1) {  // partial = incoming message + my own contribution
      Acc t[VE];
      unpack<W>(ld_ws(chain_slot + el * SW), t);
      acc_add<W>(t, acc);
#pragma unroll
      for (int i = 0; i < VE; ++i) acc[i] = t[i];
    }
    if (c > 0) {
      st_ws(R->ws[rank_of(rho, c - 1)] + a.hin_off + el * SW, pack<W>(acc));
    } else {  // leader: the row sum, rounded once (mean here if there is no vertical phase)
      if (Y == 1 && a.op == 1) acc_mean<W>(acc, a.inv_n, N);
      st_ws(chain_slot + el * SW, pack<W>(acc));  // the leader keeps its value in place
    }
  });
  if (c > 0) signal_to(rank_of(rho, c - 1), kFlagH, X - 1 - c);
  __syncthreads();

  // ---- phase 2: ring all-reduce of the full buffer among the Y leaders ----
  if (c == 0 && Y > 1) {
    const int nextl = rank_of((rho + 1) % Y, 0);
    auto rslot = [&](char* ws, int kind, int step) -> char* {
      return ws + (a.hin_off + 2 * a.hin_stride) + ((size_t)kind * (Y - 1) + step) * ring_slot;
    };
    auto part = [&](int k, unsigned long long* co, unsigned long long* cl, unsigned long long* pa,
                    unsigned long long* pz) {
      qpart(n, Y, q, k, co, cl);
      slice(*cl, pa, pz);
    };
    for (int s = 0; s <= Y - 1; ++s) {  // reduce-scatter over the leader ring
      const int k = ((rho - s - 1) % Y + Y) % Y;
      unsigned long long co, cl, pa, pz;
      part(k, &co, &cl, &pa, &pz);
      if (s > 0 && !wait_in(kFlagV, s - 1)) return;
      for (unsigned long long v = pa + tid; v < pz; v += blockDim.x) {
        const unsigned long long el = v * VE;
        Acc acc[VE];
        unpack<W>(ld_ws(chain_slot + (co + el) * SW), acc);
        if (s > 0) {
          Acc t[VE];
          unpack<W>(ld_ws(rslot(myws, 0, s - 1) + el * SW), t);
          acc_add<W>(t, acc);
#pragma unroll
          for (int i = 0; i < VE; ++i) acc[i] = t[i];
        }
        if (s < Y - 1) {
          st_ws(rslot(R->ws[nextl], 0, s) + el * SW, pack<W>(acc));
        } else {
          if (a.op == 1) acc_mean<W>(acc, a.inv_n, N);
          const uint4 out = pack<W>(acc);
          st_ws(chain_slot + (co + el) * SW, out);           // final chunk, in place
          st_ws(rslot(R->ws[nextl], 1, 0) + el * SW, out);   // all-gather step 0
        }
      }
      if (s < Y - 1) signal_to(nextl, kFlagV, s);
    }
    signal_to(nextl, kFlagAG, 0);
    for (int t = 1; t <= Y - 1; ++t) {  // all-gather over the leader ring
      const int k = ((rho - t) % Y + Y) % Y;
      unsigned long long co, cl, pa, pz;
      part(k, &co, &cl, &pa, &pz);
      if (!wait_in(kFlagAG, t - 1)) return;
      for (unsigned long long v = pa + tid; v < pz; v += blockDim.x) {
        const unsigned long long el = v * VE;
        const uint4 w = ld_ws(rslot(myws, 1, t - 1) + el * SW);
        st_ws(chain_slot + (co + el) * SW, w);
        if (t < Y - 1) st_ws(rslot(R->ws[nextl], 1, t) + el * SW, w);
      }
      if (t < Y - 1) signal_to(nextl, kFlagAG, t);
    }
    __syncthreads();
  }

  // ---- phase 3: chain broadcast from the leader (column 0 -> 1 -> ... -> X-1) ----
  const char* const src = (c == 0) ? chain_slot : bcast_slot;
  if (c > 0 && !wait_in(kFlagR, c - 1)) return;
  for_mine([&](unsigned long long el, int nrem) {
    const uint4 w = ld_ws(src + el * SW);
    store_user<DT, W>(buf, a.buf_off + el, nrem, w, aligned);
    if (c < X - 1) st_ws(R->ws[rank_of(rho, c + 1)] + a.hin_off + a.hin_stride + el * SW, w);
  });
  if (c < X - 1) signal_to(rank_of(rho, c + 1), kFlagR, c);
  __syncthreads();
  if (tid == 0) R->epoch[b] = e;
}

template <int DT, int W>
cudaError_t launch_hier_typed(const LaunchArgs& a, bool cooperative, cudaStream_t stream) {
  const dim3 grid(a.nlocal * a.G), block(512);
  if (cooperative) {
    void* args[] = {const_cast<LaunchArgs*>(&a)};
    return cudaLaunchCooperativeKernel((const void*)hier_kernel<DT, W>, grid, block, args, 0, stream);
  }
  hier_kernel<DT, W><<<grid, block, 0, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_hier(const LaunchArgs& a, int dtype, int wire, bool cooperative, cudaStream_t stream) {
  if (dtype == wire) {
    switch (dtype) {
      case DT_F32: return launch_hier_typed<DT_F32, DT_F32>(a, cooperative, stream);
      case DT_F16: return launch_hier_typed<DT_F16, DT_F16>(a, cooperative, stream);
      case DT_BF16: return launch_hier_typed<DT_BF16, DT_BF16>(a, cooperative, stream);
      case DT_I32: return launch_hier_typed<DT_I32, DT_I32>(a, cooperative, stream);
    }
  } else if (dtype == DT_F32 && wire == DT_F16) {
    return launch_hier_typed<DT_F32, DT_F16>(a, cooperative, stream);
  } else if (dtype == DT_F32 && wire == DT_BF16) {
    return launch_hier_typed<DT_F32, DT_BF16>(a, cooperative, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace torus

// ------------------------------------------------------------------------------------
// Small-message one-shot kernel (NEXT-2; BASELINE.json config 4's 4 KB - 1 MB
// range).  Below ~1 MB the torus's four dependent hand-offs (H-RS, V-RS, V-AG, H-AG,
// PAPER.md:70) cost more than the bytes: each is a fence plus an NVLink round trip.  Here
// every rank broadcasts its whole (wire-cast) buffer to every peer once, as "LL" lines that
// carry their own epoch flag in every 8-byte word ({data32, flag32}, single-copy atomic),
// so there is no fence, no flag word and no block barrier on the path -- one NVLink
// latency per call.  Each thread then holds all N ranks' values of its 16-byte vector and
// evaluates the torus fold in the paper's order (row fold over columns
// c+1..c rounded to the wire at the phase output, column fold over rows s+1..s, mean at
// the last reduce phase), so the result is bit-identical to the multi-phase kernel and to
// the oracle.  Traffic is (N-1) * 2 * S per rank instead of 2(N-1)/N * S: the right trade
// only while latency dominates (threshold TORUS_LL_MAX_BYTES).
//
// Slab region (per rank, SlabLayout::ll_off): [parity 2][src N] slots of ll_slot bytes;
// a slot holds line 0 of every vector in its first half and line 1 in its second, so a
// warp's stores are contiguous.  parity = epoch & 1 (a rank can be at most one call ahead
// of a peer still reading, so two buffers suffice); flag = epoch + 1 (slab starts zeroed).
// ------------------------------------------------------------------------------------
namespace torus {
namespace {

constexpr int kLLThreads = 256;

__device__ __forceinline__ void st_ll(char* p, uint32_t d0, uint32_t d1, uint32_t flag) {
  const unsigned long long a = ((unsigned long long)flag << 32) | d0;
  const unsigned long long b = ((unsigned long long)flag << 32) | d1;
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

// Spin until both 8-byte words of the line carry `flag`; returns false on the deadline.
__device__ __forceinline__ bool ld_ll(const char* p, uint32_t flag, unsigned long long deadline,
                                      uint32_t* d0, uint32_t* d1) {
  unsigned spin = 0;
  for (;;) {
    unsigned long long a, b;
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
    if ((uint32_t)(a >> 32) == flag && (uint32_t)(b >> 32) == flag) {
      *d0 = (uint32_t)a;
      *d1 = (uint32_t)b;
      return true;
    }
    if ((++spin & 255u) == 0 && gtimer() > deadline) return false;
  }
}

template <int DT, int W>
__global__ void __launch_bounds__(kLLThreads) ll_kernel(const LaunchArgs a) {
  constexpr int VE = Wire<W>::VE;
  using Acc = typename Wire<W>::Acc;
  const int l = blockIdx.x / a.G, b = blockIdx.x % a.G;
  const RankDev* R = a.ranks + l;
  const int X = R->X, Y = R->Y, N = R->N, me = R->rank;
  uint32_t* ctr = R->ll_ctr;  // [0] epoch, [1] CTAs done in this call
  const uint32_t ep = *reinterpret_cast<volatile uint32_t*>(ctr);
  const uint32_t flag = ep + 1;
  const unsigned long long par = ep & 1u;
  const unsigned long long half = a.ll_slot / 2;
  const unsigned long long n = a.n;
  const unsigned long long nvec = (n + VE - 1) / VE;
  const unsigned long long stride = (unsigned long long)a.G * kLLThreads;
  const unsigned long long j0 = (unsigned long long)b * kLLThreads + threadIdx.x;
  void* buf = a.buf[l];
  auto slot = [&](int owner, int src) {
    return R->ws[owner] + a.ll_off + par * a.ll_half + src * a.ll_slot;
  };

  // 1. broadcast my vectors (cast to the wire on the first read, C1) to every peer
  for (unsigned long long j = j0; j < nvec; j += stride) {
    const unsigned long long e = j * VE;
    const int nrem = (int)(n - e < (unsigned long long)VE ? n - e : VE);
    const uint4 v = load_user<DT, W>(buf, a.buf_off + e, nrem, a.aligned);
    for (int k = 1; k < N; ++k) {
      char* s = slot((me + k) % N, me);
      st_ll(s + j * 16, v.x, v.y, flag);
      st_ll(s + half + j * 16, v.z, v.w, flag);
    }
  }

  // 2. gather and fold in the torus order (C4-C8)
  const unsigned long long deadline = gtimer() + a.timeout_ns;
  bool ok = true;
  for (unsigned long long j = j0; ok && j < nvec; j += stride) {
    const unsigned long long e = j * VE;
    const int nrem = (int)(n - e < (unsigned long long)VE ? n - e : VE);
    // chunk c (row partition) and sub-chunk s (column partition) of this vector: both
    // partitions are quantum (= one 16-byte vector) aligned, so the vector is in one piece
    int c = 0, s = 0;
    unsigned long long co = 0, cl = 0, so = 0, sl = 0;
    for (c = 0; c < X; ++c) {
      qpart(n, X, a.q, c, &co, &cl);
      if (e < co + cl) break;
    }
    for (s = 0; s < Y; ++s) {
      qpart(cl, Y, a.q, s, &so, &sl);
      if (e - co < so + sl) break;
    }
    const uint4 own = load_user<DT, W>(buf, a.buf_off + e, nrem, a.aligned);
    Acc V[VE], P[VE], t[VE];
    for (int kr = 1; kr <= Y && ok; ++kr) {
      const int rho = (s + kr) % Y;
      for (int kc = 1; kc <= X; ++kc) {
        const int r = rho * X + (c + kc) % X;
        uint4 w = own;
        if (r != me) {
          const char* src = slot(me, r);
          ok = ld_ll(src + j * 16, flag, deadline, &w.x, &w.y) &&
               ld_ll(src + half + j * 16, flag, deadline, &w.z, &w.w);
          if (!ok) break;
        }
        if (kc == 1) unpack<W>(w, P);
        else { unpack<W>(w, t); acc_add<W>(P, t); }
      }
      if (!ok) break;
      if (Y == 1) {  // H-RS is the last reduce phase: mean there (C8), one rounding
        if (a.op) acc_mean<W>(P, a.inv_n, N);
        store_user<DT, W>(buf, a.buf_off + e, nrem, pack<W>(P), a.aligned);
      } else {       // phase-1 output rounded to the wire (PHASE policy, C7)
        unpack<W>(pack<W>(P), t);
        if (kr == 1) {
#pragma unroll
          for (int i = 0; i < VE; ++i) V[i] = t[i];
        } else {
          acc_add<W>(V, t);
        }
      }
    }
    if (!ok) break;
    if (Y > 1) {
      if (a.op) acc_mean<W>(V, a.inv_n, N);
      store_user<DT, W>(buf, a.buf_off + e, nrem, pack<W>(V), a.aligned);
    }
  }
  if (!ok) atomicExch_system(R->err, kErrTimeout);

  // 3. the last CTA of this rank to finish advances the epoch (every CTA read it above)
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(ctr + 1, 1u) == (uint32_t)a.G - 1) {
      ctr[1] = 0;
      ctr[0] = ep + 1;
    }
  }
}

// Two-shot variant (mid-size messages, N >= 3): the same fence-free LL lines, but only
// 2 * 2(N-1)/N * S bytes per rank.  Shot 1: every rank sends each sub-chunk C_{c,s} to
// its torus owner, rank (s, c) (PAPER.md:70's final owner after H-RS + V-RS).  The owner
// folds its sub-chunk in the torus order (C4-C8, as above).  Shot 2: it broadcasts the
// reduced sub-chunk, and every rank writes it to its buffer (the all-gather is a copy).
// Region per parity (at par * ll_half): rs[src N] then ag[owner N], slots of ll_slot
// bytes (two LL lines per 16-byte vector of the largest sub-chunk).
template <int DT, int W>
__global__ void __launch_bounds__(kLLThreads) ll2_kernel(const LaunchArgs a) {
  constexpr int VE = Wire<W>::VE;
  using Acc = typename Wire<W>::Acc;
  const int l = blockIdx.x / a.G, b = blockIdx.x % a.G;
  const RankDev* R = a.ranks + l;
  const int X = R->X, Y = R->Y, N = R->N, me = R->rank, rho = R->rho, cc = R->c;
  uint32_t* ctr = R->ll_ctr;
  const uint32_t ep = *reinterpret_cast<volatile uint32_t*>(ctr);
  const uint32_t flag = ep + 1;
  const unsigned long long par = ep & 1u;
  const unsigned long long half = a.ll_slot / 2;
  const unsigned long long n = a.n;
  const unsigned long long nvec = (n + VE - 1) / VE;
  const unsigned long long stride = (unsigned long long)a.G * kLLThreads;
  const unsigned long long j0 = (unsigned long long)b * kLLThreads + threadIdx.x;
  void* buf = a.buf[l];
  auto rs = [&](int owner, int src) {
    return R->ws[owner] + a.ll_off + par * a.ll_half + src * a.ll_slot;
  };
  auto ag = [&](int holder, int owner) {
    return R->ws[holder] + a.ll_off + par * a.ll_half + (N + owner) * a.ll_slot;
  };
  // owner rank and vector index inside the owner's sub-chunk of element e
  auto locate = [&](unsigned long long e, int* owner, unsigned long long* v) {
    unsigned long long co = 0, cl = 0, so = 0, sl = 0;
    int c = 0, s = 0;
    for (c = 0; c < X; ++c) {
      qpart(n, X, a.q, c, &co, &cl);
      if (e < co + cl) break;
    }
    for (s = 0; s < Y; ++s) {
      qpart(cl, Y, a.q, s, &so, &sl);
      if (e - co < so + sl) break;
    }
    *owner = s * X + c;
    *v = (e - co - so) / VE;
  };
  // my sub-chunk C_{c, rho}
  unsigned long long mco, mcl, mso, msl;
  qpart(n, X, a.q, cc, &mco, &mcl);
  qpart(mcl, Y, a.q, rho, &mso, &msl);
  const unsigned long long my0 = mco + mso, myvec = (msl + VE - 1) / VE;

  // shot 1: every vector to its owner
  for (unsigned long long j = j0; j < nvec; j += stride) {
    const unsigned long long e = j * VE;
    int o;
    unsigned long long v;
    locate(e, &o, &v);
    if (o == me) continue;
    const int nrem = (int)(n - e < (unsigned long long)VE ? n - e : VE);
    const uint4 w = load_user<DT, W>(buf, a.buf_off + e, nrem, a.aligned);
    char* d = rs(o, me);
    st_ll(d + v * 16, w.x, w.y, flag);
    st_ll(d + half + v * 16, w.z, w.w, flag);
  }

  const unsigned long long deadline = gtimer() + a.timeout_ns;
  bool ok = true;
  // fold my sub-chunk in the torus order, then broadcast it
  for (unsigned long long v = j0; ok && v < myvec; v += stride) {
    const unsigned long long e = my0 + v * VE;
    const int nrem = (int)(my0 + msl - e < (unsigned long long)VE ? my0 + msl - e : VE);
    const uint4 own = load_user<DT, W>(buf, a.buf_off + e, nrem, a.aligned);
    Acc V[VE], P[VE], t[VE];
    uint4 out = own;
    for (int kr = 1; kr <= Y && ok; ++kr) {
      const int r0 = (rho + kr) % Y;
      for (int kc = 1; kc <= X; ++kc) {
        const int r = r0 * X + (cc + kc) % X;
        uint4 w = own;
        if (r != me) {
          const char* src = rs(me, r);
          ok = ld_ll(src + v * 16, flag, deadline, &w.x, &w.y) &&
               ld_ll(src + half + v * 16, flag, deadline, &w.z, &w.w);
          if (!ok) break;
        }
        if (kc == 1) unpack<W>(w, P);
        else { unpack<W>(w, t); acc_add<W>(P, t); }
      }
      if (!ok) break;
      if (Y == 1) {
        if (a.op) acc_mean<W>(P, a.inv_n, N);
        out = pack<W>(P);
      } else {
        unpack<W>(pack<W>(P), t);
        if (kr == 1) {
#pragma unroll
          for (int i = 0; i < VE; ++i) V[i] = t[i];
        } else {
          acc_add<W>(V, t);
        }
      }
    }
    if (!ok) break;
    if (Y > 1) {
      if (a.op) acc_mean<W>(V, a.inv_n, N);
      out = pack<W>(V);
    }
    store_user<DT, W>(buf, a.buf_off + e, nrem, out, a.aligned);
    for (int k = 1; k < N; ++k) {
      char* d = ag((me + k) % N, me);
      st_ll(d + v * 16, out.x, out.y, flag);
      st_ll(d + half + v * 16, out.z, out.w, flag);
    }
  }
  // shot 2: write every other owner's reduced sub-chunk
  for (unsigned long long j = j0; ok && j < nvec; j += stride) {
    const unsigned long long e = j * VE;
    int o;
    unsigned long long v;
    locate(e, &o, &v);
    if (o == me) continue;
    uint4 w;
    const char* src = ag(me, o);
    ok = ld_ll(src + v * 16, flag, deadline, &w.x, &w.y) &&
         ld_ll(src + half + v * 16, flag, deadline, &w.z, &w.w);
    if (!ok) break;
    const int nrem = (int)(n - e < (unsigned long long)VE ? n - e : VE);
    store_user<DT, W>(buf, a.buf_off + e, nrem, w, a.aligned);
  }
  if (!ok) atomicExch_system(R->err, kErrTimeout);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(ctr + 1, 1u) == (uint32_t)a.G - 1) {
      ctr[1] = 0;
      ctr[0] = ep + 1;
    }
  }
}

template <int DT, int W>
cudaError_t launch_ll_typed(const LaunchArgs& a, bool cooperative, cudaStream_t stream) {
  const dim3 grid(a.nlocal * a.G), block(kLLThreads);
  const void* fn = a.ll_two_shot ? (const void*)ll2_kernel<DT, W> : (const void*)ll_kernel<DT, W>;
  if (cooperative) {
    void* args[] = {const_cast<LaunchArgs*>(&a)};
    return cudaLaunchCooperativeKernel(fn, grid, block, args, 0, stream);
  }
  if (a.ll_two_shot) ll2_kernel<DT, W><<<grid, block, 0, stream>>>(a);
  else ll_kernel<DT, W><<<grid, block, 0, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_ll(const LaunchArgs& a, int dtype, int wire, bool cooperative, cudaStream_t stream) {
  if (dtype == wire) {
    switch (dtype) {
      case DT_F32: return launch_ll_typed<DT_F32, DT_F32>(a, cooperative, stream);
      case DT_F16: return launch_ll_typed<DT_F16, DT_F16>(a, cooperative, stream);
      case DT_BF16: return launch_ll_typed<DT_BF16, DT_BF16>(a, cooperative, stream);
      case DT_I32: return launch_ll_typed<DT_I32, DT_I32>(a, cooperative, stream);
    }
  } else if (dtype == DT_F32 && wire == DT_F16) {
    return launch_ll_typed<DT_F32, DT_F16>(a, cooperative, stream);
  } else if (dtype == DT_F32 && wire == DT_BF16) {
    return launch_ll_typed<DT_F32, DT_BF16>(a, cooperative, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace torus
