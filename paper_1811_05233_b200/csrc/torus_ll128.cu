// torus_ll128.cu -- the 2D-Torus all-reduce as a fence-free push pipeline:
// every byte crosses NVLink as a STORE into the consumer's slab, in 128-byte "LL128" lines
// that carry their own 8-byte flag (120 bytes of data + the call's epoch), so the consumer
// polls the data itself: no system fence, no flag word, no tile barrier anywhere.
//
//   stage A (a2)  push my buffer's share of every row peer's chunk into its H inbox
//   stage B (a2)  fold my chunk's X shares in ring order c+1, ..., c, round to
//                 the wire, push to the V inbox of the sub-chunk's column owner
//                 (Y == 1: mean, round, final -> my buffer + the row peers' HAG inboxes)
//   stage C (a3)  fold my sub-chunk's Y rows in ring order rho+1, ..., rho, mean (C8), round
//                 once -> my buffer, the column peers' AG inboxes, the row peers' HAG inboxes
//   stage D (a4)  a column peer's reduced sub-chunk -> my buffer + the row peers' HAG inboxes
//   stage E (a5)  a row peer's completed chunk -> my buffer (up-cast fused)
//
// A warp moves one "unit" at a time: four 128-byte lines, lanes 8g..8g+7 writing line g,
// 16 bytes each; lane 8g+7 writes 8 bytes of data and the flag.  A unit holds 30 wire
// vectors: lanes with (lane & 7) < 7 carry whole vectors 0..27 (16-byte aligned in the user
// buffer), the four flag lanes carry the halves of vectors 28 and 29.  The protocol relies
// on a warp's 16-byte-per-lane store of an aligned 128-byte line reaching the peer as one
// line write, and on the reader's 8-lane load of it being one line read, so that a reader
// who sees the flag sees the line -- NCCL's LL128 protocol makes the same assumption on
// NVLink.  The bit-exact parity tests are the check that it holds here.
//
// Every stage has its own warps, each looping over its units in unit-major order, so a
// stage starts unit u of a sub-chunk as soon as that unit's lines land.  Inboxes are
// double-buffered by call parity (a rank is at most one call ahead of any row or column
// peer: every call reads lines from all of them).  Fold order, partition, rounding points
// and the mean placement are the oracle's: every dtype is bit-exact.
#include <cstdio>
#include <cstdlib>

#include "torus_device.cuh"
#include "torus_ll128.h"

namespace torus {
namespace {

#ifndef TORUS_LL128_THREADS
#define TORUS_LL128_THREADS 1024
#endif
enum { kSA = 0, kSB = 1, kSC = 2, kSD = 3, kSE = 4, kL128Stages = 5 };

// NS = 16-byte slots per lane: 1 (a lane writes 16 bytes, 8 lanes per 128-byte line, a
// warp moves 4 lines = 30 wire vectors per unit) or 2 (32-byte lanes, 4 lanes per line,
// 8 lines = 60 vectors per unit: half the memory instructions and polls per byte).  The
// last lane of every line writes the line's flag in its last 8 bytes.
template <int NS>
struct Geo {
  static constexpr int kLPL = 8 / NS;             // lanes per line
  static constexpr int kLines = 4 * NS;           // lines per unit
  static constexpr int kUnitBytes = kLines * kL128Line;
  static constexpr int kThreads = NS == 1 ? TORUS_LL128_THREADS : 512;
  static constexpr int kWarps = kThreads / 32;
};
template <int NS>
struct LV {
  uint4 s[NS];
};

template <int NS>
__device__ __forceinline__ bool flag_lane(int lane) {
  return (lane % Geo<NS>::kLPL) == Geo<NS>::kLPL - 1;
}

// slot h of this lane: element offset inside the unit and element count
template <int VE, int NS>
__device__ __forceinline__ void lane_slice(int lane, int h, int* eoff, int* cnt) {
  constexpr int LPL = Geo<NS>::kLPL, L = Geo<NS>::kLines;
  const int g = lane / LPL, li = lane % LPL;
  if (li < LPL - 1) {  // whole vectors, 16-byte aligned in the user buffer
    *eoff = ((g * (LPL - 1) + li) * NS + h) * VE;
    *cnt = VE;
  } else if (h < NS - 1) {  // NS = 2: the flag lane's first slot is a whole vector
    *eoff = (L * (LPL - 1) * NS + g) * VE;
    *cnt = VE;
  } else {  // the flag lane's last slot: half a vector (8 bytes) beside the flag
    const int base = L * (LPL - 1) * NS + L * (NS - 1);
    *eoff = (base + (g >> 1)) * VE + (g & 1) * (VE / 2);
    *cnt = VE / 2;
  }
}

template <int NS>
__device__ __forceinline__ char* lane_ptr(char* stream, unsigned long long u, int lane) {
  return stream + u * Geo<NS>::kUnitBytes + (lane / Geo<NS>::kLPL) * kL128Line + (lane % Geo<NS>::kLPL) * (16 * NS);
}

__device__ __forceinline__ uint64_t lo64(uint4 v) { return (uint64_t)v.x | ((uint64_t)v.y << 32); }
__device__ __forceinline__ uint64_t hi64(uint4 v) { return (uint64_t)v.z | ((uint64_t)v.w << 32); }
__device__ __forceinline__ uint4 mk4(uint64_t lo, uint64_t hi) {
  return make_uint4((uint32_t)lo, (uint32_t)(lo >> 32), (uint32_t)hi, (uint32_t)(hi >> 32));
}

// write this lane's share of a unit (the flag lane: its last 8 bytes are the flag)
template <int NS>
__device__ __forceinline__ void put(char* stream, unsigned long long u, int lane, const LV<NS>& v, uint64_t flag) {
  char* p = lane_ptr<NS>(stream, u, lane);
  const bool fl = flag_lane<NS>(lane);
  if constexpr (NS == 1) {
    asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(lo64(v.s[0])),
                 "l"(fl ? flag : hi64(v.s[0])) : "memory");
  } else {
    asm volatile("st.volatile.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(lo64(v.s[0])),
                 "l"(hi64(v.s[0])), "l"(lo64(v.s[1])), "l"(fl ? flag : hi64(v.s[1])) : "memory");
  }
}

// one load of this lane's share; returns the last 8 bytes (the flag on a flag lane)
template <int NS>
__device__ __forceinline__ uint64_t ld_share(const char* p, uint64_t (&w)[2 * NS]) {
  if constexpr (NS == 1) {
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(w[0]), "=l"(w[1]) : "l"(p) : "memory");
  } else {
    asm volatile("ld.volatile.global.v4.u64 {%0, %1, %2, %3}, [%4];"
                 : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3]) : "l"(p) : "memory");
  }
  return w[2 * NS - 1];
}
template <int NS>
__device__ __forceinline__ LV<NS> to_lv(const uint64_t (&w)[2 * NS], bool fl) {
  LV<NS> v;
#pragma unroll
  for (int h = 0; h < NS; ++h) v.s[h] = mk4(w[2 * h], (fl && h == NS - 1) ? 0ull : w[2 * h + 1]);
  return v;
}

// poll verdict of one unit: every line's flag lane saw `flag`.  Warp-collective.
template <int NS>
__device__ __forceinline__ bool unit_ready(int lane, uint64_t last, uint64_t flag) {
  constexpr int LPL = Geo<NS>::kLPL;
  const int mine = !flag_lane<NS>(lane) || last == flag;
  return __all_sync(0xffffffffu, __shfl_sync(0xffffffffu, mine, (lane & ~(LPL - 1)) | (LPL - 1)));
}

// back off once the lines are clearly not there yet: thousands of warps re-reading the
// same L2 lines at full speed slow the NVLink writes that must land in them
__device__ __forceinline__ bool poll_wait(unsigned& spin, int lane, unsigned long long deadline, const int* err) {
  if (++spin > 32) __nanosleep(spin > 256 ? 256 : 32);
  if ((spin & 255u) == 0) {
    int bad = 0;
    if (lane == 0) bad = gtimer() > deadline || ((spin & 4095u) == 0 && *(volatile const int*)err);
    if (__shfl_sync(0xffffffffu, bad, 0)) return false;
  }
  return true;
}

// read a unit: spin until all its lines carry `flag`.  Warp-collective.
template <int NS>
__device__ __forceinline__ bool get(const char* p, int lane, uint64_t flag, unsigned long long deadline,
                                    const int* err, LV<NS>* v) {
  unsigned spin = 0;
  for (;;) {
    uint64_t w[2 * NS];
    const uint64_t last = ld_share<NS>(p, w);
    if (unit_ready<NS>(lane, last, flag)) {
      *v = to_lv<NS>(w, flag_lane<NS>(lane));
      return true;
    }
    if (!poll_wait(spin, lane, deadline, err)) return false;
  }
}

// two units in one load round (scalar registers, no arrays indexed at run time): the copy
// stages and a two-operand fold hide one line latency behind the other
template <int NS>
__device__ __forceinline__ bool get2(const char* p0, const char* p1, int lane, uint64_t flag,
                                     unsigned long long deadline, const int* err, LV<NS>* v0, LV<NS>* v1) {
  bool need0 = true, need1 = true;
  uint64_t w0[2 * NS], w1[2 * NS];
#pragma unroll
  for (int i = 0; i < 2 * NS; ++i) w0[i] = w1[i] = 0;
  unsigned spin = 0;
  for (;;) {
    uint64_t l0 = w0[2 * NS - 1], l1 = w1[2 * NS - 1];
    if (need0) l0 = ld_share<NS>(p0, w0);
    if (need1) l1 = ld_share<NS>(p1, w1);
    if (need0 && unit_ready<NS>(lane, l0, flag)) need0 = false;
    if (need1 && unit_ready<NS>(lane, l1, flag)) need1 = false;
    if (!need0 && !need1) {
      *v0 = to_lv<NS>(w0, flag_lane<NS>(lane));
      *v1 = to_lv<NS>(w1, flag_lane<NS>(lane));
      return true;
    }
    if (!poll_wait(spin, lane, deadline, err)) return false;
  }
}

template <int DT, int W, bool MULTI, int NS>
__global__ void __launch_bounds__(Geo<NS>::kThreads, 1) torus_ll128_kernel(const L128Args a) {
  using Acc = typename Wire<W>::Acc;
  constexpr int VE = Wire<W>::VE;
  constexpr int UE = 30 * NS * VE;  // elements per unit
  using V = LV<NS>;

  const int lr = blockIdx.x / a.ctas;
  const int cta = blockIdx.x - lr * a.ctas;
  const RankDev* __restrict__ R = a.ranks + lr;
  const int X = R->X, Y = R->Y, N = R->N, rho = R->rho, c = R->c, me = R->rank;
  void* const buf = a.buf[lr];
  const bool aligned = a.aligned != 0;
  const int lane = threadIdx.x & 31;
  int wr = cta * Geo<NS>::kWarps + (threadIdx.x >> 5);  // warp index inside the rank
  int stage = 0;
  while (stage < kL128Stages - 1 && wr >= a.wk[stage]) wr -= a.wk[stage++];
  const int WS = a.wk[stage];

  __shared__ uint32_t s_epoch;
  if (threadIdx.x == 0) s_epoch = ld_acquire_gpu(R->pull_ctr);
  __syncthreads();
  const uint32_t epoch = s_epoch;
  const uint64_t flag = (uint64_t)epoch + 1u;
  const int par = (int)(epoch & 1u);
  const unsigned long long deadline = gtimer() + a.timeout_ns;
  int eoff[NS], cnt[NS];
#pragma unroll
  for (int h = 0; h < NS; ++h) lane_slice<VE, NS>(lane, h, &eoff[h], &cnt[h]);
  const uint4 zero = make_uint4(0, 0, 0, 0);
  // element count of slot h of this lane in unit u of a sub-chunk stream of length sl
  auto lane_n = [&](unsigned long long sl, unsigned long long u, int h) -> int {
    const long long r = (long long)sl - (long long)(u * UE + eoff[h]);
    return r <= 0 ? 0 : (r < cnt[h] ? (int)r : cnt[h]);
  };
  // my buffer at element e of the round: one flat buffer, or (MULTI, NEXT-1) the
  // concatenation of a bucket's tensors -- a separate instantiation, so the flat path
  // keeps its register budget.  (Flat: the whole-vector case is decided first and written
  // out here, so the ragged path's per-element arrays stay in their own cold branch.)
  const MultiSeg* const segs = MULTI ? a.segs + (size_t)lr * a.nseg : nullptr;
  int seg_hint = 0;
  auto uload1 = [&](unsigned long long e, int nrem) -> uint4 {
    if (nrem <= 0) return zero;
    if constexpr (MULTI) {
      return load_user_seg<DT, W>(segs, a.nseg, a.buf_off + e, nrem, seg_hint);
    } else {
      if (aligned && nrem == VE) {
        using T = typename Elem<DT>::T;
        const T* p = reinterpret_cast<const T*>(buf) + a.buf_off + e;
        if constexpr (DT == W) {
          return __ldcs(reinterpret_cast<const uint4*>(p));
        } else {
          const float4 x0 = __ldcs(reinterpret_cast<const float4*>(p));
          const float4 x1 = __ldcs(reinterpret_cast<const float4*>(p) + 1);
          const float f[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
          return pack<W>(f);
        }
      }
      return load_user<DT, W>(buf, a.buf_off + e, nrem, false);
    }
  };
  auto ustore1 = [&](unsigned long long e, int nrem, uint4 v) {
    if (nrem <= 0) return;
    if constexpr (MULTI) {
      store_user_seg<DT, W>(segs, a.nseg, a.buf_off + e, nrem, v, seg_hint);
    } else {
      if (aligned && nrem == VE) {
        using T = typename Elem<DT>::T;
        T* p = reinterpret_cast<T*>(buf) + a.buf_off + e;
        if constexpr (DT == W) {
          __stcs(reinterpret_cast<uint4*>(p), v);
        } else {
          float f[8];
          unpack<W>(v, f);
          __stcs(reinterpret_cast<float4*>(p), make_float4(f[0], f[1], f[2], f[3]));
          __stcs(reinterpret_cast<float4*>(p) + 1, make_float4(f[4], f[5], f[6], f[7]));
        }
        return;
      }
      store_user<DT, W>(buf, a.buf_off + e, nrem, v, false);
    }
  };
  // this lane's slots of unit u of the sub-chunk stream starting at element e0 (length sl)
  auto uload = [&](unsigned long long e0, unsigned long long sl, unsigned long long u) -> V {
    V v;
#pragma unroll
    for (int h = 0; h < NS; ++h) v.s[h] = uload1(e0 + u * UE + eoff[h], lane_n(sl, u, h));
    return v;
  };
  auto ustore = [&](unsigned long long e0, unsigned long long sl, unsigned long long u, const V& v) {
#pragma unroll
    for (int h = 0; h < NS; ++h) ustore1(e0 + u * UE + eoff[h], lane_n(sl, u, h), v.s[h]);
  };
  auto inbox = [&](int rank, unsigned long long off, unsigned long long stride, int slot) -> char* {
    return R->ws[rank] + off + (unsigned long long)slot * stride;
  };
  auto src = [&](char* stream, unsigned long long u) -> const char* { return lane_ptr<NS>(stream, u, lane); };
  // fold helpers over the slots (ring order is the caller's; f32 accumulation)
  auto fold_first = [&](Acc (&acc)[NS][VE], const V& w) {
#pragma unroll
    for (int h = 0; h < NS; ++h) unpack<W>(w.s[h], acc[h]);
  };
  auto fold_add = [&](Acc (&acc)[NS][VE], const V& w) {
#pragma unroll
    for (int h = 0; h < NS; ++h) {
      Acc t[VE];
      unpack<W>(w.s[h], t);
      acc_add<W>(acc[h], t);
    }
  };
  auto finish = [&](Acc (&acc)[NS][VE], bool mean) -> V {
    V out;
#pragma unroll
    for (int h = 0; h < NS; ++h) {
      if (mean) acc_mean<W>(acc[h], a.inv_n, N);
      out.s[h] = pack<W>(acc[h]);
    }
    return out;
  };
  // this call's inbox offsets, selected (not indexed: a parameter array indexed by a
  // runtime value is copied to local memory)
  const unsigned long long h_off = par ? a.h_off[1] : a.h_off[0], v_off = par ? a.v_off[1] : a.v_off[0],
                           ag_off = par ? a.ag_off[1] : a.ag_off[0], hag_off = par ? a.hag_off[1] : a.hag_off[0];
  bool ok = true;

  if (stage == kSA && X > 1) {
    // ---- A: my buffer's shares of my row peers' chunks -> their H inboxes ----
    const int per_u = (X - 1) * Y, nj = a.Umax * per_u;
    // job J -> (unit u, destination column j, sub-chunk js); both loads issued before
    // either store (named registers, not an array indexed by a running count: that
    // array would live in local memory)
    auto job = [&](int J, int& u, int& j, int& js) -> bool {
      if (J >= nj) return false;
      u = J / per_u;
      const int r = J % per_u;
      j = (c + 1 + r / Y) % X;
      js = j * Y + r % Y;
      return u < a.g_U[js];
    };
    auto load = [&](int u, int j, int js) -> V { return uload(a.g_co[j] + a.g_cs[js], a.g_sl[js], u); };
    auto push = [&](int u, int j, int js, const V& v) {
      put<NS>(inbox(rho * X + j, h_off, a.h_stride, c), (unsigned long long)a.g_uoff[js] + u, lane, v, flag);
    };
    for (int J0 = wr; J0 < nj; J0 += 2 * WS) {  // two units per iteration: both loads in flight
      int u0 = 0, j0 = 0, js0 = 0, u1 = 0, j1 = 0, js1 = 0;
      const bool h0 = job(J0, u0, j0, js0), h1 = job(J0 + WS, u1, j1, js1);
      V v0, v1;
      if (h0) v0 = load(u0, j0, js0);
      if (h1) v1 = load(u1, j1, js1);
      if (h0) push(u0, j0, js0, v0);
      if (h1) push(u1, j1, js1, v1);
    }
  } else if (stage == kSB) {
    // ---- B: fold my chunk (columns c+1, ..., c), round; push to the column owner ----
    for (int J = wr; J < a.Umax * Y && ok; J += WS) {
      const int u = J / Y, s = J % Y, cs = c * Y + s;
      if (u >= a.g_U[cs]) continue;
      const unsigned long long e0 = a.g_co[c] + a.g_cs[cs];
      const V own = uload(e0, a.g_sl[cs], u);  // issued first: its HBM latency overlaps the inbox polls
      Acc acc[NS][VE];
      for (int kk = 1; kk <= X && ok; ++kk) {
        const int j = (c + kk) % X;
        V w;
        if (j == c) w = own;
        else ok = get<NS>(src(inbox(me, h_off, a.h_stride, j), (unsigned long long)a.g_uoff[cs] + u), lane, flag,
                          deadline, R->err, &w);
        if (kk == 1) fold_first(acc, w);
        else fold_add(acc, w);
      }
      if (!ok) break;
      if (Y > 1) {
        put<NS>(inbox(s * X + c, v_off, a.v_stride, rho), u, lane, finish(acc, false), flag);
      } else {  // the last reduce phase: mean, round once, final
        const V out = finish(acc, a.op == 1);
        ustore(e0, a.g_sl[cs], u, out);
        for (int jj = 1; jj < X; ++jj)
          put<NS>(inbox(rho * X + (c + jj) % X, hag_off, a.hag_stride, c), (unsigned long long)a.g_uoff[cs] + u,
                  lane, out, flag);
      }
    }
  } else if (stage == kSC && Y > 1) {
    // ---- C: fold my sub-chunk (rows rho+1, ..., rho), mean, round; all-gather pushes ----
    const int cr = c * Y + rho;
    for (int u = wr; u < a.g_U[cr] && ok; u += WS) {
      Acc acc[NS][VE];
      if (Y == 2) {  // both rows in one load round: fold order rho+1, rho
        V w0, w1;
        ok = get2<NS>(src(inbox(me, v_off, a.v_stride, (rho + 1) % 2), u), src(inbox(me, v_off, a.v_stride, rho), u),
                      lane, flag, deadline, R->err, &w0, &w1);
        fold_first(acc, w0);
        fold_add(acc, w1);
      }
      for (int kk = 1; kk <= Y && ok && Y != 2; ++kk) {
        const int i = (rho + kk) % Y;
        V w;
        ok = get<NS>(src(inbox(me, v_off, a.v_stride, i), u), lane, flag, deadline, R->err, &w);
        if (kk == 1) fold_first(acc, w);
        else fold_add(acc, w);
      }
      if (!ok) break;
      const V out = finish(acc, a.op == 1);
      ustore(a.g_co[c] + a.g_cs[cr], a.g_sl[cr], u, out);
      for (int ii = 1; ii < Y; ++ii)
        put<NS>(inbox(((rho + ii) % Y) * X + c, ag_off, a.ag_stride, rho), u, lane, out, flag);
      for (int jj = 1; jj < X; ++jj)
        put<NS>(inbox(rho * X + (c + jj) % X, hag_off, a.hag_stride, c), (unsigned long long)a.g_uoff[cr] + u, lane,
                out, flag);
    }
  } else if (stage == kSD && Y > 1) {
    // ---- D: a column peer's reduced sub-chunk -> my buffer + the row peers' HAG inboxes ----
    const int nj = a.Umax * (Y - 1);
    auto job = [&](int J, int* u, int* ci) -> bool {
      if (J >= nj) return false;
      *u = J / (Y - 1);
      *ci = c * Y + (rho + 1 + J % (Y - 1)) % Y;
      return *u < a.g_U[*ci];
    };
    auto emit = [&](int u, int ci, const V& w) {
      ustore(a.g_co[c] + a.g_cs[ci], a.g_sl[ci], u, w);
      for (int jj = 1; jj < X; ++jj)
        put<NS>(inbox(rho * X + (c + jj) % X, hag_off, a.hag_stride, c), (unsigned long long)a.g_uoff[ci] + u, lane,
                w, flag);
    };
    for (int J = wr; J < nj && ok; J += 2 * WS) {  // two jobs per load round
      int u0, c0, u1, c1;
      const bool h0 = job(J, &u0, &c0), h1 = job(J + WS, &u1, &c1);
      V w0, w1;
      if (h0 && h1) {
        ok = get2<NS>(src(inbox(me, ag_off, a.ag_stride, c0 - c * Y), u0), src(inbox(me, ag_off, a.ag_stride, c1 - c * Y), u1),
                      lane, flag, deadline, R->err, &w0, &w1);
        if (!ok) break;
        emit(u0, c0, w0);
        emit(u1, c1, w1);
      } else if (h0 || h1) {
        const int u = h0 ? u0 : u1, ci = h0 ? c0 : c1;
        ok = get<NS>(src(inbox(me, ag_off, a.ag_stride, ci - c * Y), u), lane, flag, deadline, R->err, &w0);
        if (!ok) break;
        emit(u, ci, w0);
      }
    }
  } else if (stage == kSE && X > 1) {
    // ---- E: a row peer's completed chunk -> my buffer (wire -> dtype) ----
    const int per_u = (X - 1) * Y, nj = a.Umax * per_u;
    auto job = [&](int J, int* u, int* js) -> bool {
      if (J >= nj) return false;
      *u = J / per_u;
      const int r = J % per_u;
      *js = ((c + 1 + r / Y) % X) * Y + r % Y;
      return *u < a.g_U[*js];
    };
    auto at = [&](int u, int js) -> const char* {
      return src(inbox(me, hag_off, a.hag_stride, js / Y), (unsigned long long)a.g_uoff[js] + u);
    };
    auto emit = [&](int u, int js, const V& w) { ustore(a.g_co[js / Y] + a.g_cs[js], a.g_sl[js], u, w); };
    for (int J = wr; J < nj && ok; J += 2 * WS) {  // two jobs per load round
      int u0, j0, u1, j1;
      const bool h0 = job(J, &u0, &j0), h1 = job(J + WS, &u1, &j1);
      V w0, w1;
      if (h0 && h1) {
        ok = get2<NS>(at(u0, j0), at(u1, j1), lane, flag, deadline, R->err, &w0, &w1);
        if (!ok) break;
        emit(u0, j0, w0);
        emit(u1, j1, w1);
      } else if (h0 || h1) {
        const int u = h0 ? u0 : u1, js = h0 ? j0 : j1;
        ok = get<NS>(at(u, js), lane, flag, deadline, R->err, &w0);
        if (!ok) break;
        emit(u, js, w0);
      }
    }
  }
  if (!ok && lane == 0) atomicCAS_system(R->err, 0, kErrTimeout);
  __syncthreads();
  // the last CTA of this rank advances the call epoch (device-resident: graph capturable)
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t prev = atomicAdd(R->pull_ctr + 1, 1u);
    if (prev + 1 == (uint32_t)a.ctas) {
      R->pull_ctr[1] = 0;
      __threadfence();
      st_release_gpu(R->pull_ctr, epoch + 1u);
    }
  }
}

template <int DT, int W>
cudaError_t launch_ll128_typed(const L128Args& a, bool cooperative, cudaStream_t stream) {
  const dim3 grid(a.nlocal * a.ctas);
  // multi-tensor buckets and 16-byte lanes: NS = 1; flat calls with 32-byte lanes: NS = 2
  const bool wide = a.lane_bytes == 32 && a.nseg == 0;
  const void* fn = a.nseg > 0 ? (const void*)torus_ll128_kernel<DT, W, true, 1>
                              : wide ? (const void*)torus_ll128_kernel<DT, W, false, 2>
                                     : (const void*)torus_ll128_kernel<DT, W, false, 1>;
  const dim3 block(wide ? Geo<2>::kThreads : Geo<1>::kThreads);
  if (cooperative) {
    void* args[] = {const_cast<L128Args*>(&a)};
    return cudaLaunchCooperativeKernel(fn, grid, block, args, 0, stream);
  }
  void* args[] = {const_cast<L128Args*>(&a)};
  return cudaLaunchKernel(fn, grid, block, args, 0, stream);
}

}  // namespace

cudaError_t launch_ll128(const L128Args& a, int dtype, int wire, bool cooperative, cudaStream_t stream) {
  if (dtype == wire) {
    switch (dtype) {
      case DT_F32: return launch_ll128_typed<DT_F32, DT_F32>(a, cooperative, stream);
      case DT_F16: return launch_ll128_typed<DT_F16, DT_F16>(a, cooperative, stream);
      case DT_BF16: return launch_ll128_typed<DT_BF16, DT_BF16>(a, cooperative, stream);
      case DT_I32: return launch_ll128_typed<DT_I32, DT_I32>(a, cooperative, stream);
    }
  } else if (dtype == DT_F32 && wire == DT_F16) {
    return launch_ll128_typed<DT_F32, DT_F16>(a, cooperative, stream);
  } else if (dtype == DT_F32 && wire == DT_BF16) {
    return launch_ll128_typed<DT_F32, DT_BF16>(a, cooperative, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace torus
