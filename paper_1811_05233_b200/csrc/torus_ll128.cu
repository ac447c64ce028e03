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
constexpr int kL128Threads = TORUS_LL128_THREADS;
constexpr int kL128Warps = kL128Threads / 32;
enum { kSA = 0, kSB = 1, kSC = 2, kSD = 3, kSE = 4, kL128Stages = 5 };

__device__ __forceinline__ void st_line(char* p, uint64_t lo, uint64_t hi) {
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(lo), "l"(hi) : "memory");
}
__device__ __forceinline__ void ld_line(const char* p, uint64_t& lo, uint64_t& hi) {
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(p) : "memory");
}

// this lane's slice of a unit: element offset inside the unit and element count
template <int VE>
__device__ __forceinline__ void lane_slice(int lane, int* eoff, int* cnt) {
  const int g = lane >> 3, li = lane & 7;
  if (li < 7) {
    *eoff = (g * 7 + li) * VE;
    *cnt = VE;
  } else {
    *eoff = (28 + (g >> 1)) * VE + (g & 1) * (VE / 2);
    *cnt = VE / 2;
  }
}

__device__ __forceinline__ char* lane_ptr(char* stream, unsigned long long u, int lane) {
  return stream + u * kL128Unit + (lane >> 3) * kL128Line + (lane & 7) * 16;
}

// write this lane's share of a unit (the flag lane: 8 data bytes + the flag)
__device__ __forceinline__ void put(char* stream, unsigned long long u, int lane, uint4 v, uint64_t flag) {
  const uint64_t lo = (uint64_t)v.x | ((uint64_t)v.y << 32);
  const uint64_t hi = ((lane & 7) == 7) ? flag : ((uint64_t)v.z | ((uint64_t)v.w << 32));
  st_line(lane_ptr(stream, u, lane), lo, hi);
}

// read a unit: spin until all four lines carry `flag`.  Warp-collective.
__device__ __forceinline__ bool get(const char* stream, unsigned long long u, int lane, uint64_t flag,
                                    unsigned long long deadline, const int* err, uint4* v) {
  const char* p = lane_ptr(const_cast<char*>(stream), u, lane);
  unsigned spin = 0;
  for (;;) {
    uint64_t lo, hi;
    ld_line(p, lo, hi);
    const int mine = ((lane & 7) != 7) || (hi == flag);
    const int line_ok = __shfl_sync(0xffffffffu, mine, (lane & ~7) | 7);
    if (__all_sync(0xffffffffu, line_ok)) {
      const bool fl = (lane & 7) == 7;
      *v = make_uint4((uint32_t)lo, (uint32_t)(lo >> 32), fl ? 0u : (uint32_t)hi, fl ? 0u : (uint32_t)(hi >> 32));
      return true;
    }
    // back off once the lines are clearly not there yet: thousands of warps re-reading
    // the same L2 lines at full speed slow the NVLink writes that must land in them
    if (++spin > 32) __nanosleep(spin > 256 ? 256 : 32);
    if ((spin & 255u) == 0) {
      int bad = 0;
      if (lane == 0) bad = gtimer() > deadline || ((spin & 4095u) == 0 && *(volatile const int*)err);
      if (__shfl_sync(0xffffffffu, bad, 0)) return false;
    }
  }
}

// two units in one load round (scalar registers, no arrays): the copy stages and a
// two-operand fold hide one line latency behind the other
__device__ __forceinline__ bool get2(const char* p0, const char* p1, int lane, uint64_t flag,
                                     unsigned long long deadline, const int* err, uint4* v0, uint4* v1) {
  const bool fl = (lane & 7) == 7;
  bool need0 = true, need1 = true;
  uint64_t lo0 = 0, hi0 = 0, lo1 = 0, hi1 = 0;
  unsigned spin = 0;
  for (;;) {
    if (need0) ld_line(p0, lo0, hi0);
    if (need1) ld_line(p1, lo1, hi1);
    if (need0) {
      const int ok = __shfl_sync(0xffffffffu, (int)(!fl || hi0 == flag), (lane & ~7) | 7);
      if (__all_sync(0xffffffffu, ok)) need0 = false;
    }
    if (need1) {
      const int ok = __shfl_sync(0xffffffffu, (int)(!fl || hi1 == flag), (lane & ~7) | 7);
      if (__all_sync(0xffffffffu, ok)) need1 = false;
    }
    if (!need0 && !need1) {
      *v0 = make_uint4((uint32_t)lo0, (uint32_t)(lo0 >> 32), fl ? 0u : (uint32_t)hi0, fl ? 0u : (uint32_t)(hi0 >> 32));
      *v1 = make_uint4((uint32_t)lo1, (uint32_t)(lo1 >> 32), fl ? 0u : (uint32_t)hi1, fl ? 0u : (uint32_t)(hi1 >> 32));
      return true;
    }
    // back off once the lines are clearly not there yet: thousands of warps re-reading
    // the same L2 lines at full speed slow the NVLink writes that must land in them
    if (++spin > 32) __nanosleep(spin > 256 ? 256 : 32);
    if ((spin & 255u) == 0) {
      int bad = 0;
      if (lane == 0) bad = gtimer() > deadline || ((spin & 4095u) == 0 && *(volatile const int*)err);
      if (__shfl_sync(0xffffffffu, bad, 0)) return false;
    }
  }
}

template <int DT, int W, bool MULTI>
__global__ void __launch_bounds__(kL128Threads, 1) torus_ll128_kernel(const L128Args a) {
  using Acc = typename Wire<W>::Acc;
  constexpr int VE = Wire<W>::VE;
  constexpr int UE = 30 * VE;  // elements per unit

  const int lr = blockIdx.x / a.ctas;
  const int cta = blockIdx.x - lr * a.ctas;
  const RankDev* __restrict__ R = a.ranks + lr;
  const int X = R->X, Y = R->Y, N = R->N, rho = R->rho, c = R->c, me = R->rank;
  void* const buf = a.buf[lr];
  const bool aligned = a.aligned != 0;
  const int lane = threadIdx.x & 31;
  int wr = cta * kL128Warps + (threadIdx.x >> 5);  // warp index inside the rank
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
  char* const myws = R->ws[me];
  int eoff, cnt;
  lane_slice<VE>(lane, &eoff, &cnt);
  const uint4 zero = make_uint4(0, 0, 0, 0);
  // element count of this lane in unit u of a sub-chunk stream of length sl
  auto lane_n = [&](unsigned long long sl, unsigned long long u) -> int {
    const long long r = (long long)sl - (long long)(u * UE + eoff);
    return r <= 0 ? 0 : (r < cnt ? (int)r : cnt);
  };
  // my buffer at element e of the round: one flat buffer, or (MULTI, NEXT-1) the
  // concatenation of a bucket's tensors -- a separate instantiation, so the flat path
  // keeps its register budget
  const MultiSeg* const segs = MULTI ? a.segs + (size_t)lr * a.nseg : nullptr;
  int seg_hint = 0;
  // (flat: the whole-vector case is decided first and written out here, so the ragged
  // path's per-element arrays stay in its own cold branch instead of local memory on
  // every call)
  auto uload = [&](unsigned long long e, int nrem) -> uint4 {
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
  auto ustore = [&](unsigned long long e, int nrem, uint4 v) {
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
  auto inbox = [&](int rank, unsigned long long off, unsigned long long stride, int slot) -> char* {
    return R->ws[rank] + off + (unsigned long long)slot * stride;
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
    auto load = [&](int u, int j, int js) -> uint4 {
      return uload(a.g_co[j] + a.g_cs[js] + (unsigned long long)u * UE + eoff, lane_n(a.g_sl[js], u));
    };
    auto push = [&](int u, int j, int js, uint4 v) {
      put(inbox(rho * X + j, h_off, a.h_stride, c), (unsigned long long)a.g_uoff[js] + u, lane, v, flag);
    };
    for (int J0 = wr; J0 < nj; J0 += 2 * WS) {  // two units per iteration: both loads in flight
      int u0 = 0, j0 = 0, js0 = 0, u1 = 0, j1 = 0, js1 = 0;
      const bool h0 = job(J0, u0, j0, js0), h1 = job(J0 + WS, u1, j1, js1);
      const uint4 v0 = h0 ? load(u0, j0, js0) : zero;
      const uint4 v1 = h1 ? load(u1, j1, js1) : zero;
      if (h0) push(u0, j0, js0, v0);
      if (h1) push(u1, j1, js1, v1);
    }
  } else if (stage == kSB) {
    // ---- B: fold my chunk (columns c+1, ..., c), round; push to the column owner ----
    for (int J = wr; J < a.Umax * Y && ok; J += WS) {
      const int u = J / Y, s = J % Y, cs = c * Y + s;
      if (u >= a.g_U[cs]) continue;
      const int nr = lane_n(a.g_sl[cs], u);
      const unsigned long long e = a.g_co[c] + a.g_cs[cs] + (unsigned long long)u * UE + eoff;
      const uint4 own = uload(e, nr);  // issued first: its HBM latency overlaps the inbox polls
      Acc acc[VE];
      for (int kk = 1; kk <= X && ok; ++kk) {
        const int j = (c + kk) % X;
        uint4 w;
        if (j == c) w = own;
        else ok = get(inbox(me, h_off, a.h_stride, j), (unsigned long long)a.g_uoff[cs] + u, lane, flag,
                      deadline, R->err, &w);
        Acc t[VE];
        unpack<W>(w, t);
        if (kk == 1) {
#pragma unroll
          for (int i = 0; i < VE; ++i) acc[i] = t[i];
        } else {
          acc_add<W>(acc, t);
        }
      }
      if (!ok) break;
      if (Y > 1) {
        put(inbox(s * X + c, v_off, a.v_stride, rho), u, lane, pack<W>(acc), flag);
      } else {  // the last reduce phase: mean, round once, final
        if (a.op == 1) acc_mean<W>(acc, a.inv_n, N);
        const uint4 out = pack<W>(acc);
        ustore(e, nr, out);
        for (int jj = 1; jj < X; ++jj)
          put(inbox(rho * X + (c + jj) % X, hag_off, a.hag_stride, c), (unsigned long long)a.g_uoff[cs] + u,
              lane, out, flag);
      }
    }
  } else if (stage == kSC && Y > 1) {
    // ---- C: fold my sub-chunk (rows rho+1, ..., rho), mean, round; all-gather pushes ----
    const int cr = c * Y + rho;
    for (int u = wr; u < a.g_U[cr] && ok; u += WS) {
      const int nr = lane_n(a.g_sl[cr], u);
      Acc acc[VE];
      if (Y == 2) {  // both rows in one load round: fold order rho+1, rho
        uint4 w0, w1;
        ok = get2(lane_ptr(inbox(me, v_off, a.v_stride, (rho + 1) % 2), u, lane),
                  lane_ptr(inbox(me, v_off, a.v_stride, rho), u, lane), lane, flag, deadline, R->err, &w0,
                  &w1);
        Acc t[VE];
        unpack<W>(w0, acc);
        unpack<W>(w1, t);
        acc_add<W>(acc, t);
      }
      for (int kk = 1; kk <= Y && ok && Y != 2; ++kk) {
        const int i = (rho + kk) % Y;
        uint4 w;
        ok = get(inbox(me, v_off, a.v_stride, i), u, lane, flag, deadline, R->err, &w);
        Acc t[VE];
        unpack<W>(w, t);
        if (kk == 1) {
#pragma unroll
          for (int q = 0; q < VE; ++q) acc[q] = t[q];
        } else {
          acc_add<W>(acc, t);
        }
      }
      if (!ok) break;
      if (a.op == 1) acc_mean<W>(acc, a.inv_n, N);
      const uint4 out = pack<W>(acc);
      ustore(a.g_co[c] + a.g_cs[cr] + (unsigned long long)u * UE + eoff, nr, out);
      for (int ii = 1; ii < Y; ++ii)
        put(inbox(((rho + ii) % Y) * X + c, ag_off, a.ag_stride, rho), u, lane, out, flag);
      for (int jj = 1; jj < X; ++jj)
        put(inbox(rho * X + (c + jj) % X, hag_off, a.hag_stride, c), (unsigned long long)a.g_uoff[cr] + u,
            lane, out, flag);
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
    auto emit = [&](int u, int ci, uint4 w) {
      ustore(a.g_co[c] + a.g_cs[ci] + (unsigned long long)u * UE + eoff, lane_n(a.g_sl[ci], u), w);
      for (int jj = 1; jj < X; ++jj)
        put(inbox(rho * X + (c + jj) % X, hag_off, a.hag_stride, c), (unsigned long long)a.g_uoff[ci] + u,
            lane, w, flag);
    };
    for (int J = wr; J < nj && ok; J += 2 * WS) {  // two jobs per load round
      int u0, c0, u1, c1;
      const bool h0 = job(J, &u0, &c0), h1 = job(J + WS, &u1, &c1);
      uint4 w0, w1;
      if (h0 && h1) {
        ok = get2(lane_ptr(inbox(me, ag_off, a.ag_stride, c0 - c * Y), u0, lane),
                  lane_ptr(inbox(me, ag_off, a.ag_stride, c1 - c * Y), u1, lane), lane, flag, deadline,
                  R->err, &w0, &w1);
        if (!ok) break;
        emit(u0, c0, w0);
        emit(u1, c1, w1);
      } else if (h0 || h1) {
        const int u = h0 ? u0 : u1, ci = h0 ? c0 : c1;
        ok = get(inbox(me, ag_off, a.ag_stride, ci - c * Y), u, lane, flag, deadline, R->err, &w0);
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
    auto src = [&](int u, int js) -> const char* {
      return lane_ptr(inbox(me, hag_off, a.hag_stride, js / Y), (unsigned long long)a.g_uoff[js] + u, lane);
    };
    auto emit = [&](int u, int js, uint4 w) {
      ustore(a.g_co[js / Y] + a.g_cs[js] + (unsigned long long)u * UE + eoff, lane_n(a.g_sl[js], u), w);
    };
    for (int J = wr; J < nj && ok; J += 2 * WS) {  // two jobs per load round
      int u0, j0, u1, j1;
      const bool h0 = job(J, &u0, &j0), h1 = job(J + WS, &u1, &j1);
      uint4 w0, w1;
      if (h0 && h1) {
        ok = get2(src(u0, j0), src(u1, j1), lane, flag, deadline, R->err, &w0, &w1);
        if (!ok) break;
        emit(u0, j0, w0);
        emit(u1, j1, w1);
      } else if (h0 || h1) {
        const int u = h0 ? u0 : u1, js = h0 ? j0 : j1;
        ok = get(inbox(me, hag_off, a.hag_stride, js / Y), (unsigned long long)a.g_uoff[js] + u, lane, flag,
                 deadline, R->err, &w0);
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
  const dim3 grid(a.nlocal * a.ctas), block(kL128Threads);
  const void* fn = a.nseg > 0 ? (const void*)torus_ll128_kernel<DT, W, true>
                              : (const void*)torus_ll128_kernel<DT, W, false>;
  if (cooperative) {
    void* args[] = {const_cast<L128Args*>(&a)};
    return cudaLaunchCooperativeKernel(fn, grid, block, args, 0, stream);
  }
  if (a.nseg > 0) torus_ll128_kernel<DT, W, true><<<grid, block, 0, stream>>>(a);
  else torus_ll128_kernel<DT, W, false><<<grid, block, 0, stream>>>(a);
  return cudaGetLastError();
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
