// torus_device.cuh -- device primitives shared by the product kernels (torus_kernels.cu,
// torus_pull.cu): memory-model operations, TMA bulk copies + mbarriers, the wire
// traits (f32 accumulation, RNE rounding to the wire type) and the user-buffer
// loads/stores with the dtype <-> wire cast fused.  Not part of the ABI.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "torus_internal.h"

namespace torus {
namespace {

enum { DT_F32 = 0, DT_F16 = 1, DT_BF16 = 2, DT_I32 = 3 };
enum { kErrTimeout = 6 };

// ------------------------------------------------------------------------------------
// memory-model primitives
// ------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_cta(int* p, int v) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  asm volatile("st.release.cta.shared.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
  int v;
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  asm volatile("ld.acquire.cta.shared.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Wait until *f >= v (wrap-safe).  Spin with relaxed loads and a short sleep -- a hot
// loop of ld.acquire.sys (each one an L1 invalidate) slows every fence on the SM -- and
// take the acquire once the value is there.  Returns false once `deadline` passes.
// An error already posted on the comm's async error word (a peer's MISMATCH or timeout)
// also ends the wait.
__device__ __forceinline__ bool wait_flag_ge(const uint32_t* f, uint32_t v, unsigned long long deadline,
                                             unsigned sleep_ns = 64, const int* err = nullptr) {
  unsigned spin = 0;
  while ((int32_t)(ld_relaxed_sys(f) - v) < 0) {
    if (sleep_ns) __nanosleep(sleep_ns);
    if ((++spin & 63u) == 0) {
      if (gtimer() > deadline) return false;
      if (err && (spin & 1023u) == 0 && *(volatile const int*)err) return false;  // host memory: rarely
    }
  }
  (void)ld_acquire_sys(f);
  return true;
}

// Workspace traffic goes through L2 only (.cg): slots are written by peers over NVLink
// during the kernel, so L1 must never hold a stale line.
__device__ __forceinline__ uint4 ld_ws(const void* p) { return __ldcg(reinterpret_cast<const uint4*>(p)); }
__device__ __forceinline__ void st_ws(void* p, uint4 v) { __stcg(reinterpret_cast<uint4*>(p), v); }


// ------------------------------------------------------------------------------------
// TMA bulk-copy primitives (cp.async.bulk, 1-D; sm_90+/sm_100a) and mbarriers
// ------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(phase)
      : "memory");
}
// global (local or NVLink peer) -> shared, completion counted on `bar`
__device__ __forceinline__ void tma_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// shared -> global (local or NVLink peer), tracked by bulk async-groups
__device__ __forceinline__ void tma_store(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void tma_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void tma_wait_all() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async;" ::: "memory");
}

// ------------------------------------------------------------------------------------
// wire traits: a 16-byte vector holds VE wire elements; Acc is the accumulation type
// (f32 for float wires, u32 two's-complement for i32)
// ------------------------------------------------------------------------------------
template <int W> struct Wire;
template <> struct Wire<DT_F32> { static constexpr int VE = 4; using Acc = float; };
template <> struct Wire<DT_I32> { static constexpr int VE = 4; using Acc = uint32_t; };
template <> struct Wire<DT_F16> { static constexpr int VE = 8; using Acc = float; };
template <> struct Wire<DT_BF16> { static constexpr int VE = 8; using Acc = float; };

template <int W>
__device__ __forceinline__ void unpack(const uint4 v, typename Wire<W>::Acc* a) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  if constexpr (W == DT_F32) {
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = __uint_as_float(w[i]);
  } else if constexpr (W == DT_I32) {
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = w[i];
  } else if constexpr (W == DT_F16) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __half2 h = *reinterpret_cast<const __half2*>(&w[i]);
      float2 f = __half22float2(h);  // exact
      a[2 * i] = f.x;
      a[2 * i + 1] = f.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // bf16 -> f32 is a shift (exact)
      a[2 * i] = __uint_as_float(w[i] << 16);
      a[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
}

// round to the wire type: IEEE round-to-nearest-even, no FTZ
template <int W>
__device__ __forceinline__ uint4 pack(const typename Wire<W>::Acc* a) {
  uint32_t w[4];
  if constexpr (W == DT_F32) {
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = __float_as_uint(a[i]);
  } else if constexpr (W == DT_I32) {
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = a[i];
  } else if constexpr (W == DT_F16) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __half2 h = __floats2half2_rn(a[2 * i], a[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(a[2 * i], a[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

template <int W>
__device__ __forceinline__ void acc_add(typename Wire<W>::Acc* a, const typename Wire<W>::Acc* b) {
#pragma unroll
  for (int i = 0; i < Wire<W>::VE; ++i) {
    if constexpr (W == DT_I32) a[i] = a[i] + b[i];  // wraps
    else a[i] = __fadd_rn(a[i], b[i]);               // no contraction, no FTZ
  }
}

// mean = f32 sum * f32(1/N), or (i32) wrapped sum / N truncated
template <int W>
__device__ __forceinline__ void acc_mean(typename Wire<W>::Acc* a, float inv_n, int N) {
#pragma unroll
  for (int i = 0; i < Wire<W>::VE; ++i) {
    if constexpr (W == DT_I32) a[i] = (uint32_t)((int32_t)a[i] / N);
    else a[i] = __fmul_rn(a[i], inv_n);
  }
}

// ------------------------------------------------------------------------------------
// user-buffer access with the dtype <-> wire cast fused
// ------------------------------------------------------------------------------------
template <int DT> struct Elem;
template <> struct Elem<DT_F32> { using T = float; };
template <> struct Elem<DT_I32> { using T = int32_t; };
template <> struct Elem<DT_F16> { using T = __half; };
template <> struct Elem<DT_BF16> { using T = __nv_bfloat16; };

// Load `nrem` (<= VE) elements at element index e of the user buffer, converted to the
// wire type (C1: w = to_wire(in)); missing lanes are zero.
template <int DT, int W>
__device__ __forceinline__ uint4 load_user(const void* buf, unsigned long long e, int nrem,
                                           bool aligned) {
  constexpr int VE = Wire<W>::VE;
  using T = typename Elem<DT>::T;
  const T* p = reinterpret_cast<const T*>(buf) + e;
  if constexpr (DT == W) {
    if (aligned && nrem == VE) return __ldcs(reinterpret_cast<const uint4*>(p));
    uint16_t h[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t u[4] = {0, 0, 0, 0};
    if constexpr (sizeof(T) == 2) {
      for (int i = 0; i < nrem; ++i) h[i] = reinterpret_cast<const uint16_t*>(p)[i];
      return make_uint4(h[0] | (uint32_t(h[1]) << 16), h[2] | (uint32_t(h[3]) << 16),
                        h[4] | (uint32_t(h[5]) << 16), h[6] | (uint32_t(h[7]) << 16));
    } else {
      for (int i = 0; i < nrem; ++i) u[i] = reinterpret_cast<const uint32_t*>(p)[i];
      return make_uint4(u[0], u[1], u[2], u[3]);
    }
  } else {
    static_assert(DT == DT_F32 && VE == 8, "only f32 buffers take a narrower wire");
    float f[8];
    if (aligned && nrem == 8) {
      const float4 a0 = __ldcs(reinterpret_cast<const float4*>(p));
      const float4 a1 = __ldcs(reinterpret_cast<const float4*>(p) + 1);
      f[0] = a0.x; f[1] = a0.y; f[2] = a0.z; f[3] = a0.w;
      f[4] = a1.x; f[5] = a1.y; f[6] = a1.z; f[7] = a1.w;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) f[i] = (i < nrem) ? p[i] : 0.0f;
    }
    return pack<W>(f);
  }
}

// Store `nrem` elements from a wire vector into the user buffer (from_wire, exact).
template <int DT, int W>
__device__ __forceinline__ void store_user(void* buf, unsigned long long e, int nrem, uint4 v,
                                           bool aligned) {
  constexpr int VE = Wire<W>::VE;
  using T = typename Elem<DT>::T;
  T* p = reinterpret_cast<T*>(buf) + e;
  if constexpr (DT == W) {
    if (aligned && nrem == VE) { __stcs(reinterpret_cast<uint4*>(p), v); return; }
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    if constexpr (sizeof(T) == 2) {
      for (int i = 0; i < nrem; ++i)
        reinterpret_cast<uint16_t*>(p)[i] = (uint16_t)(w[i >> 1] >> (16 * (i & 1)));
    } else {
      for (int i = 0; i < nrem; ++i) reinterpret_cast<uint32_t*>(p)[i] = w[i];
    }
  } else {
    float f[8];
    unpack<W>(v, f);
    if (aligned && nrem == 8) {
      __stcs(reinterpret_cast<float4*>(p), make_float4(f[0], f[1], f[2], f[3]));
      __stcs(reinterpret_cast<float4*>(p) + 1, make_float4(f[4], f[5], f[6], f[7]));
    } else {
      for (int i = 0; i < nrem; ++i) p[i] = f[i];
    }
  }
}

// ------------------------------------------------------------------------------------
// NEXT-1: the user buffer as a concatenation of tensors (fused multi-tensor call).  A 16-byte
// wire vector normally lies inside one tensor (ResNet-50's tensor sizes are multiples of 8);
// one that straddles a boundary is gathered / scattered element by element.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ int seg_find(const MultiSeg* seg, int nseg, unsigned long long e) {
  int lo = 0, hi = nseg - 1;  // last segment with offset <= e
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (seg[mid].offset <= e) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// boundary-straddling vectors: element by element, out of line (keeps the hot path lean)
template <int DT, int W>
__device__ __noinline__ uint4 load_user_straddle(const MultiSeg* seg, int nseg, int i, unsigned long long e,
                                                 int nrem) {
  using T = typename Elem<DT>::T;
  T tmp[8];
  for (int k = 0; k < nrem; ++k) {
    while (i + 1 < nseg && e + k >= seg[i + 1].offset) ++i;
    tmp[k] = reinterpret_cast<const T*>(seg[i].ptr)[e + k - seg[i].offset];
  }
  return load_user<DT, W>(tmp, 0, nrem, false);
}
template <int DT, int W>
__device__ __noinline__ void store_user_straddle(const MultiSeg* seg, int nseg, int i, unsigned long long e,
                                                 int nrem, uint4 v) {
  using T = typename Elem<DT>::T;
  T tmp[8];
  store_user<DT, W>(tmp, 0, nrem, v, false);
  for (int k = 0; k < nrem; ++k) {
    while (i + 1 < nseg && e + k >= seg[i + 1].offset) ++i;
    reinterpret_cast<T*>(seg[i].ptr)[e + k - seg[i].offset] = tmp[k];
  }
}

// the segment of element e, starting from the caller's last one (a thread walks its tiles in
// increasing order, so the hint is nearly always right; otherwise binary search)
__device__ __forceinline__ int seg_find_hint(const MultiSeg* seg, int nseg, unsigned long long e, int& hint) {
  int i = hint;
  const unsigned long long o = seg[i].offset;
  if (e >= o && e < o + seg[i].count) return i;
  if (e >= o && i + 1 < nseg && e >= seg[i + 1].offset &&
      (i + 2 >= nseg || e < seg[i + 2].offset)) {
    hint = i + 1;
    return hint;
  }
  hint = seg_find(seg, nseg, e);
  return hint;
}

template <int DT, int W>
__device__ __forceinline__ uint4 load_user_seg(const MultiSeg* seg, int nseg, unsigned long long e, int nrem,
                                               int& hint) {
  using T = typename Elem<DT>::T;
  const int i = seg_find_hint(seg, nseg, e, hint);
  const unsigned long long local = e - seg[i].offset;
  if (local + nrem > seg[i].count) return load_user_straddle<DT, W>(seg, nseg, i, e, nrem);
  const T* p = reinterpret_cast<const T*>(seg[i].ptr) + local;
  return load_user<DT, W>(p, 0, nrem, (reinterpret_cast<uintptr_t>(p) & 15) == 0);
}

template <int DT, int W>
__device__ __forceinline__ void store_user_seg(const MultiSeg* seg, int nseg, unsigned long long e, int nrem,
                                               uint4 v, int& hint) {
  using T = typename Elem<DT>::T;
  const int i = seg_find_hint(seg, nseg, e, hint);
  const unsigned long long local = e - seg[i].offset;
  if (local + nrem > seg[i].count) {
    store_user_straddle<DT, W>(seg, nseg, i, e, nrem, v);
    return;
  }
  T* p = reinterpret_cast<T*>(seg[i].ptr) + local;
  store_user<DT, W>(p, 0, nrem, v, (reinterpret_cast<uintptr_t>(p) & 15) == 0);
}

}  // namespace
}  // namespace torus
