// torus_ll.cu -- small- and mid-message kernels (NEXT-2): one-shot and two-shot "LL"
// paths whose flag lives in every 8-byte word, bit-identical to the multi-phase torus.
#include <cstdio>
#include <cstdlib>

#include "torus_device.cuh"
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
                                      uint32_t* d0, uint32_t* d1, const int* err) {
  unsigned spin = 0;
  for (;;) {
    unsigned long long a, b;
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
    if ((uint32_t)(a >> 32) == flag && (uint32_t)(b >> 32) == flag) {
      *d0 = (uint32_t)a;
      *d1 = (uint32_t)b;
      return true;
    }
    if ((++spin & 255u) == 0) {
      if (gtimer() > deadline) return false;
      // the error word is host memory: look at it rarely (every 4096 spins)
      if ((spin & 4095u) == 0 && *(volatile const int*)err) return false;
    }
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
          ok = ld_ll(src + j * 16, flag, deadline, &w.x, &w.y, R->err) &&
               ld_ll(src + half + j * 16, flag, deadline, &w.z, &w.w, R->err);
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
  if (!ok) atomicCAS_system(R->err, 0, kErrTimeout);

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
          ok = ld_ll(src + v * 16, flag, deadline, &w.x, &w.y, R->err) &&
               ld_ll(src + half + v * 16, flag, deadline, &w.z, &w.w, R->err);
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
    ok = ld_ll(src + v * 16, flag, deadline, &w.x, &w.y, R->err) &&
         ld_ll(src + half + v * 16, flag, deadline, &w.z, &w.w, R->err);
    if (!ok) break;
    const int nrem = (int)(n - e < (unsigned long long)VE ? n - e : VE);
    store_user<DT, W>(buf, a.buf_off + e, nrem, w, a.aligned);
  }
  if (!ok) atomicCAS_system(R->err, 0, kErrTimeout);
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

