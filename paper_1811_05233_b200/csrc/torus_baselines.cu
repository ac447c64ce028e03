// torus_baselines.cu -- the comparison paths of the 2D-Torus all-reduce:
// the flat ring (ref [14]) and the hierarchical all-reduce (ref [6]) the paper measures
// against, the NVLink / fence calibration probes, and the bucketed
// pack / unpack kernel of the multi-tensor API (NEXT-1).
#include <cstdio>
#include <cstdlib>

#include "torus_device.cuh"
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
    if (!ok) atomicCAS_system(R->err, 0, kErrTimeout);
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
  if (mode == 10 || mode == 11) {
    // store-injection probe: every thread pushes a register pattern to its peers with
    // 16-byte (10) or 32-byte (11) volatile stores -- no loads in the loop
    const unsigned long long a = 0x0123456789abcdefull ^ tid, bb = a * 3;
    for (int pp = 1; pp < N; ++pp) {
      const int p = (me + pp) % N;
      char* dst = R->ws[p] + data_off + (unsigned long long)me * per * 16;
      if (mode == 10) {
        for (unsigned long long v = (unsigned long long)b * blockDim.x + tid; v < per;
             v += (unsigned long long)G * blockDim.x)
          asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(dst + v * 16), "l"(a), "l"(bb) : "memory");
      } else {
        for (unsigned long long v = (unsigned long long)b * blockDim.x + tid; v < per / 2;
             v += (unsigned long long)G * blockDim.x)
          asm volatile("st.volatile.global.v4.u64 [%0], {%1, %2, %1, %2};" ::"l"(dst + v * 32), "l"(a), "l"(bb)
                       : "memory");
      }
    }
    return;
  }
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
    if (tid == 0 && !wait_flag_ge(flag(myws, kind, step), e, deadline, 64, R->err)) {
      atomicCAS_system(R->err, 0, kErrTimeout);
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
    if (tid == 0 && !wait_flag_ge(flag(myws, kind, step), e, deadline, 64, R->err)) {
      atomicCAS_system(R->err, 0, kErrTimeout);
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
