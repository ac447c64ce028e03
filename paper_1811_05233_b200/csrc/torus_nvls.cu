// torus_nvls.cu -- NVLink-SHARP (NVLS) variant, NEXT-4.
//
// The copy-based torus moves 2(N-1)/N * S bytes per GPU per direction over NVLink.  With
// in-switch reduction a GPU reads its 1/N shard already summed over all N GPUs by the
// NVSwitch (multimem.ld_reduce on a multicast address) and writes the result back to every
// GPU with one multicast store (multimem.st): per GPU about S + S/N out and S/N + S in.
// The switch's summation order is unspecified, so this variant matches the oracle within
// the float tolerance only (not bit for bit) and is an opt-in alternative to the torus
// (PAPER.md:70 defines the torus; the paper has no in-switch reduction).
//
// Per call (CTA b owns slice b of every rank's shard, in every phase):
//   1. copy my buffer's slice into my multicast-bound staging (dtype -> wire cast)
//   2. per-CTA barrier with every peer (st.release.sys / ld.acquire.sys flags)
//   3. multimem.ld_reduce my shard's slice (f32 accumulation in the switch), mean,
//      multimem.st it to every GPU's staging
//   4. per-CTA barrier
//   5. copy every shard's slice from staging to my buffer (wire -> dtype)
// Setup (collective, three steps around two host exchanges): rank 0 creates the
// multicast object and exports it as a POSIX fd; the other ranks duplicate that fd with
// pidfd_getfd, every rank adds its device, then binds its physical staging memory and
// maps the multicast address.  Driver calls go through cudaGetDriverEntryPoint, so the
// library does not link libcuda.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cstring>

#include "torus_internal.h"

namespace torus {
namespace {

// ---------------- driver entry points ----------------
struct Drv {
  CUresult (*memCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
  CUresult (*memGetAllocationGranularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags);
  CUresult (*multicastGetGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags);
  CUresult (*multicastCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*);
  CUresult (*memExportToShareableHandle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long);
  CUresult (*memImportFromShareableHandle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType);
  CUresult (*multicastAddDevice)(CUmemGenericAllocationHandle, CUdevice);
  CUresult (*multicastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t, unsigned long long);
  CUresult (*multicastUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t);
  CUresult (*memAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
  CUresult (*memAddressFree)(CUdeviceptr, size_t);
  CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
  CUresult (*memUnmap)(CUdeviceptr, size_t);
  CUresult (*memSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
  CUresult (*memRelease)(CUmemGenericAllocationHandle);
  CUresult (*deviceGet)(CUdevice*, int);
  bool ok = false;
};

bool load_drv(Drv* d) {
  if (d->ok) return true;
  auto get = [](const char* name, void** fn) {
    cudaDriverEntryPointQueryResult q;
    return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
           q == cudaDriverEntryPointSuccess && *fn != nullptr;
  };
  bool ok = true;
  ok &= get("cuMemCreate", reinterpret_cast<void**>(&d->memCreate));
  ok &= get("cuMemGetAllocationGranularity", reinterpret_cast<void**>(&d->memGetAllocationGranularity));
  ok &= get("cuMulticastGetGranularity", reinterpret_cast<void**>(&d->multicastGetGranularity));
  ok &= get("cuMulticastCreate", reinterpret_cast<void**>(&d->multicastCreate));
  ok &= get("cuMemExportToShareableHandle", reinterpret_cast<void**>(&d->memExportToShareableHandle));
  ok &= get("cuMemImportFromShareableHandle", reinterpret_cast<void**>(&d->memImportFromShareableHandle));
  ok &= get("cuMulticastAddDevice", reinterpret_cast<void**>(&d->multicastAddDevice));
  ok &= get("cuMulticastBindMem", reinterpret_cast<void**>(&d->multicastBindMem));
  ok &= get("cuMulticastUnbind", reinterpret_cast<void**>(&d->multicastUnbind));
  ok &= get("cuMemAddressReserve", reinterpret_cast<void**>(&d->memAddressReserve));
  ok &= get("cuMemAddressFree", reinterpret_cast<void**>(&d->memAddressFree));
  ok &= get("cuMemMap", reinterpret_cast<void**>(&d->memMap));
  ok &= get("cuMemUnmap", reinterpret_cast<void**>(&d->memUnmap));
  ok &= get("cuMemSetAccess", reinterpret_cast<void**>(&d->memSetAccess));
  ok &= get("cuMemRelease", reinterpret_cast<void**>(&d->memRelease));
  ok &= get("cuDeviceGet", reinterpret_cast<void**>(&d->deviceGet));
  d->ok = ok;
  return ok;
}

Drv g_drv;

// ---------------- device side ----------------
__device__ __forceinline__ uint32_t ld_acquire_sys32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_sys32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// 16-byte in-switch reduce / multicast store per wire type
template <int W> struct Mm;
template <> struct Mm<1> {  // f16: f32 accumulation in the switch
  __device__ static uint4 ld_reduce(const void* mc) {
    uint4 r;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.f16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(mc) : "memory");
    return r;
  }
  __device__ static void scale(uint4& v, float s) {
    uint32_t* w = &v.x;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __half2 h = *reinterpret_cast<__half2*>(&w[i]);
      float2 f = __half22float2(h);
      h = __floats2half2_rn(f.x * s, f.y * s);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
  }
  __device__ static void st(void* mc, uint4 v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f16x2 [%0], {%1,%2,%3,%4};" ::"l"(mc), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
  }
};
template <> struct Mm<2> {  // bf16
  __device__ static uint4 ld_reduce(const void* mc) {
    uint4 r;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(mc) : "memory");
    return r;
  }
  __device__ static void scale(uint4& v, float s) {
    uint32_t* w = &v.x;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float lo = __uint_as_float(w[i] << 16) * s, hi = __uint_as_float(w[i] & 0xffff0000u) * s;
      __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
  }
  __device__ static void st(void* mc, uint4 v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.bf16x2 [%0], {%1,%2,%3,%4};" ::"l"(mc), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
  }
};
template <> struct Mm<0> {  // f32
  __device__ static uint4 ld_reduce(const void* mc) {
    uint4 r;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(mc) : "memory");
    return r;
  }
  __device__ static void scale(uint4& v, float s) {
    v.x = __float_as_uint(__uint_as_float(v.x) * s);
    v.y = __float_as_uint(__uint_as_float(v.y) * s);
    v.z = __float_as_uint(__uint_as_float(v.z) * s);
    v.w = __float_as_uint(__uint_as_float(v.w) * s);
  }
  __device__ static void st(void* mc, uint4 v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
  }
};

template <int DT> struct NElem;
template <> struct NElem<0> { using T = float; };
template <> struct NElem<1> { using T = __half; };
template <> struct NElem<2> { using T = __nv_bfloat16; };

struct NvlsArgs {
  const RankDev* ranks;
  void* buf;
  char* uc;                      // my staging (unicast view)
  char* mc;                      // multicast view of everyone's staging
  unsigned long long n, buf_off;
  unsigned long long timeout_ns;
  int G, q, op;
  float inv_n;
};

// wire element of user element i (cast on the first read / last write)
template <int DT, int W>
__device__ __forceinline__ void to_wire(const void* buf, unsigned long long i, void* dst) {
  using UT = typename NElem<DT>::T;
  const UT x = reinterpret_cast<const UT*>(buf)[i];
  if constexpr (DT == W) *reinterpret_cast<UT*>(dst) = x;
  else if constexpr (W == 1) *reinterpret_cast<__half*>(dst) = __float2half_rn((float)x);
  else *reinterpret_cast<__nv_bfloat16*>(dst) = __float2bfloat16_rn((float)x);
}
template <int DT, int W>
__device__ __forceinline__ void from_wire(void* buf, unsigned long long i, const void* src) {
  using UT = typename NElem<DT>::T;
  using WT = typename NElem<W>::T;
  const WT w = *reinterpret_cast<const WT*>(src);
  if constexpr (DT == W) reinterpret_cast<UT*>(buf)[i] = w;
  else reinterpret_cast<UT*>(buf)[i] = (float)w;
}

template <int DT, int W>
__global__ void __launch_bounds__(512, 1) nvls_kernel(const NvlsArgs a) {
  constexpr int SW = (W == 0) ? 4 : 2;
  constexpr int VE = 16 / SW;
  const RankDev* R = a.ranks;
  const int N = R->N, me = R->rank, b = blockIdx.x, G = a.G, tid = threadIdx.x;
  __shared__ uint32_t s_e;
  __shared__ int s_abort;
  if (tid == 0) {
    s_e = R->epoch[b] + 1u;
    s_abort = 0;
  }
  __syncthreads();
  const uint32_t e = s_e;
  const unsigned long long deadline = gtime() + a.timeout_ns;
  auto flag = [&](char* ws, int kind, int src) -> uint32_t* {
    return reinterpret_cast<uint32_t*>(ws) + ((size_t)(kind * kMaxDim + src) * G + b);
  };
  auto barrier = [&](int kind) -> bool {  // CTA b of every rank
    __syncthreads();
    if (tid < N && tid != me) {
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      uint32_t* f = flag(R->ws[tid], kind, me);
      asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(f), "r"(e) : "memory");
    }
    if (tid < N && tid != me) {
      const uint32_t* f = flag(R->ws[me], kind, tid);
      unsigned spin = 0;
      while ((int32_t)(ld_relaxed_sys32(f) - e) < 0) {
        __nanosleep(64);
        if ((++spin & 63u) == 0 && gtime() > deadline) {
          atomicCAS_system(R->err, 0, 6);
          s_abort = 1;
          break;
        }
      }
      (void)ld_acquire_sys32(f);
    }
    __syncthreads();
    return s_abort == 0;
  };
  // CTA b's slice [v0, v1) (vectors) of shard k
  auto shard_slice = [&](int k, unsigned long long* off, unsigned long long* len,
                         unsigned long long* v0, unsigned long long* v1) {
    qpart(a.n, N, a.q, k, off, len);
    const unsigned long long nv = (*len + VE - 1) / VE;
    *v0 = nv * (unsigned long long)b / G;
    *v1 = nv * (unsigned long long)(b + 1) / G;
  };
  // 16-byte vector path when the user buffer (at this round's offset) is 16-byte aligned
  using UT = typename NElem<DT>::T;
  constexpr int UB = (int)sizeof(UT) * VE;  // user bytes per wire vector (16 or 32)
  const bool vec = ((reinterpret_cast<uintptr_t>(a.buf) + a.buf_off * sizeof(UT)) & 15) == 0;
  auto copy_in = [&](unsigned long long i0, unsigned long long i1) {  // elements [i0, i1)
    unsigned long long i = i0;
    if (vec) {
      for (unsigned long long v = i0 / VE + tid; (v + 1) * VE <= i1; v += blockDim.x) {
        const char* src = reinterpret_cast<const char*>(a.buf) + (a.buf_off + v * VE) * sizeof(UT);
        uint4 w;
        if constexpr (DT == W) {
          w = __ldcs(reinterpret_cast<const uint4*>(src));
        } else {
          const float4 f0 = __ldcs(reinterpret_cast<const float4*>(src));
          const float4 f1 = __ldcs(reinterpret_cast<const float4*>(src) + 1);
          const float f[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
          uint32_t* o = &w.x;
#pragma unroll
          for (int k2 = 0; k2 < 4; ++k2) {
            if constexpr (W == 1) {
              __half2 h = __floats2half2_rn(f[2 * k2], f[2 * k2 + 1]);
              o[k2] = *reinterpret_cast<uint32_t*>(&h);
            } else {
              __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * k2], f[2 * k2 + 1]);
              o[k2] = *reinterpret_cast<uint32_t*>(&h);
            }
          }
        }
        *reinterpret_cast<uint4*>(a.uc + v * VE * SW) = w;
      }
      i = i0 + (i1 - i0) / VE * VE;
    }
    for (unsigned long long j = i + tid; j < i1; j += blockDim.x) to_wire<DT, W>(a.buf, a.buf_off + j, a.uc + j * SW);
  };
  auto copy_out = [&](unsigned long long i0, unsigned long long i1) {
    unsigned long long i = i0;
    if (vec) {
      for (unsigned long long v = i0 / VE + tid; (v + 1) * VE <= i1; v += blockDim.x) {
        const uint4 w = *reinterpret_cast<const uint4*>(a.uc + v * VE * SW);
        char* dst = reinterpret_cast<char*>(a.buf) + (a.buf_off + v * VE) * sizeof(UT);
        if constexpr (DT == W) {
          __stcs(reinterpret_cast<uint4*>(dst), w);
        } else {
          const uint32_t* o = &w.x;
          float f[8];
#pragma unroll
          for (int k2 = 0; k2 < 4; ++k2) {
            if constexpr (W == 1) {
              const float2 t = __half22float2(*reinterpret_cast<const __half2*>(&o[k2]));
              f[2 * k2] = t.x;
              f[2 * k2 + 1] = t.y;
            } else {
              f[2 * k2] = __uint_as_float(o[k2] << 16);
              f[2 * k2 + 1] = __uint_as_float(o[k2] & 0xffff0000u);
            }
          }
          __stcs(reinterpret_cast<float4*>(dst), make_float4(f[0], f[1], f[2], f[3]));
          __stcs(reinterpret_cast<float4*>(dst) + 1, make_float4(f[4], f[5], f[6], f[7]));
        }
      }
      i = i0 + (i1 - i0) / VE * VE;
    }
    for (unsigned long long j = i + tid; j < i1; j += blockDim.x) from_wire<DT, W>(a.buf, a.buf_off + j, a.uc + j * SW);
  };
  (void)UB;
  // 1. my buffer -> my staging (all shards, my slices)
  for (int k = 0; k < N; ++k) {
    unsigned long long off, len, v0, v1;
    shard_slice(k, &off, &len, &v0, &v1);
    copy_in(off + v0 * VE, off + min(len, v1 * VE));
  }
  if (!barrier(kFlagH)) return;
  // 3. my shard: in-switch sum over all GPUs, mean, multicast back to everyone
  {
    constexpr int U = 4;  // in-switch reductions in flight per thread
    unsigned long long off, len, v0, v1;
    shard_slice(me, &off, &len, &v0, &v1);
    for (unsigned long long vb = v0 + tid; vb < v1; vb += U * blockDim.x) {
      uint4 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const unsigned long long v = vb + (unsigned long long)u * blockDim.x;
        if (v < v1) r[u] = Mm<W>::ld_reduce(a.mc + (off + v * VE) * SW);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const unsigned long long v = vb + (unsigned long long)u * blockDim.x;
        if (v < v1) {
          if (a.op == 1) Mm<W>::scale(r[u], a.inv_n);
          Mm<W>::st(a.mc + (off + v * VE) * SW, r[u]);
        }
      }
    }
  }
  if (!barrier(kFlagR)) return;
  // 5. staging -> my buffer (all shards, my slices)
  for (int k = 0; k < N; ++k) {
    unsigned long long off, len, v0, v1;
    shard_slice(k, &off, &len, &v0, &v1);
    copy_out(off + v0 * VE, off + min(len, v1 * VE));
  }
  __syncthreads();
  if (tid == 0) R->epoch[b] = e;
}

template <int DT, int W>
cudaError_t launch_nvls_typed(const NvlsArgs& a, cudaStream_t s) {
  nvls_kernel<DT, W><<<a.G, 512, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

// ---------------- host side (called from torus_abi.cu) ----------------
int nvls_prepare(int device, int rank, size_t bytes, int world, NvlsState* st, long long blob[2]) {
  if (!load_drv(&g_drv)) return 4;
  CUdevice dev;
  if (g_drv.deviceGet(&dev, device) != CUDA_SUCCESS) return 4;
  CUmemAllocationProp prop;
  memset(&prop, 0, sizeof prop);
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = dev;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t ga = 0, gm = 0;
  if (g_drv.memGetAllocationGranularity(&ga, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS) return 4;
  CUmulticastObjectProp mp;
  memset(&mp, 0, sizeof mp);
  mp.numDevices = (unsigned)world;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.size = bytes;
  if (g_drv.multicastGetGranularity(&gm, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS) return 3;
  const size_t g = ga > gm ? ga : gm;
  const size_t sz = (bytes + g - 1) / g * g;
  mp.size = sz;
  st->size = sz;
  st->gran = g;
  st->dev = dev;
  if (g_drv.memCreate(&st->mem, sz, &prop, 0) != CUDA_SUCCESS) return 4;
  blob[0] = blob[1] = -1;
  if (rank == 0) {
    if (g_drv.multicastCreate(&st->mc_handle, &mp) != CUDA_SUCCESS) return 3;
    int fd = -1;
    if (g_drv.memExportToShareableHandle(&fd, st->mc_handle, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0) != CUDA_SUCCESS)
      return 3;
    blob[0] = (long long)getpid();
    blob[1] = fd;
    st->export_fd = fd;
    st->have_mc = true;
  }
  // map my physical memory (unicast view)
  CUdeviceptr uc = 0;
  if (g_drv.memAddressReserve(&uc, sz, g, 0, 0) != CUDA_SUCCESS) return 4;
  if (g_drv.memMap(uc, sz, 0, st->mem, 0) != CUDA_SUCCESS) return 4;
  CUmemAccessDesc acc;
  memset(&acc, 0, sizeof acc);
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (g_drv.memSetAccess(uc, sz, &acc, 1) != CUDA_SUCCESS) return 4;
  st->uc = uc;
  return 0;
}

int nvls_attach(NvlsState* st, const long long blob0[2]) {
  if (!st->have_mc) {
#ifndef SYS_pidfd_open
#define SYS_pidfd_open 434
#endif
#ifndef SYS_pidfd_getfd
#define SYS_pidfd_getfd 438
#endif
    const int pidfd = (int)syscall(SYS_pidfd_open, (pid_t)blob0[0], 0);
    if (pidfd < 0) return 5;
    const int fd = (int)syscall(SYS_pidfd_getfd, pidfd, (int)blob0[1], 0);
    close(pidfd);
    if (fd < 0) return 5;
    const CUresult r = g_drv.memImportFromShareableHandle(&st->mc_handle, (void*)(uintptr_t)fd,
                                                          CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    close(fd);
    if (r != CUDA_SUCCESS) return 5;
    st->have_mc = true;
  }
  return g_drv.multicastAddDevice(st->mc_handle, st->dev) == CUDA_SUCCESS ? 0 : 3;
}

int nvls_bind(NvlsState* st) {
  if (g_drv.multicastBindMem(st->mc_handle, 0, st->mem, 0, st->size, 0) != CUDA_SUCCESS) return 3;
  CUdeviceptr mc = 0;
  if (g_drv.memAddressReserve(&mc, st->size, st->gran, 0, 0) != CUDA_SUCCESS) return 4;
  if (g_drv.memMap(mc, st->size, 0, st->mc_handle, 0) != CUDA_SUCCESS) return 4;
  CUmemAccessDesc acc;
  memset(&acc, 0, sizeof acc);
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = st->dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (g_drv.memSetAccess(mc, st->size, &acc, 1) != CUDA_SUCCESS) return 4;
  st->mc = mc;
  st->ready = true;
  return 0;
}

void nvls_release(NvlsState* st) {
  if (!g_drv.ok) return;
  if (st->mc) {
    g_drv.memUnmap(st->mc, st->size);
    g_drv.memAddressFree(st->mc, st->size);
  }
  if (st->have_mc && st->ready) g_drv.multicastUnbind(st->mc_handle, st->dev, 0, st->size);
  if (st->uc) {
    g_drv.memUnmap(st->uc, st->size);
    g_drv.memAddressFree(st->uc, st->size);
  }
  if (st->mem) g_drv.memRelease(st->mem);
  if (st->have_mc) g_drv.memRelease(st->mc_handle);
  if (st->export_fd >= 0) close(st->export_fd);
  *st = NvlsState{};
}

cudaError_t launch_nvls(const RankDev* ranks, const NvlsState* st, void* buf, unsigned long long n,
                        unsigned long long buf_off, int dtype, int wire, int op, float inv_n, int G,
                        unsigned long long timeout_ns, cudaStream_t s) {
  NvlsArgs a;
  a.ranks = ranks;
  a.buf = buf;
  a.uc = reinterpret_cast<char*>(st->uc);
  a.mc = reinterpret_cast<char*>(st->mc);
  a.n = n;
  a.buf_off = buf_off;
  a.timeout_ns = timeout_ns;
  a.G = G;
  a.q = (wire == 0) ? 4 : 8;
  a.op = op;
  a.inv_n = inv_n;
  if (dtype == wire) {
    if (dtype == 0) return launch_nvls_typed<0, 0>(a, s);
    if (dtype == 1) return launch_nvls_typed<1, 1>(a, s);
    if (dtype == 2) return launch_nvls_typed<2, 2>(a, s);
  } else if (dtype == 0 && wire == 1) {
    return launch_nvls_typed<0, 1>(a, s);
  } else if (dtype == 0 && wire == 2) {
    return launch_nvls_typed<0, 2>(a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace torus
