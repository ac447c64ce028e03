// torus_cast.cu -- the degenerate N = 1 case of the all-reduce (SURVEY 8(a) row a7,
// BASELINE.json north_star: "The 1-GPU point is the fused cast/scale-only degenerate
// case"): buf = from_wire(to_wire(buf)) for an f32 buffer with an fp16 / bf16 wire
// (PAPER.md:121), the mean over one rank being x * 1.
//
// HBM-bound: 8 B per element (read + write f32).  This variant streams the buffer through
// shared memory with TMA bulk copies (cp.async.bulk global -> shared, convert in place,
// shared -> global): a persistent grid of one CTA per SM, a ring of NB 32 KiB buffers per
// CTA, one thread issuing the bulk copies -- so ~148 * NB * 32 KiB are in flight with a
// handful of instructions, where the LDG/STG variant (torus_kernels.cu castscale_kernel)
// needs every thread's registers for it.  The rounding is the same pack / unpack pair
// as every other kernel (RNE, no FTZ), so the result is bit-identical.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "torus_device.cuh"

namespace torus {
namespace {

constexpr int kCastThreads = 256;
constexpr int kCastTile = 32 * 1024;  // bytes per ring buffer (8192 floats)

template <int W, int NB>
__global__ void __launch_bounds__(kCastThreads, 1) castscale_tma_kernel(float* buf, unsigned long long n) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NB * kCastTile);
  const int tid = threadIdx.x;
  const unsigned long long nvec4 = n / 4;                         // whole float4s
  const unsigned long long per_tile = kCastTile / 16;            // float4s per tile
  const unsigned long long ntiles = (nvec4 + per_tile - 1) / per_tile;
  const unsigned long long first = blockIdx.x, step = gridDim.x;
  if (tid == 0) {
    for (int i = 0; i < NB; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto tile_bytes = [&](unsigned long long t) -> uint32_t {
    const unsigned long long v0 = t * per_tile;
    const unsigned long long nv = (nvec4 - v0) < per_tile ? (nvec4 - v0) : per_tile;
    return (uint32_t)(nv * 16);
  };
  auto issue = [&](unsigned long long t, int b) {
    const uint32_t bytes = tile_bytes(t);
    mbar_expect_tx(&full[b], bytes);
    tma_load(smem + (size_t)b * kCastTile, buf + t * per_tile * 4, bytes, &full[b]);
  };
  // prologue: fill the ring
  if (tid == 0)
    for (int b = 0; b < NB; ++b) {
      const unsigned long long t = first + (unsigned long long)b * step;
      if (t < ntiles) issue(t, b);
    }
  unsigned long long i = 0;
  for (unsigned long long t = first; t < ntiles; t += step, ++i) {
    const int b = (int)(i % NB);
    mbar_wait(&full[b], (uint32_t)((i / NB) & 1));
    // convert in place: 8 floats at a time through the wire type (C9: RNE, no FTZ)
    const uint32_t bytes = tile_bytes(t);
    float* f = reinterpret_cast<float*>(smem + (size_t)b * kCastTile);
    const int n8 = (int)(bytes / 32);
    for (int k = tid; k < n8; k += kCastThreads) {
      float4* p = reinterpret_cast<float4*>(f + 8 * k);
      const float4 x0 = p[0], x1 = p[1];
      const float x[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
      float y[8];
      unpack<W>(pack<W>(x), y);
      p[0] = make_float4(y[0], y[1], y[2], y[3]);
      p[1] = make_float4(y[4], y[5], y[6], y[7]);
    }
    if ((bytes & 31) && tid == 0) {  // a last odd float4
      float4* p = reinterpret_cast<float4*>(f + 8 * n8);
      const float4 x0 = p[0];
      const float x[8] = {x0.x, x0.y, x0.z, x0.w, 0.f, 0.f, 0.f, 0.f};
      float y[8];
      unpack<W>(pack<W>(x), y);
      p[0] = make_float4(y[0], y[1], y[2], y[3]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      tma_store(buf + t * per_tile * 4, smem + (size_t)b * kCastTile, bytes);
      tma_commit();
      // refill the PREVIOUS buffer once its store has read it (one iteration of slack)
      if (i > 0) {
        tma_wait_read<1>();
        const unsigned long long tn = t - step + (unsigned long long)NB * step;  // tile for buffer (i-1)%NB
        if (tn < ntiles) issue(tn, (int)((i - 1) % NB));
      }
    }
  }
  if (tid == 0) {
    // the last buffer's refill (no later iteration did it)
    tma_wait_all<0>();
  }
  // the < 4 trailing floats
  if (blockIdx.x == 0 && tid < (int)(n - nvec4 * 4)) {
    const float x[8] = {buf[nvec4 * 4 + tid], 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    float y[8];
    unpack<W>(pack<W>(x), y);
    buf[nvec4 * 4 + tid] = y[0];
  }
}

template <int W, int NB>
cudaError_t launch_cast_tma_typed(float* buf, unsigned long long n, int ctas, cudaStream_t stream) {
  const int smem = NB * kCastTile + NB * 8;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(castscale_tma_kernel<W, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  castscale_tma_kernel<W, NB><<<ctas, kCastThreads, smem, stream>>>(buf, n);
  return cudaGetLastError();
}

}  // namespace

// TMA-streamed cast round trip; the caller guarantees a 16-byte aligned buffer.
// env TORUS_CS_TMA = "<buffers>x<ctas per SM>" (default 6x1).
cudaError_t launch_castscale_tma(void* buf, unsigned long long n, int wire, cudaStream_t stream) {
  int nb = 6, cps = 1;
  if (const char* v = getenv("TORUS_CS_TMA")) sscanf(v, "%dx%d", &nb, &cps);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const unsigned long long tiles = (n / 4 * 16 + kCastTile - 1) / kCastTile;
  int ctas = (int)std::min<unsigned long long>((unsigned long long)sms * cps, tiles > 0 ? tiles : 1);
  float* f = reinterpret_cast<float*>(buf);
  auto go = [&](auto tag) -> cudaError_t {
    constexpr int Wt = decltype(tag)::value;
    if (nb == 3) return launch_cast_tma_typed<Wt, 3>(f, n, ctas, stream);
    if (nb == 4) return launch_cast_tma_typed<Wt, 4>(f, n, ctas, stream);
    if (nb == 2) return launch_cast_tma_typed<Wt, 2>(f, n, ctas, stream);
    return launch_cast_tma_typed<Wt, 6>(f, n, ctas, stream);
  };
  if (wire == DT_F16) return go(std::integral_constant<int, DT_F16>{});
  if (wire == DT_BF16) return go(std::integral_constant<int, DT_BF16>{});
  return cudaErrorInvalidValue;
}

}  // namespace torus
