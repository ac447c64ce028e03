// torus_ll128.h -- launch arguments of the LL128 push kernel (torus_ll128.cu), shared by
// torus_abi.cu and torus_ll128.cu only.  Not part of the public ABI.
#pragma once
#include "torus_internal.h"

namespace torus {

constexpr int kL128Line = 128;      // bytes per line: 120 bytes of data + an 8-byte flag
constexpr int kL128Unit = 4 * kL128Line;  // 16-byte lanes: one warp moves four lines = 30 wire vectors
#ifndef TORUS_LL128_THREADS
#define TORUS_LL128_THREADS 1024
#endif
constexpr int kL128CtaWarps = TORUS_LL128_THREADS / 32;

struct L128Args {
  const RankDev* ranks;          // device array [nlocal]
  void* buf[kMaxLocal];          // user buffer of each local rank
  unsigned long long n;          // elements in this round
  unsigned long long buf_off;    // element offset of the round inside the user buffers
  unsigned long long timeout_ns;
  int nlocal;
  int op;                        // 0 sum, 1 mean
  float inv_n;                   // f32(1/N)
  int aligned;                   // all user buffers 16-byte aligned
  const MultiSeg* segs;          // NEXT-1: device table [nlocal][nseg] of the bucket's tensors
  int nseg;                      //   (nullptr / 0: one flat buffer per rank)
  // round geometry, host-computed: chunk j offset, sub-chunk (j, s) at [j*Y+s]:
  // offset inside the chunk, length, units (30 wire vectors each), unit offset of the
  // sub-chunk inside its chunk's stream
  unsigned long long g_co[kMaxRanks], g_cs[kMaxRanks], g_sl[kMaxRanks];
  int g_U[kMaxRanks], g_uoff[kMaxRanks];
  int Umax;                      // units of the largest sub-chunk
  // inboxes (slab byte offsets by call parity) and bytes per source slot
  unsigned long long h_off[2], v_off[2], ag_off[2], hag_off[2];
  unsigned long long h_stride, v_stride, ag_stride, hag_stride;
  int wk[5];                     // warps per rank of each stage: A, B, C, D, E
  int wsum;                      // warps per rank
  int ctas;                      // CTAs per rank
  int lane_bytes;                // 16 (1024-thread CTAs) or 32 (512-thread CTAs, flat calls only)
};

cudaError_t launch_ll128(const L128Args& a, int dtype, int wire, bool cooperative, cudaStream_t stream);

}  // namespace torus
