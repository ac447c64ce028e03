// torus_pull.h -- launch arguments of the pull (dataflow) kernel, shared by torus_abi.cu
// and torus_pull.cu only.  Not part of the public ABI.
#pragma once
#include "torus_internal.h"

namespace torus {

// Per-launch arguments of the pull (dataflow) kernel, torus_pull.cu.  Everything that
// decides WHICH bytes and flags a tile touches (n, q, TV, Kmax, region and flag offsets)
// must be equal on every rank; the CTA split g[] and the ring (nslots, slot_bytes) are
// rank-local choices.
struct PullArgs {
  const RankDev* ranks;          // device array [nlocal]
  void* buf[kMaxLocal];          // user buffer of each local rank
  unsigned long long n;          // elements in this round
  unsigned long long buf_off;    // element offset of the round inside the user buffers
  unsigned long long win_off[2], p1_off[2], chunk_off[2];  // slab byte offsets by parity
  unsigned long long flag_off;   // slab byte offset of the pull flag region
  unsigned long long fl_win, fl_p1, fl_v, fl_c, fl_pres;   // word offsets of the flag kinds
  unsigned long long timeout_ns;
  int nlocal;
  int q;                         // partition quantum (elements) = one 16-byte wire vector
  int TV;                        // 16-byte wire vectors per tile
  int Kmax;                      // tiles of the largest sub-chunk
  int op;                        // 0 sum, 1 mean
  float inv_n;                   // f32(1/N)
  int aligned;                   // all user buffers 16-byte aligned
  int g[6];                      // CTAs per rank of each kind: S0, R, VR, VA, H, SIG
  int gsum;
  int nslots, slot_bytes;        // shared-memory ring
  unsigned long long* trace;     // optional [nlocal*gsum][kPullTraceJobs][kPullTraceEv] stamps
  int fence;                     // publish: 0 fence.acq_rel.sys in the data CTA; 1 .gpu (measurement
                                 // only); 2 none (measurement only); 3 the data CTA releases at gpu
                                 // scope to SIG CTAs, which fence at sys scope and raise the flags
  unsigned long long* pub;       // fence 3: [nlocal * gsum] (epoch << 32 | jobs published) per CTA
  int fault;                     // negative controls (tests only): 1 corrupt one reduced element,
                                 // 2 skip one P1 wait (read before the peer wrote); 0 off
  unsigned delay_ns;             // robustness: each CTA starts after a pseudo-random delay < this
  int zc;                        // zero-copy: the peers' user buffers are mapped here (registered,
                                 // dtype == wire, 16-byte aligned on every rank) -- no S0 copy
  char* peer_buf[kMaxRanks];     // zc: every rank's user buffer as mapped in this process
  // round geometry (SURVEY C3 nested quantum partition), computed on the host per round:
  unsigned long long g_co[kMaxRanks];    // chunk j: offset in the round (elements)
  unsigned long long g_cs[kMaxRanks];    // sub-chunk (j, s) at [j * Y + s]: offset inside chunk j
  unsigned long long g_sl[kMaxRanks];    // sub-chunk (j, s): length (elements)
  int g_K[kMaxRanks];                    // sub-chunk (j, s): tiles
};
constexpr int kPullTraceJobs = 64;  // trace: first 63 jobs of every CTA; slot 63 = CTA start/end
constexpr int kPullTraceEv = 8;     // stamps per job
inline size_t pull_smem_bytes(int nslots, int slot_bytes) {
  return (size_t)nslots * slot_bytes + 2 * (size_t)nslots * 8;
}
constexpr size_t kPullFlagBytes = 8ull << 20;  // pull flag region per slab

cudaError_t launch_pull(const PullArgs& a, int dtype, int wire, bool cooperative, cudaStream_t stream);
// per-call header check (TORUS_CHECK=1): every rank posts a descriptor of the call
// (count, dtype, wire, op, route) to its peers and compares theirs with its own
cudaError_t launch_check(const RankDev* ranks, int nlocal, unsigned long long hdr_off, unsigned seq,
                         unsigned desc, unsigned long long timeout_ns, cudaStream_t stream);
int pull_ctas_per_sm(size_t smem);

}  // namespace torus
