/*
 * torus_oracle.h -- CPU oracle for the 2D-Torus all-reduce (TEST INFRASTRUCTURE ONLY).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  The product path (paper_1811_05233_b200/) never links,
 * imports or executes anything under oracle/, and this file shares no code with it.
 *
 * What it computes (Sec. 2.2): N = X*Y ranks arranged in an X-by-Y grid;
 * "Firstly, reduce-scatter is performed horizontally. Then, all-reduce is performed
 * vertically. Finally, all-gather is performed horizontally."  Every rank ends with the
 * element-wise sum (or mean, "synchronize and average gradients") of all N
 * input buffers, communicated in the wire precision (FP16 communication).
 *
 * The oracle SIMULATES every rank executing the ring schedule step by step
 * (SURVEY.md Sec. 8(c), C1-C13), single-threaded, scalar, plain C.  Readings of the
 * paper where it is silent are listed in DESIGN.md Sec. 3 (R1..R17).
 *
 * Parity status: every function here is pinned by tests/test_oracle.py against
 * hand-computed values, SPEC worked examples, closed forms and brute force.  No function
 * is "parity unpinned".
 */
#ifndef TORUS_ORACLE_H
#define TORUS_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* element / wire types (values equal to the product ABI's codes by coincidence of the
 * north star's list {f32,f16,bf16,i32}; the oracle does not include the product header) */
enum { ORC_F32 = 0, ORC_F16 = 1, ORC_BF16 = 2, ORC_I32 = 3 };
enum { ORC_SUM = 0, ORC_MEAN = 1 };
/* accumulation policy: PHASE rounds to the wire type only at phase outputs;
 * HOP rounds every ring message to the wire type (NCCL-ring-like). */
enum { ORC_PHASE = 0, ORC_HOP = 1 };
/* phases, in the paper's order */
enum { ORC_H_RS = 0, ORC_V_RS = 1, ORC_V_AG = 2, ORC_H_AG = 3 };

enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_EGRID = 2, ORC_EUNSUP = 3, ORC_ENOMEM = 4 };

/* per-rank trace counters (SPEC.md:278-302 CostReport analogue) */
typedef struct {
    long long steps[4]; /* sequential send steps this rank took in each phase   */
    long long sent[4];  /* elements this rank sent in each phase                */
    long long recv[4];  /* elements this rank received in each phase            */
} orc_counters;

/* ---- conversions: IEEE round-to-nearest-even, bit-level, no FTZ ---- */
uint16_t orc_f32_to_f16(float f);
float    orc_f16_to_f32(uint16_t h);
uint16_t orc_f32_to_bf16(float f);
float    orc_bf16_to_f32(uint16_t h);
void orc_f32_to_f16_array(const float* x, uint16_t* y, long long n);
void orc_f16_to_f32_array(const uint16_t* x, float* y, long long n);
void orc_f32_to_bf16_array(const float* x, uint16_t* y, long long n);
void orc_bf16_to_f32_array(const uint16_t* x, float* y, long long n);

/* ---- partition (SPEC.md:67-75 when q == 1) ----
 * Split n elements into `parts` contiguous ranges, quantum q: Q = ceil(n/q) quanta are
 * split into balanced counts (larger first), multiplied by q, and the overflow is trimmed
 * from the tail.  Fills off[parts], len[parts]. */
int orc_qpart(long long n, int parts, int q, long long* off, long long* len);

/* ---- the 2D-Torus all-reduce, simulated ----
 * in[r]  : rank r's input buffer, D elements of `dtype` (host memory)
 * out[r] : rank r's output buffer, D elements of `dtype` (may alias in[r])
 * wire   : communication type; == dtype, or F16/BF16 when dtype == F32
 * q      : partition quantum in elements (1 reproduces SPEC's partition)
 * round_elems : the call is processed in consecutive rounds of this many elements
 *               (SURVEY C13); <= 0 means a single round
 * ctr    : optional [X*Y] per-rank counters (accumulated over rounds)                   */
int orc_torus_allreduce(int X, int Y, long long D, int dtype, int wire, int op, int policy,
                        int q, long long round_elems, const void* const* in, void* const* out,
                        orc_counters* ctr);

/* Closed-form value of ONE output element i of orc_torus_allreduce (the
 * ring leaves chunk c folded as w[c+1] + w[c+2] + ... + w[c]).  Writes one element of
 * `dtype` to out_elem.  Used to check sampled outputs at full size. */
int orc_torus_element(int X, int Y, long long D, int dtype, int wire, int op, int policy,
                      int q, long long round_elems, long long i, const void* const* in,
                      void* out_elem);

/* Flat ring all-reduce over R ranks (ref [14]; SPEC.md:199-224 with the
 * ownership fix of SURVEY Q5): R-1 reduce-scatter steps then R-1 all-gather steps. */
int orc_ring_allreduce(int R, long long D, int dtype, int wire, int op, int policy, int q,
                       long long round_elems, const void* const* in, void* const* out,
                       orc_counters* ctr);

/* Hierarchical all-reduce [6]: ring reduce to the
 * column-0 leader of each row, ring all-reduce of the full buffer among the Y leaders,
 * ring broadcast back along each row. */
int orc_hier_allreduce(int X, int Y, long long D, int dtype, int wire, int op, int policy,
                       int q, const void* const* in, void* const* out, orc_counters* ctr);

/* Naive brute force: out[i] = sum_r (double) in[r][i] (mean: / N), from the ORIGINAL
 * inputs (before the wire cast).  i32 is summed exactly in int64. */
size_t orc_type_size(int t);
int orc_brute_sum_f64(int N, long long D, int dtype, int op, const void* const* in,
                      double* out);

#ifdef __cplusplus
}
#endif
#endif
