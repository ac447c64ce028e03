/*
 * torus_oracle.c -- plain, slow, obviously-correct CPU oracle (TEST INFRASTRUCTURE ONLY).
 *
 * See torus_oracle.h for the contract and the import rule: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this.  It shares no
 * code with paper_1811_05233_b200/ (neither includes nor links the other).
 *
 * Structure follows the paper's three steps (Sec. 2.2) executed as rings
 * (Figure 1: "multiple rings in horizontal and vertical orientations"),
 * every rank simulated explicitly, every message copied into a message buffer before it
 * is delivered.  Accumulation values are held as 32-bit patterns: an IEEE binary32 for
 * float wires (f32 accumulation, PAPER.md:121 / SPEC.md:198), a uint32 for i32 wires
 * (two's-complement wrap).
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared (no -ffast-math: no FTZ,
 * no contraction; x86-64 evaluates float in SSE single precision, FLT_EVAL_METHOD 0).
 */
#include "torus_oracle.h"

#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------ */
/* conversions                                                              */
/* ------------------------------------------------------------------------------------ */

static uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* binary32 -> binary16, round to nearest even, overflow -> inf, subnormals kept. */
uint16_t orc_f32_to_f16(float f)
{
    uint32_t x = f2u(f);
    uint32_t sign = (x >> 16) & 0x8000u;
    uint32_t ax = x & 0x7fffffffu;
    if (ax > 0x7f800000u) return (uint16_t)(sign | 0x7e00u);   /* NaN -> quiet NaN */
    if (ax == 0x7f800000u) return (uint16_t)(sign | 0x7c00u);  /* inf */
    int e = (int)(ax >> 23) - 127;                               /* unbiased exponent */
    uint32_t m = ax & 0x7fffffu;
    if ((ax >> 23) == 0) return (uint16_t)sign;                  /* f32 subnormal: |x| < 2^-126 -> 0 */
    if (e >= -14) {
        /* normal binary16 candidate: keep 10 of 23 mantissa bits */
        uint32_t h = ((uint32_t)(e + 15) << 10) | (m >> 13);
        uint32_t rest = m & 0x1fffu;
        if (rest > 0x1000u || (rest == 0x1000u && (h & 1u))) h += 1u; /* carry may reach inf */
        if (h >= 0x7c00u) h = 0x7c00u;                           /* overflow -> inf */
        return (uint16_t)(sign | h);
    }
    /* binary16 subnormal: value = (m | 2^23) * 2^(e-23); unit 2^-24 -> shift by -(e+1) */
    int shift = -(e + 1);
    if (shift > 24) return (uint16_t)sign;                       /* < 2^-25: rounds to 0 */
    uint32_t full = m | 0x800000u;
    uint32_t h = full >> shift;
    uint32_t rest = full & ((1u << shift) - 1u);
    uint32_t half = 1u << (shift - 1);
    if (rest > half || (rest == half && (h & 1u))) h += 1u;      /* may become min normal */
    return (uint16_t)(sign | h);
}

float orc_f16_to_f32(uint16_t h)
{
    uint32_t sign = ((uint32_t)h & 0x8000u) << 16;
    uint32_t e = ((uint32_t)h >> 10) & 0x1fu;
    uint32_t m = (uint32_t)h & 0x3ffu;
    if (e == 0x1fu) return u2f(sign | 0x7f800000u | (m << 13));  /* inf / NaN */
    if (e == 0) {
        if (m == 0) return u2f(sign);
        /* subnormal: m * 2^-24, exact in binary32 */
        float v = (float)m * (1.0f / 16777216.0f);
        return sign ? -v : v;
    }
    return u2f(sign | ((e + 112u) << 23) | (m << 13));
}

/* binary32 -> bfloat16, round to nearest even (bfloat16 keeps binary32's exponent). */
uint16_t orc_f32_to_bf16(float f)
{
    uint32_t x = f2u(f);
    if ((x & 0x7fffffffu) > 0x7f800000u) return (uint16_t)(((x >> 16) & 0x8000u) | 0x7fc0u);
    uint32_t upper = x >> 16;
    uint32_t rest = x & 0xffffu;
    if (rest > 0x8000u || (rest == 0x8000u && (upper & 1u))) upper += 1u; /* may reach inf */
    return (uint16_t)upper;
}

float orc_bf16_to_f32(uint16_t h) { return u2f((uint32_t)h << 16); }

/* ------------------------------------------------------------------------------------ */
/* partition                                                                */
/* ------------------------------------------------------------------------------------ */

int orc_qpart(long long n, int parts, int q, long long* off, long long* len)
{
    if (n < 0 || parts < 1 || q < 1 || !off || !len) return ORC_EINVAL;
    long long Q = (n + q - 1) / q;          /* quanta */
    long long base = Q / parts, rem = Q % parts;
    long long start_q = 0;
    for (int i = 0; i < parts; ++i) {
        long long cnt = base + (i < rem ? 1 : 0);
        long long a = start_q * q, b = (start_q + cnt) * q;
        if (a > n) a = n;                    /* trim the overflow from the tail */
        if (b > n) b = n;
        off[i] = a;
        len[i] = b - a;
        start_q += cnt;
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------------------ */
/* element helpers                                                                      */
/* ------------------------------------------------------------------------------------ */

static int valid_types(int dtype, int wire)
{
    if (dtype < ORC_F32 || dtype > ORC_I32 || wire < ORC_F32 || wire > ORC_I32) return 0;
    if (dtype == wire) return 1;
    return dtype == ORC_F32 && (wire == ORC_F16 || wire == ORC_BF16);
}

static size_t type_size(int t) { return (t == ORC_F16 || t == ORC_BF16) ? 2 : 4; }

/* C1: w = to_wire(in[i]), returned as an accumulator pattern (f32 bits or u32) */
static uint32_t load_wire(const void* in, int dtype, int wire, long long i)
{
    if (dtype == ORC_I32) return (uint32_t)((const int32_t*)in)[i];
    if (dtype == ORC_F16) return f2u(orc_f16_to_f32(((const uint16_t*)in)[i]));
    if (dtype == ORC_BF16) return f2u(orc_bf16_to_f32(((const uint16_t*)in)[i]));
    float x = ((const float*)in)[i];
    if (wire == ORC_F16) return f2u(orc_f16_to_f32(orc_f32_to_f16(x)));
    if (wire == ORC_BF16) return f2u(orc_bf16_to_f32(orc_f32_to_bf16(x)));
    return f2u(x);
}

/* the "+" of every reduce step: f32 add, or u32 wrapping add */
static uint32_t acc_add(uint32_t a, uint32_t b, int wire)
{
    if (wire == ORC_I32) return a + b;
    return f2u(u2f(a) + u2f(b));
}

/* round an f32 accumulator to the wire type and back (identity for f32 / i32) */
static uint32_t round_wire(uint32_t a, int wire)
{
    if (wire == ORC_F16) return f2u(orc_f16_to_f32(orc_f32_to_f16(u2f(a))));
    if (wire == ORC_BF16) return f2u(orc_bf16_to_f32(orc_f32_to_bf16(u2f(a))));
    return a;
}

/* C8 / C10: mean = f32 sum * f32(1/N); i32 mean = wrapped sum / N truncated (C99 /) */
static uint32_t scale_mean(uint32_t a, int wire, int op, int N)
{
    if (op != ORC_MEAN) return a;
    if (wire == ORC_I32) return (uint32_t)((int32_t)a / (int32_t)N);
    float inv = 1.0f / (float)N;
    return f2u(u2f(a) * inv);
}

/* C11: out = from_wire(final) cast to dtype (exact: the value is representable) */
static void store_out(void* out, int dtype, long long i, uint32_t a)
{
    if (dtype == ORC_I32) ((int32_t*)out)[i] = (int32_t)a;
    else if (dtype == ORC_F32) ((float*)out)[i] = u2f(a);
    else if (dtype == ORC_F16) ((uint16_t*)out)[i] = orc_f32_to_f16(u2f(a));
    else ((uint16_t*)out)[i] = orc_f32_to_bf16(u2f(a));
}

static long long mod(long long a, long long m) { long long r = a % m; return r < 0 ? r + m : r; }

/* ------------------------------------------------------------------------------------ */
/* ring primitives over a group of ranks (ownership fix SURVEY Q5)     */
/* ------------------------------------------------------------------------------------ */

/* Ring reduce-scatter among the R ranks listed in grp[], over the range [base, base+n)
 * of each rank's accumulator array acc[rank], with partition quantum q.  At step s,
 * position p sends its partial of part (p - s - 1) mod R to position p+1, which sets
 * partial = incoming + partial.  Afterwards position p holds the ring sum of part p.
 * If finalize: the owner applies scale_mean (when last_reduce) and round_wire (always:
 * the phase output is in the wire type).  HOP policy rounds every message. */
static int ring_rs(int R, const int* grp, uint32_t** acc, long long base, long long n, int q,
                   int wire, int op, int N, int policy, int last_reduce, int phase,
                   orc_counters* ctr)
{
    long long* off = (long long*)malloc(sizeof(long long) * R);
    long long* len = (long long*)malloc(sizeof(long long) * R);
    uint32_t** msg = (uint32_t**)calloc(R, sizeof(uint32_t*));
    if (!off || !len || !msg) { free(off); free(len); free(msg); return ORC_ENOMEM; }
    orc_qpart(n, R, q, off, len);
    int rc = ORC_OK;
    for (int p = 0; p < R; ++p) {
        msg[p] = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
        if (!msg[p]) rc = ORC_ENOMEM;
    }
    for (int s = 0; rc == ORC_OK && s < R - 1; ++s) {
        /* every position sends simultaneously: copy all messages first */
        for (int p = 0; p < R; ++p) {
            long long k = mod(p - s - 1, R);
            for (long long i = 0; i < len[k]; ++i) {
                uint32_t v = acc[grp[p]][base + off[k] + i];
                msg[p][i] = (policy == ORC_HOP) ? round_wire(v, wire) : v;
            }
            if (ctr) {
                ctr[grp[p]].steps[phase] += 1;
                ctr[grp[p]].sent[phase] += len[k];
                ctr[grp[(p + 1) % R]].recv[phase] += len[k];
            }
        }
        for (int p = 0; p < R; ++p) {
            long long k = mod(p - s - 1, R);
            int dst = grp[(p + 1) % R];
            for (long long i = 0; i < len[k]; ++i) {
                uint32_t* a = &acc[dst][base + off[k] + i];
                *a = acc_add(msg[p][i], *a, wire);
            }
        }
    }
    if (rc == ORC_OK) {
        for (int p = 0; p < R; ++p)
            for (long long i = 0; i < len[p]; ++i) {
                uint32_t* a = &acc[grp[p]][base + off[p] + i];
                uint32_t v = *a;
                if (last_reduce) v = scale_mean(v, wire, op, N);
                *a = round_wire(v, wire);
            }
    }
    for (int p = 0; p < R; ++p) free(msg[p]);
    free(msg); free(off); free(len);
    return rc;
}

/* Ring all-gather among grp[] over [base, base+n): at step t, position p sends part
 * (p - t) mod R to position p+1, which stores it (a pure copy). */
static int ring_ag(int R, const int* grp, uint32_t** acc, long long base, long long n, int q,
                   int phase, orc_counters* ctr)
{
    long long* off = (long long*)malloc(sizeof(long long) * R);
    long long* len = (long long*)malloc(sizeof(long long) * R);
    uint32_t** msg = (uint32_t**)calloc(R, sizeof(uint32_t*));
    if (!off || !len || !msg) { free(off); free(len); free(msg); return ORC_ENOMEM; }
    orc_qpart(n, R, q, off, len);
    int rc = ORC_OK;
    for (int p = 0; p < R; ++p) {
        msg[p] = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
        if (!msg[p]) rc = ORC_ENOMEM;
    }
    for (int t = 0; rc == ORC_OK && t < R - 1; ++t) {
        for (int p = 0; p < R; ++p) {
            long long k = mod(p - t, R);
            memcpy(msg[p], &acc[grp[p]][base + off[k]], sizeof(uint32_t) * (size_t)len[k]);
            if (ctr) {
                ctr[grp[p]].steps[phase] += 1;
                ctr[grp[p]].sent[phase] += len[k];
                ctr[grp[(p + 1) % R]].recv[phase] += len[k];
            }
        }
        for (int p = 0; p < R; ++p) {
            long long k = mod(p - t, R);
            memcpy(&acc[grp[(p + 1) % R]][base + off[k]], msg[p], sizeof(uint32_t) * (size_t)len[k]);
        }
    }
    for (int p = 0; p < R; ++p) free(msg[p]);
    free(msg); free(off); free(len);
    return rc;
}

static uint32_t** alloc_acc(int N, long long n)
{
    uint32_t** acc = (uint32_t**)calloc(N, sizeof(uint32_t*));
    if (!acc) return NULL;
    for (int r = 0; r < N; ++r) {
        acc[r] = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
        if (!acc[r]) {
            for (int k = 0; k < r; ++k) free(acc[k]);
            free(acc);
            return NULL;
        }
    }
    return acc;
}

static void free_acc(uint32_t** acc, int N)
{
    if (!acc) return;
    for (int r = 0; r < N; ++r) free(acc[r]);
    free(acc);
}

/* ------------------------------------------------------------------------------------ */
/* 2D-Torus all-reduce                                                    */
/* ------------------------------------------------------------------------------------ */

int orc_torus_allreduce(int X, int Y, long long D, int dtype, int wire, int op, int policy,
                        int q, long long round_elems, const void* const* in, void* const* out,
                        orc_counters* ctr)
{
    if (X < 1 || Y < 1) return ORC_EGRID;
    if (D < 0 || q < 1 || !in || !out || !valid_types(dtype, wire)) return ORC_EINVAL;
    if (op != ORC_SUM && op != ORC_MEAN) return ORC_EINVAL;
    if (policy != ORC_PHASE && policy != ORC_HOP) return ORC_EINVAL;
    const int N = X * Y;
    if (ctr) memset(ctr, 0, sizeof(orc_counters) * (size_t)N);
    if (D == 0) return ORC_OK;
    long long R = (round_elems > 0 && round_elems < D) ? round_elems : D;

    uint32_t** acc = alloc_acc(N, R);
    int* grp = (int*)malloc(sizeof(int) * (size_t)(X > Y ? X : Y));
    long long* coff = (long long*)malloc(sizeof(long long) * X);
    long long* clen = (long long*)malloc(sizeof(long long) * X);
    if (!acc || !grp || !coff || !clen) {
        free_acc(acc, N); free(grp); free(coff); free(clen);
        return ORC_ENOMEM;
    }
    int rc = ORC_OK;
    for (long long r0 = 0; rc == ORC_OK && r0 < D; r0 += R) {
        long long n = (D - r0 < R) ? D - r0 : R;
        /* C1: every rank's contribution in the wire type */
        for (int r = 0; r < N; ++r)
            for (long long i = 0; i < n; ++i) acc[r][i] = load_wire(in[r], dtype, wire, r0 + i);

        /* Phase 1 (C4): reduce-scatter horizontally, a ring over the columns of each row.
         * When Y == 1 this is the last reduce phase and carries the mean (C8). */
        for (int rho = 0; rc == ORC_OK && rho < Y; ++rho) {
            for (int c = 0; c < X; ++c) grp[c] = rho * X + c;
            rc = ring_rs(X, grp, acc, 0, n, q, wire, op, N, policy, Y == 1, ORC_H_RS, ctr);
        }
        /* Phase 2 (C6): all-reduce vertically on each column's chunk = ring RS + ring AG
         * over the rows. */
        orc_qpart(n, X, q, coff, clen);
        if (Y > 1) {
            for (int c = 0; rc == ORC_OK && c < X; ++c) {
                for (int i = 0; i < Y; ++i) grp[i] = i * X + c;
                rc = ring_rs(Y, grp, acc, coff[c], clen[c], q, wire, op, N, policy, 1, ORC_V_RS, ctr);
                if (rc == ORC_OK) rc = ring_ag(Y, grp, acc, coff[c], clen[c], q, ORC_V_AG, ctr);
            }
        }
        /* Phase 3 (C11): all-gather horizontally. */
        for (int rho = 0; rc == ORC_OK && rho < Y; ++rho) {
            for (int c = 0; c < X; ++c) grp[c] = rho * X + c;
            rc = ring_ag(X, grp, acc, 0, n, q, ORC_H_AG, ctr);
        }
        for (int r = 0; rc == ORC_OK && r < N; ++r)
            for (long long i = 0; i < n; ++i) store_out(out[r], dtype, r0 + i, acc[r][i]);
    }
    free_acc(acc, N); free(grp); free(coff); free(clen);
    return rc;
}

/* Closed form of one element.  Element i lies in round r0, chunk c of that
 * round's X-partition and sub-chunk s of chunk c's Y-partition.  Row rho's phase-1 value
 * is the fold w[rho,c+1] + w[rho,c+2] + ... + w[rho,c] (the order the ring leaves it in);
 * the phase-2 value is the fold P1[s+1] + ... + P1[s] over rows. */
int orc_torus_element(int X, int Y, long long D, int dtype, int wire, int op, int policy,
                      int q, long long round_elems, long long i, const void* const* in,
                      void* out_elem)
{
    if (X < 1 || Y < 1) return ORC_EGRID;
    if (D <= 0 || i < 0 || i >= D || q < 1 || !in || !out_elem || !valid_types(dtype, wire))
        return ORC_EINVAL;
    const int N = X * Y;
    long long R = (round_elems > 0 && round_elems < D) ? round_elems : D;
    long long r0 = (i / R) * R;
    long long n = (D - r0 < R) ? D - r0 : R;
    long long li = i - r0;
    long long* off = (long long*)malloc(sizeof(long long) * (size_t)(X > Y ? X : Y));
    long long* len = (long long*)malloc(sizeof(long long) * (size_t)(X > Y ? X : Y));
    uint32_t* p1 = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)Y);
    if (!off || !len || !p1) { free(off); free(len); free(p1); return ORC_ENOMEM; }
    int c = 0, s = 0;
    orc_qpart(n, X, q, off, len);
    for (int k = 0; k < X; ++k) if (li >= off[k] && li < off[k] + len[k]) c = k;
    long long cbase = off[c], clen = len[c];
    orc_qpart(clen, Y, q, off, len);
    for (int k = 0; k < Y; ++k) if (li - cbase >= off[k] && li - cbase < off[k] + len[k]) s = k;

    for (int rho = 0; rho < Y; ++rho) {
        uint32_t a = 0;
        for (int k = 1; k <= X; ++k) {
            int col = (c + k) % X;
            uint32_t w = load_wire(in[rho * X + col], dtype, wire, i);
            if (k == 1) a = w;
            else a = acc_add(policy == ORC_HOP ? round_wire(a, wire) : a, w, wire);
        }
        if (Y == 1) a = scale_mean(a, wire, op, N);
        p1[rho] = round_wire(a, wire);
    }
    uint32_t v = p1[0];
    if (Y > 1) {
        uint32_t a = 0;
        for (int k = 1; k <= Y; ++k) {
            uint32_t w = p1[(s + k) % Y];
            if (k == 1) a = w;
            else a = acc_add(policy == ORC_HOP ? round_wire(a, wire) : a, w, wire);
        }
        v = round_wire(scale_mean(a, wire, op, N), wire);
    }
    store_out(out_elem, dtype, 0, v);
    free(off); free(len); free(p1);
    return ORC_OK;
}

/* ------------------------------------------------------------------------------------ */
/* flat ring all-reduce (baseline)                                      */
/* ------------------------------------------------------------------------------------ */

int orc_ring_allreduce(int R, long long D, int dtype, int wire, int op, int policy, int q,
                       long long round_elems, const void* const* in, void* const* out,
                       orc_counters* ctr)
{
    if (R < 1) return ORC_EGRID;
    if (D < 0 || q < 1 || !in || !out || !valid_types(dtype, wire)) return ORC_EINVAL;
    if (op != ORC_SUM && op != ORC_MEAN) return ORC_EINVAL;
    if (ctr) memset(ctr, 0, sizeof(orc_counters) * (size_t)R);
    if (D == 0) return ORC_OK;
    long long RE = (round_elems > 0 && round_elems < D) ? round_elems : D;
    uint32_t** acc = alloc_acc(R, RE);
    int* grp = (int*)malloc(sizeof(int) * (size_t)R);
    if (!acc || !grp) { free_acc(acc, R); free(grp); return ORC_ENOMEM; }
    for (int p = 0; p < R; ++p) grp[p] = p;
    int rc = ORC_OK;
    for (long long r0 = 0; rc == ORC_OK && r0 < D; r0 += RE) {
        long long n = (D - r0 < RE) ? D - r0 : RE;
        for (int r = 0; r < R; ++r)
            for (long long i = 0; i < n; ++i) acc[r][i] = load_wire(in[r], dtype, wire, r0 + i);
        rc = ring_rs(R, grp, acc, 0, n, q, wire, op, R, policy, 1, ORC_H_RS, ctr);
        if (rc == ORC_OK) rc = ring_ag(R, grp, acc, 0, n, q, ORC_H_AG, ctr);
        for (int r = 0; rc == ORC_OK && r < R; ++r)
            for (long long i = 0; i < n; ++i) store_out(out[r], dtype, r0 + i, acc[r][i]);
    }
    free_acc(acc, R); free(grp);
    return rc;
}

/* ------------------------------------------------------------------------------------ */
/* hierarchical all-reduce [6]                                        */
/* ------------------------------------------------------------------------------------ */

int orc_hier_allreduce(int X, int Y, long long D, int dtype, int wire, int op, int policy,
                       int q, const void* const* in, void* const* out, orc_counters* ctr)
{
    if (X < 1 || Y < 1) return ORC_EGRID;
    if (D < 0 || q < 1 || !in || !out || !valid_types(dtype, wire)) return ORC_EINVAL;
    if (op != ORC_SUM && op != ORC_MEAN) return ORC_EINVAL;
    const int N = X * Y;
    if (ctr) memset(ctr, 0, sizeof(orc_counters) * (size_t)N);
    if (D == 0) return ORC_OK;
    uint32_t** acc = alloc_acc(N, D);
    uint32_t* msg = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)D);
    int* grp = (int*)malloc(sizeof(int) * (size_t)Y);
    if (!acc || !msg || !grp) { free_acc(acc, N); free(msg); free(grp); return ORC_ENOMEM; }
    for (int r = 0; r < N; ++r)
        for (long long i = 0; i < D; ++i) acc[r][i] = load_wire(in[r], dtype, wire, i);
    int rc = ORC_OK;
    /* Phase 1: chain reduce to the leader (column 0) of each row: at step s, column
     * X-1-s sends its full partial to column X-2-s, which adds its own. */
    for (int rho = 0; rho < Y; ++rho) {
        for (int s = 0; s < X - 1; ++s) {
            int src = rho * X + (X - 1 - s), dst = rho * X + (X - 2 - s);
            for (long long i = 0; i < D; ++i)
                msg[i] = (policy == ORC_HOP) ? round_wire(acc[src][i], wire) : acc[src][i];
            for (long long i = 0; i < D; ++i) acc[dst][i] = acc_add(msg[i], acc[dst][i], wire);
            if (ctr) { ctr[src].steps[ORC_H_RS]++; ctr[src].sent[ORC_H_RS] += D; ctr[dst].recv[ORC_H_RS] += D; }
        }
        int lead = rho * X;
        for (long long i = 0; i < D; ++i) {
            uint32_t v = acc[lead][i];
            if (Y == 1) v = scale_mean(v, wire, op, N);
            acc[lead][i] = round_wire(v, wire);
        }
    }
    /* Phase 2: ring all-reduce of the FULL buffer among the Y leaders */
    if (Y > 1) {
        for (int i = 0; i < Y; ++i) grp[i] = i * X;
        rc = ring_rs(Y, grp, acc, 0, D, q, wire, op, N, policy, 1, ORC_V_RS, ctr);
        if (rc == ORC_OK) rc = ring_ag(Y, grp, acc, 0, D, q, ORC_V_AG, ctr);
    }
    /* Phase 3: chain broadcast from the leader: at step s, column s sends to s+1 */
    for (int rho = 0; rc == ORC_OK && rho < Y; ++rho)
        for (int s = 0; s < X - 1; ++s) {
            int src = rho * X + s, dst = rho * X + s + 1;
            memcpy(acc[dst], acc[src], sizeof(uint32_t) * (size_t)D);
            if (ctr) { ctr[src].steps[ORC_H_AG]++; ctr[src].sent[ORC_H_AG] += D; ctr[dst].recv[ORC_H_AG] += D; }
        }
    for (int r = 0; rc == ORC_OK && r < N; ++r)
        for (long long i = 0; i < D; ++i) store_out(out[r], dtype, i, acc[r][i]);
    free_acc(acc, N); free(msg); free(grp);
    return rc;
}

/* ------------------------------------------------------------------------------------ */
/* brute force                                                                          */
/* ------------------------------------------------------------------------------------ */

int orc_brute_sum_f64(int N, long long D, int dtype, int op, const void* const* in, double* out)
{
    if (N < 1 || D < 0 || !in || !out || dtype < ORC_F32 || dtype > ORC_I32) return ORC_EINVAL;
    for (long long i = 0; i < D; ++i) {
        if (dtype == ORC_I32) {
            long long s = 0;
            for (int r = 0; r < N; ++r) s += ((const int32_t*)in[r])[i];
            out[i] = (double)s;
        } else {
            double s = 0.0;
            for (int r = 0; r < N; ++r) {
                double x;
                if (dtype == ORC_F32) x = ((const float*)in[r])[i];
                else if (dtype == ORC_F16) x = orc_f16_to_f32(((const uint16_t*)in[r])[i]);
                else x = orc_bf16_to_f32(((const uint16_t*)in[r])[i]);
                s += x;
            }
            out[i] = s;
        }
        if (op == ORC_MEAN) out[i] /= (double)N;
    }
    return ORC_OK;
}

/* suppress unused warning for type_size in some builds */
size_t orc_type_size(int t) { return type_size(t); }

/* array forms of the conversions (for exhaustive / random-pattern pins) */
void orc_f32_to_f16_array(const float* x, uint16_t* y, long long n)
{ for (long long i = 0; i < n; ++i) y[i] = orc_f32_to_f16(x[i]); }
void orc_f16_to_f32_array(const uint16_t* x, float* y, long long n)
{ for (long long i = 0; i < n; ++i) y[i] = orc_f16_to_f32(x[i]); }
void orc_f32_to_bf16_array(const float* x, uint16_t* y, long long n)
{ for (long long i = 0; i < n; ++i) y[i] = orc_f32_to_bf16(x[i]); }
void orc_bf16_to_f32_array(const uint16_t* x, float* y, long long n)
{ for (long long i = 0; i < n; ++i) y[i] = orc_bf16_to_f32(x[i]); }
