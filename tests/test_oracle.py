"""Pins for the CPU oracle (oracle/torus_oracle.c) -- nothing here touches the GPU path.

Each test pins the oracle to something other than itself (SURVEY.md Sec. 8(c) "What pins
each part"): worked examples printed in SPEC.md, hand-derived fold-order values,
closed forms from the paper (PAPER.md:70 step counts and volumes), brute force, library
conversions (numpy / torch RNE casts), and invariants.
"""
import json
import os

import numpy as np
import pytest

import oracle
import synthetic

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


GRIDS = [(1, 1), (2, 1), (1, 2), (2, 2), (2, 4), (4, 2), (1, 8), (8, 1), (3, 3), (2, 3), (3, 2)]


# --------------------------------------------------------------------------------------
# SPEC worked examples (tests/golden/spec_examples.json)
# --------------------------------------------------------------------------------------

def test_partition_spec_examples():
    for ex in _gold("spec_examples.json")["partition"]:
        off, ln = oracle.qpart(ex["n"], ex["parts"], 1)
        assert ln == ex["len"], ex["cite"]
        assert off == list(np.concatenate([[0], np.cumsum(ex["len"])[:-1]])), ex["cite"]


@pytest.mark.parametrize("n", [0, 1, 7, 8, 9, 63, 64, 65, 1000, 25_557_032])
@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("q", [1, 4, 8])
def test_partition_properties(n, parts, q):
    """C3: contiguous cover of [0,n); every boundary except the end is a multiple of q;
    quanta counts differ by at most one, larger first."""
    off, ln = oracle.qpart(n, parts, q)
    assert sum(ln) == n
    pos = 0
    for o, l in zip(off, ln):
        assert o == pos and l >= 0
        pos += l
    for o in off:
        assert o % q == 0 or o == n
    quanta = [(l + q - 1) // q for l in ln]
    nz = [k for k in quanta]
    assert max(nz) - min(nz) <= 1 or n % q != 0
    assert all(a >= b for a, b in zip(quanta, quanta[1:])) or n % q != 0


def test_torus_spec_2x2_example():
    for ex in _gold("spec_examples.json")["torus"]:
        ins = synthetic.make_all("rank", ex["D"], ex["x"] * ex["y"], ex["dtype"])
        outs = oracle.torus_allreduce(ins, ex["x"], ex["y"], ex["dtype"])
        for o in outs:
            assert (o == ex["expect_all"]).all(), ex["cite"]


def test_ring_spec_examples():
    for ex in _gold("spec_examples.json")["ring_rs_ag"]:
        ins = [np.array(v, dtype=np.int32) for v in ex["inputs"]]
        outs = oracle.ring_allreduce(ins, "i32")
        if "expect" in ex:
            for o, e in zip(outs, ex["expect"]):
                assert o.tolist() == e, ex["cite"]
        else:
            for o in outs:
                assert (o == ex["expect_all"]).all(), ex["cite"]


def test_mixed_precision_example():
    """f16 wire with f32 accumulation keeps precision that f16 accumulation
    (HOP policy) loses."""
    for ex in _gold("spec_examples.json")["mixed_precision"]:
        ins = [np.array([v], dtype=np.float32) for v in ex["inputs"]]
        for pol in ("phase", "hop"):
            outs = oracle.ring_allreduce(ins, "f32", wire=ex["wire"], policy=pol)
            for o in outs:
                assert o[0] == ex[pol], (pol, ex["cite"])
            # the torus with Y=1 is the same ring (SURVEY 8(c) degenerate grids)
            t = oracle.torus_allreduce(ins, ex["ring"], 1, "f32", wire=ex["wire"], policy=pol)
            assert all(o[0] == ex[pol] for o in t)


def test_step_counts_spec_and_table4():
    """torus = 2(X-1) horizontal GPU-to-GPU operations, ring = 2(N-1); the
    vertical ring adds 2(Y-1).  Grids from Table 4."""
    g = _gold("spec_examples.json")["steps"]
    ring4 = g[0]
    _, ctr = oracle.ring_allreduce([np.zeros(4, np.float32)] * ring4["n"], "f32", counters=True)
    assert all(c["steps"]["h_rs"] + c["steps"]["h_ag"] == ring4["steps"] for c in ctr), ring4["cite"]
    grids = [(32, 32)] + [(r["horizontal"], r["vertical"]) for r in _gold("table4_grids.json")["rows"]]
    for X, Y in grids:
        N = X * Y
        ins = [np.zeros(1, np.int32)] * N
        _, ctr = oracle.torus_allreduce(ins, X, Y, "i32", counters=True)
        for c in ctr[:3] + ctr[-3:]:
            assert c["steps"]["h_rs"] + c["steps"]["h_ag"] == 2 * (X - 1)
            assert c["steps"]["v_rs"] + c["steps"]["v_ag"] == 2 * (Y - 1)
        if (X, Y) == (32, 32):
            assert 2 * (X - 1) == g[1]["horizontal_steps"] and 2 * (N - 1) == g[1]["ring_steps"]
    # ring over the same N takes 2(N-1) steps (checked on N=1024 explicitly)
    _, ctr = oracle.ring_allreduce([np.zeros(1, np.int32)] * 1024, "i32", counters=True)
    assert ctr[5]["steps"]["h_rs"] + ctr[5]["steps"]["h_ag"] == 2046


# --------------------------------------------------------------------------------------
# fold-order pins (tests/golden/fold_order.json)
# --------------------------------------------------------------------------------------

def test_fold_order_2x4():
    ex = _gold("fold_order.json")["cases"][0]
    X, Y, D = ex["x"], ex["y"], ex["D"]
    T = np.array(ex["T"], dtype=np.float32)
    ins = [np.array([T[(2 * r + 4 * i) % 8] for i in range(D)], dtype=np.float32)
           for r in range(X * Y)]
    outs = oracle.torus_allreduce(ins, X, Y, "f32", q=ex["q"])
    for o in outs:
        assert (o == np.float32(ex["torus"])).all(), ex["cite"]
    el = oracle.torus_elements(ins, X, Y, range(D), "f32", q=ex["q"])
    assert (el == np.float32(ex["torus"])).all()
    # the alternatives the golden file lists really differ
    naive = np.float32(0)
    for r in range(X * Y):
        naive = np.float32(naive + ins[r][0])
    assert naive == np.float32(ex["naive_rank_order"])
    assert ex["exact_sum"] == sum(float(ins[r][0]) for r in range(X * Y))
    assert len({ex["torus"], ex["exact_sum"], ex["naive_rank_order"], ex["spec_literal_owner"]}) == 4


def test_fold_order_2x2():
    ex = _gold("fold_order.json")["cases"][1]
    ins = [np.array([v], dtype=np.float32) for v in ex["w"]]
    outs = oracle.torus_allreduce(ins, ex["x"], ex["y"], "f32", q=ex["q"])
    assert all(o[0] == ex["torus"] for o in outs), ex["cite"]
    assert float(oracle.brute_sum_f64(ins, "f32")[0]) == ex["exact_sum"]


# --------------------------------------------------------------------------------------
# brute force (exact for i32; within the summation bound for floats)
# --------------------------------------------------------------------------------------

@pytest.mark.parametrize("X,Y", GRIDS)
def test_i32_matches_brute_force(X, Y):
    N, D = X * Y, 1037
    for dist in ("full", "small"):
        ins = synthetic.make_all(dist, D, N, "i32")
        exact = np.zeros(D, dtype=np.int64)
        for a in ins:
            exact += a
        exact = (exact & 0xFFFFFFFF).astype(np.uint32).view(np.int32)  # two's-complement wrap
        for q in (1, 4):
            outs = oracle.torus_allreduce(ins, X, Y, "i32", q=q)
            for o in outs:
                np.testing.assert_array_equal(o, exact)


@pytest.mark.parametrize("X,Y", [(2, 2), (2, 4), (4, 2), (1, 8), (8, 1), (3, 3)])
def test_i32_routing_and_ramp_pins(X, Y):
    """onehot: every rank counted exactly once gives 2^N-1; ramp: D*N(N-1)/2 + N*i."""
    N, D = X * Y, 777
    outs = oracle.torus_allreduce(synthetic.make_all("onehot", D, N, "i32"), X, Y, "i32", q=4)
    for o in outs:
        assert (o == (1 << N) - 1).all()
    outs = oracle.torus_allreduce(synthetic.make_all("ramp", D, N, "i32"), X, Y, "i32", q=4)
    expect = D * N * (N - 1) // 2 + N * np.arange(D, dtype=np.int64)
    for o in outs:
        np.testing.assert_array_equal(o.astype(np.int64), expect)


def test_i32_mean_truncates_toward_zero():
    """SURVEY C10 reading: i32 mean = wrapped sum / N, C truncation."""
    ins = [np.array([-7, 7, 5, -1], dtype=np.int32), np.array([0, 0, 0, 0], dtype=np.int32),
           np.array([0, 0, 0, 0], dtype=np.int32), np.array([0, 1, 0, -2], dtype=np.int32)]
    outs = oracle.torus_allreduce(ins, 2, 2, "i32", op="mean")
    for o in outs:
        assert o.tolist() == [-1, 2, 1, 0]


@pytest.mark.parametrize("X,Y", GRIDS)
@pytest.mark.parametrize("dtype,wire", [("f32", "f32"), ("f16", "f16"), ("bf16", "bf16"),
                                        ("f32", "f16"), ("f32", "bf16")])
@pytest.mark.parametrize("op", ["sum", "mean"])
def test_float_within_bound_of_f64(X, Y, dtype, wire, op):
    """|torus - exact| <= bound * sum|x|.  f32: (N+1)*2^-24 (recursive
    summation bound + the mean scale); f16: 4 roundings of 2^-11 plus the f32 adds, with an
    absolute floor for binary16 subnormals; bf16: the north-star 1e-2 bar."""
    N, D = X * Y, 1000
    for dist in ("uniform", "normal", "wide"):
        ins = synthetic.make_all(dist, D, N, dtype)
        outs = oracle.torus_allreduce(ins, X, Y, dtype, wire=wire, op=op, q=8 if wire != "f32" else 4)
        ref = oracle.brute_sum_f64(ins, dtype, op)
        mag = sum(np.abs(synthetic.as_float64(a, dtype)) for a in ins)
        if op == "mean":
            mag = mag / N
        if wire == "f32":
            bound = (N + 1) * 2.0 ** -24
        elif wire == "f16":
            bound = 4 * 2.0 ** -11 + N * 2.0 ** -24
        else:
            bound = 1e-2
        # absolute floor: binary16 subnormal spacing 2^-24 (each of <= 3 roundings per value)
        floor = 3 * N * 2.0 ** -25 if wire == "f16" else 1e-30
        for o in outs:
            err = np.abs(synthetic.as_float64(o, dtype) - ref)
            assert (err <= bound * mag + floor).all(), (dist, float((err / np.maximum(mag, 1e-30)).max()))


# --------------------------------------------------------------------------------------
# simulation vs closed form, degenerate grids, invariants
# --------------------------------------------------------------------------------------

@pytest.mark.parametrize("X,Y", GRIDS)
@pytest.mark.parametrize("dtype,wire", [("f32", "f32"), ("f16", "f16"), ("bf16", "bf16"),
                                        ("f32", "f16"), ("i32", "i32")])
@pytest.mark.parametrize("policy", ["phase", "hop"])
def test_simulation_equals_closed_form(X, Y, dtype, wire, policy):
    """C5: the ring simulation and the per-element fold agree bit for bit, including
    multi-round calls (C13) and a ragged tail."""
    N = X * Y
    for D, q, R in ((1, 1, 0), (7, 1, 0), (64, 4, 0), (203, 8, 0), (203, 8, 48)):
        ins = synthetic.make_all("full" if dtype == "i32" else "wide", D, N, dtype)
        outs = oracle.torus_allreduce(ins, X, Y, dtype, wire=wire, op="mean", policy=policy, q=q,
                                      round_elems=R)
        el = oracle.torus_elements(ins, X, Y, range(D), dtype, wire=wire, op="mean",
                                   policy=policy, q=q, round_elems=R)
        for o in outs:
            np.testing.assert_array_equal(o.view(np.uint8), el.view(np.uint8))


@pytest.mark.parametrize("N", [2, 3, 4, 8])
@pytest.mark.parametrize("dtype,wire", [("f32", "f32"), ("f16", "f16"), ("f32", "bf16")])
def test_degenerate_grids_equal_ring(N, dtype, wire):
    """1xN == Nx1 == ring(N), bit-exact."""
    ins = synthetic.make_all("wide", 517, N, dtype)
    a = oracle.torus_allreduce(ins, 1, N, dtype, wire=wire, op="mean", q=8)
    b = oracle.torus_allreduce(ins, N, 1, dtype, wire=wire, op="mean", q=8)
    c = oracle.ring_allreduce(ins, dtype, wire=wire, op="mean", q=8)
    for x, y, z in zip(a, b, c):
        np.testing.assert_array_equal(x.view(np.uint8), y.view(np.uint8))
        np.testing.assert_array_equal(x.view(np.uint8), z.view(np.uint8))


def test_single_rank_is_cast_only():
    """N=1: out = from_wire(to_wire(in)) (a7)."""
    x = synthetic.make("wide", 1000, 0, "f32")
    out = oracle.torus_allreduce([x], 1, 1, "f32", wire="f16", op="mean")[0]
    np.testing.assert_array_equal(out, x.astype(np.float16).astype(np.float32))
    out = oracle.torus_allreduce([x], 1, 1, "f32", op="sum")[0]
    np.testing.assert_array_equal(out, x)


@pytest.mark.parametrize("X,Y", [(2, 2), (2, 4), (3, 2)])
def test_invariants(X, Y):
    N, D = X * Y, 333
    ins = synthetic.make_all("wide", D, N, "f32")
    outs = oracle.torus_allreduce(ins, X, Y, "f32", q=4)
    for o in outs[1:]:
        np.testing.assert_array_equal(o, outs[0])                      # identical on every rank
    again = oracle.torus_allreduce(ins, X, Y, "f32", q=4)
    np.testing.assert_array_equal(again[0], outs[0])                   # deterministic
    z = oracle.torus_allreduce([np.zeros(D, np.float32)] * N, X, Y, "f32")
    assert all((o == 0).all() for o in z)                              # zero in -> zero out
    sc = oracle.torus_allreduce([a * np.float32(8.0) for a in ins], X, Y, "f32", q=4)
    np.testing.assert_array_equal(sc[0], outs[0] * np.float32(8.0))    # 2^k scaling commutes


@pytest.mark.parametrize("X,Y", [(2, 2), (2, 4), (4, 2), (3, 3), (1, 8), (8, 1)])
@pytest.mark.parametrize("D", [64, 1000, 1001])
def test_phase_volumes_closed_form(X, Y, D):
    """Per-group totals (exact for any D) and per-rank means (the north star's
    (X-1)/X*D, 2(Y-1)/Y*D/X, (X-1)/X*D)."""
    N = X * Y
    _, ctr = oracle.torus_allreduce([np.zeros(D, np.int32)] * N, X, Y, "i32", counters=True)
    coff, clen = oracle.qpart(D, X, 1)
    for rho in range(Y):
        row = ctr[rho * X:(rho + 1) * X]
        assert sum(c["sent"]["h_rs"] for c in row) == (X - 1) * D
        assert sum(c["sent"]["h_ag"] for c in row) == (X - 1) * D
        for col, c in enumerate(row):
            assert c["sent"]["h_rs"] == D - clen[col]                       # a2
    for col in range(X):
        colr = [ctr[i * X + col] for i in range(Y)]
        assert sum(c["sent"]["v_rs"] for c in colr) == (Y - 1) * clen[col]
        assert sum(c["sent"]["v_ag"] for c in colr) == (Y - 1) * clen[col]
    tot = {p: sum(c["sent"][p] for c in ctr) for p in oracle.PHASES}
    assert tot["h_rs"] / N == pytest.approx((X - 1) / X * D)
    assert (tot["v_rs"] + tot["v_ag"]) / N == pytest.approx(2 * (Y - 1) / Y * D / X)
    assert tot["h_ag"] / N == pytest.approx((X - 1) / X * D)
    # bandwidth-optimal total: 2(N-1)/N * D per rank (SURVEY 8(a) derivation)
    assert sum(tot.values()) / N == pytest.approx(2 * (N - 1) / N * D)
    for p in oracle.PHASES:                                                  # conservation
        assert sum(c["sent"][p] for c in ctr) == sum(c["recv"][p] for c in ctr)


def test_hierarchical_same_ops_x_times_more_vertical_data():
    """hierarchical does the same number of GPU-to-GPU operations, but the
    torus's vertical step handles X times less data per rank."""
    X, Y, D = 4, 2, 4096
    ins = synthetic.make_all("small", D, X * Y, "i32")
    h, hc = oracle.hier_allreduce(ins, X, Y, "i32", counters=True)
    t, tc = oracle.torus_allreduce(ins, X, Y, "i32", counters=True)
    for a, b in zip(h, t):
        np.testing.assert_array_equal(a, b)
    lead = hc[0]
    # the chain reduce and chain broadcast of one row take X-1 sequential sends each
    row = hc[:X]
    horiz_h = sum(c["steps"]["h_rs"] for c in row) + sum(c["steps"]["h_ag"] for c in row)
    assert horiz_h == 2 * (X - 1) == tc[0]["steps"]["h_rs"] + tc[0]["steps"]["h_ag"]
    v_h = lead["sent"]["v_rs"] + lead["sent"]["v_ag"]
    v_t = tc[0]["sent"]["v_rs"] + tc[0]["sent"]["v_ag"]
    assert v_h == X * v_t


def test_hierarchical_float_chain_order():
    """DESIGN R14: the hierarchical baseline's chain reduce runs from the highest column to
    the leader (column 0), so a row's sum is ((w[X-1] + w[X-2]) + ...) + w[0].  Hand-derived
    f32 pin, X=3, Y=1, one element: inputs [2^24, 1, 1] (columns 0, 1, 2): the chain gives
    (1 + 1) + 2^24 = 16777218 exactly; the opposite order would give (2^24 + 1) + 1 ->
    16777216 (2^24 + 1 ties to even).  And with an f16 wire every hop is rounded (HOP,
    SURVEY C7): inputs [2048, 1, 1] give (1 + 1) + 2048 = 2050, representable in binary16."""
    ins = [np.array([v], dtype=np.float32) for v in (2.0 ** 24, 1.0, 1.0)]
    out = oracle.hier_allreduce(ins, 3, 1, "f32", op="sum", policy="hop")
    assert all(o[0] == np.float32(16777218.0) for o in out)
    ins16 = [np.array([v], dtype=np.float16) for v in (2048.0, 1.0, 1.0)]
    out16 = oracle.hier_allreduce(ins16, 3, 1, "f16", op="sum", policy="hop")
    assert all(o[0] == np.float16(2050.0) for o in out16)
    # the torus on the same row folds c+1, ..., c: chunk owner 0 sums 1 + 1 + 2^24 as well
    t = oracle.torus_allreduce(ins, 3, 1, "f32", op="sum")
    assert all(o[0] == np.float32(16777218.0) for o in t)


def test_mixed_precision_phase_not_worse_than_hop():
    """over random trials (U[0,1), N=16, D=256) the mean abs error of
    f16 wire + f32 accumulation is <= that of f16 accumulation."""
    pe, he = [], []
    for t in range(100):
        ins = synthetic.make_all("uniform", 256, 16, "f32", salt=t + 1)
        ref = oracle.brute_sum_f64(ins, "f32")
        p = oracle.ring_allreduce(ins, "f32", wire="f16", policy="phase")[0]
        h = oracle.ring_allreduce(ins, "f32", wire="f16", policy="hop")[0]
        pe.append(np.abs(p - ref).mean())
        he.append(np.abs(h - ref).mean())
    assert np.mean(pe) <= np.mean(he)


# --------------------------------------------------------------------------------------
# conversions (C9) against library routines
# --------------------------------------------------------------------------------------

def test_f16_exhaustive_against_numpy():
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    f = oracle.f16_to_f32_array(bits)
    ref = bits.view(np.float16).astype(np.float32)
    nan = np.isnan(ref)
    assert (np.isnan(f) == nan).all()
    np.testing.assert_array_equal(f[~nan].view(np.uint32), ref[~nan].view(np.uint32))
    back = oracle.f32_to_f16_array(f)
    np.testing.assert_array_equal(back[~nan], bits[~nan])


def test_f32_to_f16_random_patterns_against_numpy():
    g = np.random.Generator(np.random.PCG64(7))
    pats = g.integers(0, 2 ** 32, size=2_000_000, dtype=np.uint64).astype(np.uint32)
    # concentrate half the draws near the binary16 range, incl. subnormals and ties
    pats[::2] = (pats[::2] & 0x807FFFFF) | ((g.integers(100, 145, size=pats[::2].size) << 23)
                                            .astype(np.uint32))
    x = pats.view(np.float32)
    mine = oracle.f32_to_f16_array(x)
    with np.errstate(over="ignore"):
        ref = x.astype(np.float16).view(np.uint16)
    nan = np.isnan(x)
    np.testing.assert_array_equal(mine[~nan], ref[~nan])
    assert (np.isnan(mine.view(np.float16)[nan])).all()


def test_bf16_against_torch():
    torch = pytest.importorskip("torch")
    g = np.random.Generator(np.random.PCG64(11))
    pats = g.integers(0, 2 ** 32, size=2_000_000, dtype=np.uint64).astype(np.uint32)
    x = pats.view(np.float32)
    mine = oracle.f32_to_bf16_array(x)
    ref = torch.from_numpy(x.copy()).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    nan = np.isnan(x)
    np.testing.assert_array_equal(mine[~nan], ref[~nan])
    assert (((mine[nan] & 0x7F80) == 0x7F80) & ((mine[nan] & 0x7F) != 0)).all()
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    f = oracle.bf16_to_f32_array(bits)
    tref = torch.from_numpy(bits.view(np.int16).copy()).view(torch.bfloat16).float().numpy()
    np.testing.assert_array_equal(f.view(np.uint32), tref.view(np.uint32))
