"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle, element by element.

Single GPU: whole X-by-Y grids emulated as virtual ranks (one cooperative launch of the
product kernel, peer pointers aimed at local slabs) -- bit-exact for every dtype under
the oracle's PHASE policy with the library's quantum and round size.
Full size: the 25,557,032-element fp16 mean 2x4 case, sampled outputs vs the oracle's
closed form, plus properties that hold at any size.
"""
import numpy as np
import pytest

import oracle
import synthetic

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TD = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16, "i32": torch.int32}
PAIRS = [("f32", "f32"), ("f16", "f16"), ("bf16", "bf16"), ("i32", "i32"), ("f32", "f16"),
         ("f32", "bf16")]
GRIDS = [(2, 1), (1, 2), (2, 2), (2, 4), (4, 2), (1, 8), (8, 1), (3, 3), (2, 3)]


def from_dev(t, dtype):
    if dtype == "bf16":
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def _np_to_dev(a, dtype):
    if dtype == "bf16":
        return torch.from_numpy(a.view(np.int16).copy()).view(torch.bfloat16).cuda()
    return torch.from_numpy(a.copy()).cuda()


def q_of(wire):
    return 16 // (2 if wire in ("f16", "bf16") else 4)


def _isnan_bits(a):
    if a.dtype == np.uint16:  # bf16 bit patterns
        return ((a & 0x7F80) == 0x7F80) & ((a & 0x7F) != 0)
    if a.dtype in (np.float16, np.float32):
        return np.isnan(a)
    return np.zeros(a.shape, dtype=bool)


def assert_same(got, ref, what):
    """Bit-exact equality; NaNs compare as a class (payloads are not compared, C9)."""
    w = {1: np.uint8, 2: np.uint16, 4: np.uint32}[got.dtype.itemsize]
    gn, rn = _isnan_bits(got), _isnan_bits(ref)
    eq = (got.view(w) == ref.view(w)) | (gn & rn)
    if not eq.all():
        i = int(np.flatnonzero(~eq)[0])
        raise AssertionError(f"{what}: {int((~eq).sum())} mismatches, first at {i}: "
                             f"{got[i]!r} vs {ref[i]!r}")


def run_virtual(vt, ins, dtype, wire, op):
    ts = [_np_to_dev(a, dtype) for a in ins]
    vt.all_reduce(ts, op=op, wire=TD[wire])
    torch.cuda.synchronize()
    assert vt.async_error() == 0
    return [from_dev(t, dtype) for t in ts]


# pull: the default large-message kernel (torus_pull.cu: TMA peer pulls, per-tile flags)
# ldg: the round-1 push kernel (TORUS_KERNEL=push: LDG/STG lock-step wavefront)
# ldgt: the push kernel with 256-vector tiles, so small calls run the multi-tile
# wavefront (stage distance 2) that the auto rule keeps for large slices
# tma: the push kernel's TMA-staged variant
# ll / ll2: the one-shot / two-shot small-message kernels (NEXT-2) forced for every size
# these tests use (ll2: grids with N >= 3; N = 2 falls back to the multi-phase path)
KERNELS = ["ll128", "pull", "ldg", "ldgt", "tma", "ll", "ll2"]
LL_FORCED = 1 << 20  # 1 MiB of wire per rank: covers D = 200,003 f32


def make_vt(X, Y, ws=0, kernel="ll128", ll=None):
    """The kernel is chosen from TORUS_KERNEL / TORUS_LL_MAX_BYTES when the communicator
    is built; the multi-phase variants run with the one-shot path off (ll=0)."""
    import os
    from paper_1811_05233_b200 import VirtualTorus
    env = {"TORUS_KERNEL": {"tma": "tma", "ldg": "push", "ldgt": "push", "pull": "pull"}.get(kernel, "ll128"),
           "TORUS_TILE": "256" if kernel == "ldgt" else "0",
           "TORUS_LL_MAX_BYTES": str(ll if ll is not None else (LL_FORCED if kernel == "ll" else 0)),
           "TORUS_LL2_MAX_BYTES": str(LL_FORCED if kernel == "ll2" else 0)}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        vt = VirtualTorus(X, Y, device=0, ws_bytes=ws)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v
    if kernel == "ll" and not ws:
        assert vt.ll_max_bytes() == LL_FORCED
    elif ll is None:
        assert vt.ll_max_bytes() == 0
    return vt


@pytest.fixture(scope="module")
def vgrids():
    """Virtual grids, built on demand; at most a few stay alive (each holds N slabs)."""
    from collections import OrderedDict
    made = OrderedDict()

    def get(X, Y, ws=0, kernel="ll128"):
        key = (X, Y, ws, kernel)
        if key in made:
            made.move_to_end(key)
        else:
            while len(made) >= 4:
                made.popitem(last=False)[1].destroy()
            made[key] = make_vt(X, Y, ws, kernel)
        return made[key]
    yield get
    for vt in made.values():
        vt.destroy()


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("X,Y", GRIDS)
@pytest.mark.parametrize("dtype,wire", PAIRS)
@pytest.mark.parametrize("op", ["sum", "mean"])
def test_virtual_grid_bit_exact(vgrids, X, Y, dtype, wire, op, kernel):
    vt = vgrids(X, Y, kernel=kernel)
    N = X * Y
    R = vt.round_elems(TD[wire])
    for D in (1, 7, 1000, 4099, 200_003):
        dist = "full" if dtype == "i32" else ("wide" if D < 5000 else "normal")
        ins = synthetic.make_all(dist, D, N, dtype, salt=D % 97)
        got = run_virtual(vt, ins, dtype, wire, op)
        ref = oracle.torus_allreduce(ins, X, Y, dtype, wire=wire, op=op, q=q_of(wire),
                                     round_elems=R)
        for r in range(N):
            assert_same(got[r], ref[r], f"{X}x{Y} {dtype}/{wire} {op} D={D} rank {r}")


@pytest.mark.parametrize("kernel", ["ll128", "pull", "ldg", "ldgt", "tma"])
@pytest.mark.parametrize("X,Y", [(2, 2), (2, 4), (1, 4)])
@pytest.mark.parametrize("dtype,wire", [("f16", "f16"), ("f32", "bf16"), ("i32", "i32")])
def test_multi_round(vgrids, X, Y, dtype, wire, kernel):
    """A slab far smaller than the message forces several rounds."""
    vt = vgrids(X, Y, ws=1 << 20, kernel=kernel)  # 1 MiB slab
    R = vt.round_elems(TD[wire])
    assert 0 < R < 300_000
    D = 3 * R + 12345
    N = X * Y
    ins = synthetic.make_all("full" if dtype == "i32" else "normal", D, N, dtype)
    got = run_virtual(vt, ins, dtype, wire, "mean")
    ref = oracle.torus_allreduce(ins, X, Y, dtype, wire=wire, op="mean", q=q_of(wire), round_elems=R)
    for r in range(N):
        assert_same(got[r], ref[r], f"rounds {X}x{Y} {dtype}/{wire} rank {r}")
    assert vt.launches(D, TD[dtype], TD[wire]) == 4


@pytest.mark.parametrize("kernel", KERNELS)
def test_unaligned_buffers(vgrids, kernel):
    """Buffers offset by one element take the scalar (non-vector) user-buffer path."""
    X, Y, D = 2, 2, 5001
    vt = vgrids(X, Y, kernel=kernel)
    ins = synthetic.make_all("normal", D, 4, "f32")
    ts = []
    for a in ins:
        base = torch.zeros(D + 1, dtype=torch.float32, device="cuda")
        base[1:] = torch.from_numpy(a)
        ts.append(base[1:])
    vt.all_reduce(ts, op="sum", wire=torch.float16)
    torch.cuda.synchronize()
    ref = oracle.torus_allreduce(ins, X, Y, "f32", wire="f16", op="sum", q=8,
                                 round_elems=vt.round_elems(torch.float16))
    for r in range(4):
        assert_same(ts[r].cpu().numpy(), ref[r], f"unaligned rank {r}")


@pytest.mark.parametrize("kernel", KERNELS)
def test_repeated_calls_and_zero_count(vgrids, kernel):
    """Back-to-back calls (epoch flags advance, slots are reused) with varying counts."""
    X, Y = 2, 4
    vt = vgrids(X, Y, kernel=kernel)
    R = vt.round_elems(torch.float16)
    for it, D in enumerate((0, 33, 100_000, 8, 77_777, 1)):
        ins = synthetic.make_all("normal", D, 8, "f16", salt=it)
        got = run_virtual(vt, ins, "f16", "f16", "mean")
        if D == 0:
            continue
        ref = oracle.torus_allreduce(ins, X, Y, "f16", op="mean", q=8, round_elems=R)
        for r in range(8):
            assert_same(got[r], ref[r], f"call {it} D={D} rank {r}")


@pytest.mark.parametrize("kernel", KERNELS)
def test_special_values(vgrids, kernel):
    """inf / nan / subnormal / signed zero go through the same rounding as the oracle."""
    X, Y, D = 2, 2, 64
    vt = vgrids(X, Y, kernel=kernel)
    specials = np.array([np.inf, -np.inf, np.nan, 0.0, -0.0, 1e-45, -1e-45, 6e-8, 65504.0,
                         65520.0, -65536.0, 3.4e38, 1e-38, 5.9e-8, 2.98e-8], dtype=np.float32)
    g = np.random.Generator(np.random.PCG64(5))
    ins = [g.choice(specials, D).astype(np.float32) for _ in range(4)]
    for wire in ("f32", "f16", "bf16"):
        got = run_virtual(vt, ins, "f32", wire, "mean")
        ref = oracle.torus_allreduce(ins, X, Y, "f32", wire=wire, op="mean", q=q_of(wire),
                                     round_elems=vt.round_elems(TD[wire]))
        for r in range(4):
            assert_same(got[r], ref[r], f"specials {wire} rank {r}")


@pytest.mark.parametrize("cs_kernel", ["default", "tma"])
def test_single_rank_cast_scale(cs_kernel, monkeypatch):
    """N = 1 (a7): f32 buffer with f16/bf16 wire -> fused cast round trip; same-type no-op.
    Both kernels: the one-shot castscale_kernel (default) and the TMA ring (TORUS_CS_KERNEL=tma),
    at sizes spanning one partial tile, several tiles and a ragged tail."""
    from paper_1811_05233_b200 import VirtualTorus
    if cs_kernel == "tma":
        monkeypatch.setenv("TORUS_CS_KERNEL", "tma")
    vt = VirtualTorus(1, 1, device=0)
    try:
        want = "castscale_tma_kernel" if cs_kernel == "tma" else "castscale_kernel"
        assert vt.route(1 << 20, torch.float32, torch.float16) == want
        for wire in ("f16", "bf16", "f32"):
            for D in (1, 13, 8195, 1 << 20, 3_000_017):
                x = synthetic.make("wide", D, 0, "f32")
                got = run_virtual(vt, [x], "f32", wire, "mean")[0]
                ref = oracle.torus_allreduce([x], 1, 1, "f32", wire=wire, op="mean")[0]
                assert_same(got, ref, f"N=1 {wire} D={D}")
        assert vt.launches(1000, torch.float32, torch.float32) == 0
        assert vt.launches(1000, torch.float32, torch.float16) == 1
    finally:
        vt.destroy()


def test_allreduce_host_single_rank():
    """torus_allreduce_host at N = 1 (the e2e path of the bench's 1-GPU line): pinned host
    f32 buffer, fp16 / bf16 wire, pieces with a ragged last one -> the cast round trip."""
    from paper_1811_05233_b200 import TorusComm
    comm = TorusComm.init()
    try:
        for wire, D, piece in [("f16", 3_000_017, 1 << 20), ("bf16", 777_777, 0), ("f16", 13, 4)]:
            x = synthetic.make("wide", D, 0, "f32")
            host = torch.from_numpy(x.copy()).pin_memory()
            dev = torch.empty(D, dtype=torch.float32, device="cuda")
            comm.all_reduce_host(host, dev, op="mean", wire=TD[wire], piece=piece)
            torch.cuda.synchronize()
            ref = oracle.torus_allreduce([x], 1, 1, "f32", wire=wire, op="mean")[0]
            assert_same(host.numpy(), ref, f"host N=1 {wire} D={D} piece={piece}")
    finally:
        comm.destroy()


@pytest.mark.parametrize("kernel", ["ll128", "pull", "ldg"])
def test_full_size_resnet50_exhaustive(kernel):
    """BASELINE config 2 at full size, in the bench's launch configuration (2x4 grid,
    fp16, mean, one round): EVERY element of every rank vs the oracle's step-by-step
    simulation of all 8 ranks (orc_torus_allreduce, ~6 s on one core), plus the north-star
    error bound vs the f64 sum with the f16-subnormal reading R13."""
    X, Y, D = 2, 4, synthetic.RESNET50_NUMEL
    vt = make_vt(X, Y, ws=512 << 20, kernel=kernel)
    try:
        R = vt.round_elems(torch.float16)
        assert R >= D, "north-star message must be a single round"
        assert vt.route(D, torch.float16) == {"pull": "torus_pull_kernel", "ldg": "torus_kernel"}.get(
            kernel, "torus_ll128_kernel")
        ins = synthetic.make_all("grad", D, 8, "f16")
        ts = [_np_to_dev(a, "f16") for a in ins]
        vt.all_reduce(ts, op="mean")
        torch.cuda.synchronize()
        assert vt.async_error() == 0
        ref = oracle.torus_allreduce(ins, X, Y, "f16", op="mean", q=8, round_elems=R)
        for r in range(8):
            assert_same(ts[r].cpu().numpy(), ref[r], f"full-size {kernel} rank {r}")
        got = ref[0].astype(np.float64)
        exact = oracle.brute_sum_f64(ins, "f16", "mean")
        mag = sum(np.abs(a.astype(np.float64)) for a in ins) / 8
        # R13: |err| <= 1e-2 * sum|x|/N, with an absolute floor of one binary16 subnormal
        # spacing (2^-24): results below the f16 normal range are quantized to 2^-24
        assert (np.abs(got - exact) <= 1e-2 * mag + 2.0 ** -24).all()
    finally:
        vt.destroy()


@pytest.mark.parametrize("X,Y", [(2, 2), (2, 4), (4, 1)])
def test_small_and_large_calls_interleaved(X, Y):
    """With a 512 KiB threshold, calls alternate between the one-shot kernel and the
    multi-phase kernel; both epochs (LL parity, per-CTA flags) must stay in step,
    and every result equals the oracle's torus fold bit for bit."""
    vt = make_vt(X, Y, ll=512 << 10)
    try:
        assert vt.ll_max_bytes() == 512 << 10
        N, R = X * Y, vt.round_elems(torch.float16)
        sizes = (5, 262_144, 262_145, 1000, 300_000, 8, 9, 131_071, 3)  # f16: 512 KiB = 262,144
        for it, D in enumerate(sizes):
            ins = synthetic.make_all("normal", D, N, "f16", salt=50 + it)
            got = run_virtual(vt, ins, "f16", "f16", "mean" if it % 2 else "sum")
            ref = oracle.torus_allreduce(ins, X, Y, "f16", op="mean" if it % 2 else "sum", q=8,
                                         round_elems=R)
            for r in range(N):
                assert_same(got[r], ref[r], f"interleaved call {it} D={D} rank {r}")
    finally:
        vt.destroy()


@pytest.mark.parametrize("X,Y", [(2, 1), (2, 2), (2, 4)])
def test_default_ll_threshold(X, Y):
    """Default thresholds: one-shot 6 MiB at N = 2, 1.5 MiB / (N-1) (16-byte multiple) at
    N >= 3; two-shot 4 MiB at N >= 3, off at N = 2."""
    import os
    if "TORUS_LL_MAX_BYTES" in os.environ or "TORUS_LL2_MAX_BYTES" in os.environ:
        pytest.skip("threshold overridden in the environment")
    from paper_1811_05233_b200 import VirtualTorus
    vt = VirtualTorus(X, Y, device=0)
    try:
        N = X * Y
        assert vt.ll_max_bytes() == (6 << 20 if N == 2 else ((3 << 19) // (N - 1)) & ~15)
        assert vt.ll2_max_bytes() == (0 if N == 2 else 4 << 20)
    finally:
        vt.destroy()


def test_errors_are_reported():
    from paper_1811_05233_b200 import TorusError, VirtualTorus
    vt = VirtualTorus(2, 2, device=0)
    try:
        t = [torch.zeros(10, dtype=torch.int32, device="cuda") for _ in range(4)]
        with pytest.raises(TorusError, match="UNSUPPORTED"):
            vt.all_reduce(t, wire=torch.float16)       # i32 buffer with a float wire
        t16 = [torch.zeros(10, dtype=torch.float16, device="cuda") for _ in range(4)]
        with pytest.raises(TorusError, match="UNSUPPORTED"):
            vt.all_reduce(t16, wire=torch.float32)     # wire wider than the buffer
    finally:
        vt.destroy()
    with pytest.raises(TorusError, match="GRID"):
        VirtualTorus(5, 5, device=0)                   # > 16 virtual ranks


@pytest.mark.parametrize("N", [2, 3, 4, 8])
@pytest.mark.parametrize("dtype,wire", PAIRS)
@pytest.mark.parametrize("op", ["sum", "mean"])
def test_virtual_ring_baseline_bit_exact(vgrids, N, dtype, wire, op):
    """The flat-ring BASELINE kernel (ref [14]) vs the oracle's ring with
    the HOP policy (every message rounded to the wire type)."""
    vt = vgrids(N, 1)
    R = vt.ring_round_elems(TD[wire])
    for D in (1, 1000, 4099, 100_003):
        ins = synthetic.make_all("full" if dtype == "i32" else "normal", D, N, dtype, salt=D % 7)
        ts = [_np_to_dev(a, dtype) for a in ins]
        vt.ring_all_reduce(ts, op=op, wire=TD[wire])
        torch.cuda.synchronize()
        assert vt.async_error() == 0
        ref = oracle.ring_allreduce(ins, dtype, wire=wire, op=op, policy="hop", q=q_of(wire),
                                    round_elems=R)
        for r in range(N):
            assert_same(from_dev(ts[r], dtype), ref[r], f"ring N={N} {dtype}/{wire} {op} D={D} rank {r}")


def test_ring_multi_round(vgrids):
    vt = vgrids(4, 1, ws=1 << 20)
    R = vt.ring_round_elems(torch.float16)
    D = 2 * R + 999
    ins = synthetic.make_all("normal", D, 4, "f16")
    ts = [_np_to_dev(a, "f16") for a in ins]
    vt.ring_all_reduce(ts, op="mean")
    torch.cuda.synchronize()
    ref = oracle.ring_allreduce(ins, "f16", op="mean", policy="hop", q=8, round_elems=R)
    for r in range(4):
        assert_same(from_dev(ts[r], "f16"), ref[r], f"ring rounds rank {r}")


def test_multi_tensor_single_rank():
    """NEXT-1 at N = 1: pack (f32 -> f16/bf16 RNE) and unpack (exact) around the degenerate
    cast pass equal the oracle on the concatenation."""
    from paper_1811_05233_b200 import TorusComm
    comm = TorusComm.init()
    try:
        sizes = synthetic.resnet50_param_numels()[:30]
        D = sum(sizes)
        x = synthetic.make("wide", D, 0, "f32")
        for wire in ("f16", "bf16", "f32"):
            parts = [p.contiguous() for p in torch.split(torch.from_numpy(x.copy()).cuda(), sizes)]
            comm.all_reduce_multi(parts, op="mean", wire=TD[wire])
            torch.cuda.synchronize()
            got = torch.cat(parts).cpu().numpy()
            ref = oracle.torus_allreduce([x], 1, 1, "f32", wire=wire, op="mean")[0]
            assert_same(got, ref, f"multi N=1 {wire}")
    finally:
        comm.destroy()


@pytest.mark.parametrize("X,Y", [(2, 1), (1, 2), (2, 2), (2, 4), (4, 2), (3, 2)])
@pytest.mark.parametrize("dtype,wire", PAIRS)
@pytest.mark.parametrize("op", ["sum", "mean"])
def test_virtual_hierarchical_baseline_bit_exact(vgrids, X, Y, dtype, wire, op):
    """The hierarchical BASELINE kernel [6] vs the oracle's hierarchical all-reduce (HOP)."""
    vt = vgrids(X, Y)
    N = X * Y
    assert vt.hier_round_elems(TD[wire]) > 100_003
    for D in (1, 999, 4099, 100_003):
        ins = synthetic.make_all("full" if dtype == "i32" else "normal", D, N, dtype, salt=D % 5)
        ts = [_np_to_dev(a, dtype) for a in ins]
        vt.hier_all_reduce(ts, op=op, wire=TD[wire])
        torch.cuda.synchronize()
        assert vt.async_error() == 0
        ref = oracle.hier_allreduce(ins, X, Y, dtype, wire=wire, op=op, policy="hop", q=q_of(wire))
        for r in range(N):
            assert_same(from_dev(ts[r], dtype), ref[r], f"hier {X}x{Y} {dtype}/{wire} {op} D={D} rank {r}")


def test_cuda_graph_capture_and_replay():
    """The call path is CUDA-graph capturable (include/torus.h): no host sync, no
    allocation, epochs device-resident.  Capture one call of each path -- one-shot,
    two-shot, multi-phase -- on a virtual 2x2 grid, then replay the graph with fresh
    inputs; every replay must equal the oracle (the epochs advance on the device)."""
    X, Y, N = 2, 2, 4
    from paper_1811_05233_b200 import VirtualTorus
    vt = VirtualTorus(X, Y, device=0)
    try:
        R = vt.round_elems(torch.float16)
        sizes = (1000, 1_000_000, 5_000_000)  # 2 KB one-shot, 2 MB two-shot, 10 MB multi-phase
        assert 2 * sizes[0] <= vt.ll_max_bytes() < 2 * sizes[1] <= vt.ll2_max_bytes() < 2 * sizes[2]
        bufs = [[torch.zeros(D, dtype=torch.float16, device="cuda") for _ in range(N)] for D in sizes]
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):  # warm-up outside the capture
            for ts in bufs:
                vt.all_reduce(ts, op="mean", stream=s)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for ts in bufs:
                vt.all_reduce(ts, op="mean", stream=s)
        for rep in range(2):
            ins = [synthetic.make_all("normal", D, N, "f16", salt=70 + 3 * rep + k)
                   for k, D in enumerate(sizes)]
            for ts, arrs in zip(bufs, ins):
                for t, a in zip(ts, arrs):
                    t.copy_(torch.from_numpy(a))
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            assert vt.async_error() == 0
            for ts, arrs, D in zip(bufs, ins, sizes):
                ref = oracle.torus_allreduce(arrs, X, Y, "f16", op="mean", q=8, round_elems=R)
                for r in range(N):
                    assert_same(from_dev(ts[r], "f16"), ref[r], f"graph replay {rep} D={D} rank {r}")
    finally:
        vt.destroy()


def _vt_env(X, Y, env, ws=0):
    import os
    from paper_1811_05233_b200 import VirtualTorus
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        return VirtualTorus(X, Y, device=0, ws_bytes=ws)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


PULL_ONLY = {"TORUS_KERNEL": "pull", "TORUS_LL_MAX_BYTES": 0, "TORUS_LL2_MAX_BYTES": 0}


@pytest.mark.parametrize("zc", [0, 1])
@pytest.mark.parametrize("fence", [0, 3])
@pytest.mark.parametrize("X,Y", [(2, 2), (2, 4), (1, 4), (4, 1)])
def test_pull_variants_bit_exact(X, Y, zc, fence):
    """The pull kernel with and without zero-copy (S0 pre-pass copy), with the publishing
    fence in the data CTA (0) or in SIG CTAs (3): bit-exact vs the oracle, several calls
    in a row (parity double-buffering), a ragged length and a multi-tile one."""
    vt = _vt_env(X, Y, {**PULL_ONLY, "TORUS_PULL_ZC": zc, "TORUS_PULL_FENCE": fence})
    try:
        N = X * Y
        for it, (dt, D) in enumerate((("f16", 300_007), ("f32", 123_457), ("bf16", 1_000_003), ("f16", 8))):
            ins = synthetic.make_all("normal", D, N, dt, salt=20 + it)
            got = run_virtual(vt, ins, dt, dt, "mean")
            ref = oracle.torus_allreduce(ins, X, Y, dt, op="mean", q=q_of(dt), round_elems=vt.round_elems(TD[dt]))
            for r in range(N):
                assert_same(got[r], ref[r], f"pull zc={zc} fence={fence} {X}x{Y} {dt} D={D} rank {r}")
    finally:
        vt.destroy()


def test_pull_random_start_delays_bit_exact():
    """random per-rank (here per-CTA, up to 50 us) start delays leave the
    result unchanged -- the flag protocol, not timing, orders every hand-off."""
    X, Y = 2, 4
    vt = _vt_env(X, Y, {**PULL_ONLY, "TORUS_DELAY_NS": 50_000})
    try:
        for it in range(3):
            ins = synthetic.make_all("wide", 400_009, 8, "f32", salt=40 + it)
            got = run_virtual(vt, ins, "f32", "f32", "sum")
            ref = oracle.torus_allreduce(ins, X, Y, "f32", op="sum", q=4, round_elems=vt.round_elems(torch.float32))
            for r in range(8):
                assert_same(got[r], ref[r], f"delayed call {it} rank {r}")
    finally:
        vt.destroy()


@pytest.mark.parametrize("fault", [1, 2])
def test_fault_injection_is_caught(fault):
    """SPEC.md:509 negative control: with one reduced element corrupted (1) or one P1 wait
    skipped so a peer's slot is read before it is written (2), parity vs the oracle FAILS
    -- the parity tests have teeth.  Without injection the same calls are bit-exact."""
    X, Y, D = 2, 2, 600_000
    bad_calls = 0
    vt = _vt_env(X, Y, {**PULL_ONLY, "TORUS_FAULT": fault})
    try:
        for it in range(3):
            ins = synthetic.make_all("normal", D, 4, "f16", salt=60 + it)
            got = run_virtual(vt, ins, "f16", "f16", "sum")
            ref = oracle.torus_allreduce(ins, X, Y, "f16", op="sum", q=8, round_elems=vt.round_elems(torch.float16))
            if any(not np.array_equal(got[r].view(np.uint16), ref[r].view(np.uint16)) for r in range(4)):
                bad_calls += 1
    finally:
        vt.destroy()
    assert bad_calls >= 1, "fault injection went undetected"


def test_header_check_consistent_calls():
    """TORUS_CHECK=1: the per-call header agrees on consistent calls (no false MISMATCH)."""
    vt = _vt_env(2, 2, {**PULL_ONLY, "TORUS_CHECK": 1})
    try:
        for D in (1000, 300_000, 7):
            ins = synthetic.make_all("normal", D, 4, "f16", salt=D % 11)
            got = run_virtual(vt, ins, "f16", "f16", "mean")
            ref = oracle.torus_allreduce(ins, 2, 2, "f16", op="mean", q=8, round_elems=vt.round_elems(torch.float16))
            for r in range(4):
                assert_same(got[r], ref[r], f"checked D={D} rank {r}")
        assert vt.async_error() == 0
    finally:
        vt.destroy()


@pytest.mark.parametrize("X,Y", [(2, 2), (2, 4), (1, 2)])
@pytest.mark.parametrize("dtype,wire", [("f32", "f16"), ("f32", "bf16"), ("f16", "f16")])
def test_fused_multi_tensor_bucket(X, Y, dtype, wire):
    """NEXT-1 fused: a ResNet-50 gradient bucket (132 tensors in
    backprop order) reduced in ONE multi-phase launch that reads the tensors with the cast
    fused and writes them back with the up-cast fused; equal, bit for bit, to the oracle's
    all-reduce of the concatenation.  A second bucket with sizes that are not multiples of
    the 16-byte quantum exercises the vectors that straddle tensor boundaries."""
    sizes = synthetic.resnet50_param_numels()[::-1][29:161]  # DDP's third bucket shape
    odd = [1, 7, 8, 1000, 12_345, 3, 70_001, 9, 16, 33]
    vt = _vt_env(X, Y, {"TORUS_LL_MAX_BYTES": 0, "TORUS_LL2_MAX_BYTES": 0})
    try:
        N = X * Y
        for k, sz in enumerate((sizes, odd)):
            D = sum(sz)
            ins = synthetic.make_all("grad" if dtype == "f16" else "normal", D, N, dtype, salt=80 + k)
            buckets = [list(torch.split(_np_to_dev(a, dtype), sz)) for a in ins]
            buckets = [[t.contiguous() for t in b] for b in buckets]
            assert vt.route(D, TD[dtype], TD[wire]) in ("torus_kernel", "torus_ll128_kernel")
            vt.all_reduce_multi(buckets, op="mean", wire=TD[wire])
            torch.cuda.synchronize()
            assert vt.async_error() == 0
            ref = oracle.torus_allreduce(ins, X, Y, dtype, wire=wire, op="mean", q=q_of(wire),
                                         round_elems=vt.round_elems(TD[wire]))
            for r in range(N):
                got = from_dev(torch.cat(buckets[r]), dtype)
                assert_same(got, ref[r], f"fused bucket {k} {X}x{Y} {dtype}/{wire} rank {r}")
    finally:
        vt.destroy()
