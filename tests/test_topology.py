"""The topology layer's alpha-beta cost model (torus_predict_time / torus_pick_grid_model;
north_star (3), SPEC.md:303-311 predict_time), CPU only.

Pins: SPEC's worked example, the bandwidth-only and latency-only limits (closed forms),
the paper's step counts (2(X-1) vs 2(N-1), Table 4 grids), the torus < ring property for
any alpha > 0, monotonicity, the hierarchical all-reduce's
X-times-larger vertical data, and grid choices on synthetic link matrices."""
import itertools
import json
import os

import pytest

from paper_1811_05233_b200 import _lib, pick_grid, pick_grid_model, predict_time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INF = 1e12  # GB/s: "beta -> infinity"


def test_spec_ring_example():
    """ring N=4, D=4 B, alpha=1 s, beta=1 B/s -> 6 x (1 + 1) = 12 s."""
    us = predict_time(4, 1, 4.0, 1e6, beta_gbs=1e-9, algo="ring")
    assert us == pytest.approx(12e6)


@pytest.mark.parametrize("X,Y", [(2, 4), (4, 2), (1, 8), (8, 1), (2, 2), (3, 5), (32, 32)])
def test_bandwidth_only_limit(X, Y):
    """alpha = 0: the ring-phase schedule moves 2(N-1)/N * S bytes per rank."""
    S, beta = 51_114_064.0, 500.0
    N = X * Y
    us = predict_time(X, Y, S, 0.0, beta_gbs=beta, schedule="ring")
    assert us == pytest.approx(2 * (N - 1) / N * S / (beta * 1e9) * 1e6, rel=1e-12)
    # the one-shot schedule moves the same bytes
    assert predict_time(X, Y, S, 0.0, beta_gbs=beta) == pytest.approx(us, rel=1e-12)


def test_latency_only_limit_table4():
    """beta -> inf: alpha x steps; 2(X-1) + 2(Y-1) for the torus, 2(N-1) for the ring
    (PAPER.md:70).  Table 4 grids from tests/golden/table4_grids.json."""
    rows = json.load(open(os.path.join(ROOT, "tests", "golden", "table4_grids.json")))["rows"]
    for g in rows:
        X, Y = g["horizontal"], g["vertical"]
        torus = predict_time(X, Y, 1.0, 1.0, beta_gbs=INF, schedule="ring")
        ring = predict_time(X * Y, 1, 1.0, 1.0, beta_gbs=INF, algo="ring")
        assert torus == pytest.approx(2 * (X - 1) + 2 * (Y - 1), abs=1e-6)
        assert ring == pytest.approx(2 * (X * Y - 1), abs=1e-6)
    assert predict_time(32, 32, 1.0, 1.0, beta_gbs=INF, schedule="ring") == pytest.approx(124, abs=1e-6)


@pytest.mark.parametrize("X,Y", [(2, 2), (2, 4), (4, 4), (32, 32), (72, 48)])
@pytest.mark.parametrize("alpha", [1e-3, 1.0, 100.0])
def test_torus_beats_ring_for_any_alpha(X, Y, alpha):
    """alpha > 0, X, Y >= 2, fixed D: torus < ring."""
    for S in (1e3, 1e6, 1e9):
        t = predict_time(X, Y, S, alpha, beta_gbs=100.0, schedule="ring")
        r = predict_time(X * Y, 1, S, alpha, beta_gbs=100.0, algo="ring")
        assert t < r


def test_monotone_in_alpha_and_inverse_beta():
    """SPEC.md:327."""
    prev = None
    for a in (0.0, 0.5, 1, 2, 8, 64):
        t = predict_time(2, 4, 5e7, a, beta_gbs=300)
        assert prev is None or t >= prev
        prev = t
    prev = None
    for b in (1000, 500, 100, 10, 1):
        t = predict_time(2, 4, 5e7, 2.0, beta_gbs=b)
        assert prev is None or t >= prev
        prev = t


def test_hierarchical_vertical_data_is_x_times_larger():
    """same number of GPU-to-GPU operations, X times more vertical data."""
    S, X, Y = 1e9, 4, 2
    # isolate the vertical term: horizontal links infinitely fast, alpha 0
    bw = [[INF if i // X == j // X else 10.0 for j in range(X * Y)] for i in range(X * Y)]
    torus = predict_time(X, Y, S, 0.0, bw=bw, schedule="ring")
    hier = predict_time(X, Y, S, 0.0, bw=bw, algo="hier")
    assert hier / torus == pytest.approx(X, rel=1e-9)
    t_steps = predict_time(X, Y, 1.0, 1.0, beta_gbs=INF, schedule="ring")
    h_steps = predict_time(X, Y, 1.0, 1.0, beta_gbs=INF, algo="hier")
    assert t_steps == pytest.approx(h_steps)  # same GPU-to-GPU operation count


def _islands(n, per, fast, slow):
    return [[fast if i // per == j // per else slow for j in range(n)] for i in range(n)]


def test_pick_uniform_domain_prefers_fewest_handoffs():
    """One NVSwitch domain: every grid moves 2(N-1)/N*S; the widest grid has 2 hand-offs."""
    for n in (2, 4, 8):
        X, Y, _ = pick_grid_model(n, 51_114_064, 4.0, beta_gbs=560)
        assert (X, Y) == (n, 1)


def test_pick_two_islands_puts_rows_inside_islands():
    bw = _islands(8, 4, 560.0, 25.0)
    assert pick_grid_model(8, 51_114_064, 4.0, bw=bw)[:2] == (4, 2)
    bw = _islands(8, 2, 560.0, 25.0)
    assert pick_grid_model(8, 51_114_064, 4.0, bw=bw)[:2] == (2, 4)


def test_pick_depends_on_message_size():
    """Islands joined by a moderately slower fabric: small messages are latency-bound (the
    flat grid's 2 hand-offs win), large ones bandwidth-bound (rows inside the islands)."""
    bw = _islands(8, 4, 560.0, 150.0)
    small = pick_grid_model(8, 4096, 20.0, bw=bw)[:2]
    large = pick_grid_model(8, 1e9, 20.0, bw=bw)[:2]
    assert small == (8, 1)
    assert large == (4, 2)
    # and the choice is the argmin of the per-grid predictions
    for S in (4096, 1e6, 1e9):
        X, Y, best = pick_grid_model(8, S, 20.0, bw=bw)
        for x in (1, 2, 4, 8):
            assert predict_time(x, 8 // x, S, 20.0, bw=bw) >= best * (1 - 1e-12)


def test_infeasible_grid_is_an_error():
    bw = [[560.0, 0.0], [0.0, 560.0]]
    with pytest.raises(_lib.TorusError, match="GRID"):
        predict_time(2, 1, 1e6, 1.0, bw=bw)
    with pytest.raises(_lib.TorusError, match="GRID"):
        pick_grid_model(2, 1e6, 1.0, bw=bw)


def test_bad_arguments():
    with pytest.raises(_lib.TorusError, match="INVALID"):
        predict_time(0, 1, 1.0, 1.0)
    with pytest.raises(_lib.TorusError, match="INVALID"):
        predict_time(2, 2, 1.0, -1.0)
