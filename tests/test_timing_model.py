"""Pins for the P:573-574 cost model and the two-stream simulation (CPU)."""
import itertools
import json
import os

import pytest

from oracle import default_cost, simulate, subpipelined_cost

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "timing_model.json")))


@pytest.mark.parametrize("case", GOLD["cases"], ids=lambda c: f"K{c['K']}-Tm{c['Tm']}-Ta{c['Ta']}")
def test_formula_golden(case):
    d = default_cost(case["K"], case["Tm"], case["Ta"])
    s = subpipelined_cost(case["K"], case["Tm"], case["Ta"])
    assert d["total"] == pytest.approx(case["default_total"])
    assert s["fwd"] == pytest.approx(case["sub_fwd"])
    assert s["bwd"] == pytest.approx(case["sub_bwd"])
    assert s["total"] == pytest.approx(case["sub_total"])


def test_simulation_equals_formula_grid():
    """Reading R15 (T_a/2 per block): a two-stream FIFO simulation with n=2 reproduces the
    paper's forward and backward formulas exactly, and fwd+bwd == the printed total."""
    for K, Tm, Ta in itertools.product([1, 2, 4, 8, 24], [0.5, 1, 2], [0, 0.5, 1, 2, 4]):
        f = subpipelined_cost(K, Tm, Ta)
        assert simulate(K, Tm, Ta, 2, "fwd") == pytest.approx(f["fwd"], rel=1e-12, abs=1e-12)
        assert simulate(K, Tm, Ta, 2, "bwd") == pytest.approx(f["bwd"], rel=1e-12, abs=1e-12)
        assert f["fwd"] + f["bwd"] == pytest.approx(f["total"], rel=1e-12)
        assert f["total"] <= default_cost(K, Tm, Ta)["total"] + 1e-12


def test_n1_simulation_is_default():
    """With one sub-batch nothing overlaps: the simulation is the default cost."""
    for K, Tm, Ta in itertools.product([1, 3], [0.5, 1], [0, 1, 2]):
        assert simulate(K, Tm, Ta, 1, "fwd") == pytest.approx(K * (Tm + Ta))
        assert simulate(K, Tm, Ta, 1, "bwd") == pytest.approx(K * (2 * Tm + Ta))


def test_ceiling_is_seven_quarters():
    """default/sub-pipelined -> 7/4 at T_a = 2 T_m as K -> inf (and 1.6 at K=4, T_a=T_m)."""
    r = default_cost(10 ** 6, 1, 2)["total"] / subpipelined_cost(10 ** 6, 1, 2)["total"]
    assert r == pytest.approx(1.75, rel=1e-5)
    assert default_cost(4, 1, 1)["total"] / subpipelined_cost(4, 1, 1)["total"] == pytest.approx(1.6)
    best = max(default_cost(10 ** 6, 1, ta)["total"] / subpipelined_cost(10 ** 6, 1, ta)["total"]
               for ta in [x / 100 for x in range(0, 600)])
    assert best == pytest.approx(1.75, rel=1e-4)


def test_trace_streams_are_serial_and_respect_deps():
    tr = []
    simulate(3, 1.0, 0.7, 2, "fwd", tr)
    for stream in ("comp", "comm"):
        iv = [t for t in tr if t[0] == stream]
        for a, b in zip(iv, iv[1:]):
            assert b[4] >= a[5] - 1e-12
    comp = {(t[1], t[2], t[3]): t for t in tr if t[0] == "comp"}
    comm = {(t[1], t[2], t[3]): t for t in tr if t[0] == "comm"}
    for key, c in comm.items():
        assert c[4] >= comp[key][5] - 1e-12
