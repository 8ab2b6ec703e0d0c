"""Stage-aware recomputation: the oracle pinned against hand-evaluated
values of the paper's recursion and the invariants the paper states, and the C-ABI planner
(include/merak_sched.h) against the oracle (CPU only: host functions, no GPU)."""
import ctypes
import json
import os
import random

import pytest

from oracle.stage import stage_alphas, stage_memory, tune_alpha1

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "stage_alpha.json")))


@pytest.mark.parametrize("case", GOLD["cases"], ids=lambda c: f"s{c['s']}-a{c['alpha1']}")
def test_oracle_golden(case):
    assert stage_alphas(case["s"], case["alpha1"]) == pytest.approx(case["alphas"], rel=1e-12)


def test_oracle_invariants():
    """P:521 equal memory: (s-i) alpha_i = (s-1) alpha_1 wherever the min(1, .) does not clip (i < s-1);
    alpha_s = 1; alpha_{s-1} = alpha_{s-2}; every alpha in [0, 1]; non-decreasing in i."""
    for s in range(3, 17):
        for a1 in [0.0, 0.01, 0.05, 0.1, 0.25, 0.5, 0.9, 1.0]:
            al = stage_alphas(s, a1)
            assert al[-1] == 1.0 and al[s - 2] == al[s - 3]
            assert all(0.0 <= a <= 1.0 for a in al)
            assert all(al[k] <= al[k + 1] + 1e-15 for k in range(s - 1))
            for i in range(2, s - 1):
                if al[i - 1] < 1.0:
                    assert (s - i) * al[i - 1] == pytest.approx((s - 1) * a1, rel=1e-12, abs=1e-15)
            mem = stage_memory(s, al, 10.0, 1.0)
            for i in range(1, s - 1):  # unclipped stages use the same memory as stage 1
                if al[i - 1] < 1.0:
                    assert mem[i - 1] == pytest.approx(mem[0], rel=1e-12)


def test_oracle_tune_saturated_capacity():
    """capacity = M_r + (s-1) M_a (room for every microbatch's activations on stage 1) -> alpha_1 = 1."""
    for s in (2, 4, 8):
        assert tune_alpha1(s, 0.05, 10.0 + (s - 1) * 2.0, 10.0, 2.0) == 1.0
        assert tune_alpha1(s, 0.05, 10.0, 10.0, 2.0) == 0.0
        assert tune_alpha1(s, 0.05, 9.0, 10.0, 2.0) is None


@pytest.fixture(scope="module")
def lib():
    from paper_2206_04959_b200.binding import lib as load
    L = load()
    L.merak_stage_alpha.argtypes = [ctypes.c_int32, ctypes.c_double, ctypes.POINTER(ctypes.c_double)]
    L.merak_tune_alpha1.argtypes = [ctypes.c_int32] + [ctypes.c_double] * 4 + [ctypes.POINTER(ctypes.c_double)]
    L.merak_layers_kept.argtypes = [ctypes.c_double, ctypes.c_int32]
    L.merak_layers_kept.restype = ctypes.c_int32
    return L


def test_abi_alpha_matches_oracle(lib):
    for s in range(1, 33):
        for a1 in [0.0, 0.03, 0.1, 1 / 3, 0.5, 0.77, 1.0]:
            out = (ctypes.c_double * s)()
            assert lib.merak_stage_alpha(s, a1, out) == 0
            assert list(out) == pytest.approx(stage_alphas(s, a1), rel=1e-15, abs=0)
    out = (ctypes.c_double * 4)()
    assert lib.merak_stage_alpha(4, 1.5, out) == -1
    assert lib.merak_stage_alpha(0, 0.5, out) == -1


def test_abi_tune_matches_bruteforce(lib):
    rng = random.Random(220604959)
    for _ in range(2000):
        s = rng.randint(1, 16)
        m_r, m_a = rng.uniform(1, 100), rng.uniform(0.1, 20)
        cap = max(0.0, m_r + rng.uniform(-5, (s - 1) * m_a + 5))
        step = rng.choice([0.01, 0.05, 0.1, 0.125, 0.3])
        want = tune_alpha1(s, step, cap, m_r, m_a)
        got = ctypes.c_double(-1)
        st = lib.merak_tune_alpha1(s, step, cap, m_r, m_a, ctypes.byref(got))
        if want is None:
            assert st == -6  # MERAK_ENOMEM
        else:
            assert st == 0 and got.value == pytest.approx(want, abs=1e-12)


def test_abi_layers_kept(lib):
    assert [lib.merak_layers_kept(a, 4) for a in (0.0, 0.2, 0.25, 0.3, 0.5, 0.99, 1.0)] == [0, 0, 1, 1, 2, 3, 4]
