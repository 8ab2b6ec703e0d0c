"""Pipeline schedules of a K-layer TMP stage: the C-ABI generator
(merak_pipeline_schedule) checked with the oracle's discrete-event simulation against the paper's bubble
formulas (P:460 1F1B, P:461 early recomputation, P:470 shifted critical path), plus the schedule invariants
and the properties the paper states for SCP (CPU only: host functions)."""
import ctypes

import pytest

from oracle.pipeline import check_schedule, paper_bubble, paper_run_time, simulate

POL = {"1f1b": 0, "early": 1, "scp": 2, "none": 3}
KIND = {0: "F", 1: "R", 2: "B", 3: "BR"}


@pytest.fixture(scope="module")
def lib():
    from paper_2206_04959_b200.binding import lib as load
    L = load()
    L.merak_pipeline_schedule.argtypes = [ctypes.c_int32] * 3 + [ctypes.POINTER(ctypes.c_int32), ctypes.c_int32,
                                                                  ctypes.POINTER(ctypes.c_int32)]
    return L


def sched(lib, policy, s, m):
    cap = 3 * m
    acts = (ctypes.c_int32 * (s * cap))()
    cnt = (ctypes.c_int32 * s)()
    st = lib.merak_pipeline_schedule(POL[policy], s, m, acts, cap, cnt)
    assert st == 0, st
    return [[(KIND[acts[j * cap + k] >> 24], acts[j * cap + k] & 0xFFFFFF) for k in range(cnt[j])] for j in range(s)]


@pytest.mark.parametrize("policy", ["1f1b", "early", "none", "scp"])
def test_makespan_equals_paper_formula(lib, policy):
    for s in range(2 if policy == "scp" else 1, 13):
        for m in range(1, 25):
            if policy == "scp" and m < max(s, 3):
                continue
            sc = sched(lib, policy, s, m)
            assert not check_schedule(sc, m), (s, m)
            mk = simulate(sc)[0]
            assert mk == paper_run_time(policy, m) + paper_bubble(policy, s), (policy, s, m, mk)


def test_valid_and_monotone_for_all_sizes(lib):
    for s in range(2, 13):
        for m in range(1, 25):
            mk = {}
            for p in ("1f1b", "early", "scp"):
                sc = sched(lib, p, s, m)
                assert not check_schedule(sc, m), (p, s, m)
                mk[p] = simulate(sc)[0]  # raises on a deadlock
            assert mk["scp"] <= mk["early"] <= mk["1f1b"], (s, m, mk)


def test_golden_ratios_s4_m5(lib):
    """P:461 / P:470 evaluated at s = 4, m = 5: early 3*3/(4*5) = 0.45, SCP 3*2/(4*5) = 0.30; 1F1B 3/5."""
    for p, ratio in (("1f1b", 0.6), ("early", 0.45), ("scp", 0.30)):
        mk = simulate(sched(lib, p, 4, 5))[0]
        assert (mk - 20) / 20 == pytest.approx(ratio)


def test_scp_structure(lib):
    """no recomputation on the last stage ("the last stage only stores one activation"); the
    second-to-last stage recomputes every microbatch and runs one more forward before its first backward."""
    for s in (2, 4, 8):
        m = 2 * s
        sc = sched(lib, "scp", s, m)
        assert not any(k in ("R", "BR") for k, _ in sc[-1])
        assert sum(k == "R" for k, _ in sc[s - 2]) == m
        early = sched(lib, "early", s, m)
        lead = lambda acts: next(i for i, a in enumerate(acts) if a[0] != "F")  # noqa: E731
        assert lead(sc[s - 2]) == lead(early[s - 2]) + 1


def test_scp_critical_path_shifted(lib):
    """with early recomputation every stage is busy 4m T_m and the critical path runs through the
    last stage; SCP drops the last stage's recomputation (busy 3m T_m), so the critical path moves to stage
    s-2, whose bubble is what remains: 3(s-2) T_m."""
    for s in (3, 4, 6, 8):
        m = 2 * s
        _, _, busy_e, _ = simulate(sched(lib, "early", s, m))
        mk, _, busy, _ = simulate(sched(lib, "scp", s, m))
        assert busy_e == [4 * m] * s
        assert busy[-1] == 3 * m and busy[:-1] == [4 * m] * (s - 1)
        assert mk - busy[s - 2] == 3 * (s - 2)


def test_scp_head_layers_tolerated(lib):
    """head layers on the last stage ("could adequately handle the extra calculations"): extra
    last-stage forward work h <= T_m per microbatch lengthens SCP by less than it lengthens 1F1B / early."""
    for s in (4, 8):
        m = 2 * s
        for h in (0.25, 0.5, 1.0):
            d_scp = simulate(sched(lib, "scp", s, m), head=h)[0] - simulate(sched(lib, "scp", s, m))[0]
            for p in ("1f1b", "early"):
                d = simulate(sched(lib, p, s, m), head=h)[0] - simulate(sched(lib, p, s, m))[0]
                assert d_scp < d, (s, h, p, d_scp, d)


def test_1f1b_warmup_count(lib):
    """Stage j of 1F1B holds at most min(s - j, m) microbatches' activations: min(s-1-j, m) warm-up forwards
    plus the one of the first 1F1B pair precede its first backward."""
    for s, m in ((4, 4), (4, 2), (8, 16)):
        sc = sched(lib, "1f1b", s, m)
        for j in range(s):
            first_b = next(i for i, a in enumerate(sc[j]) if a[0] != "F")
            assert first_b == min(s - j, m)


def test_errors(lib):
    acts = (ctypes.c_int32 * 30)()
    cnt = (ctypes.c_int32 * 4)()
    assert lib.merak_pipeline_schedule(2, 1, 5, acts, 15, cnt) == -1   # SCP needs s >= 2
    assert lib.merak_pipeline_schedule(9, 2, 5, acts, 15, cnt) == -1   # bad policy
    assert lib.merak_pipeline_schedule(0, 2, 5, acts, 14, cnt) == -6   # capacity < 3 m
