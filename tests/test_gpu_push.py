"""Fused GEMM -> reduce-scatter push (MERAK_AR_PUSH=1, tile-granular fusion): the row-parallel
GEMMs (proj, fc2, fc1 dgrad, QKV dgrad) store every 32-row output box straight into the slot of the rank that owns
those rows, so the reduce-scatter phase (sequence-parallel layout, or phase 1 of the two-shot all-reduce) sums T
LOCAL row blocks in rank order.  The arithmetic is unchanged (P:107 / P:558: the owner sums the T row-parallel
partials), so every output and gradient must be bit-identical to the pull layout -- checked on ONE GPU with
in-process T = 2/4/8 groups, over a 3-layer chain (slot reuse across layers and sub-batches), and against the
fp64 oracle."""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from synth import CONFIGS, make_activations, make_all, make_params  # noqa: E402

torch = pytest.importorskip("torch")

# tokens per sub-batch m = 4 * 128 / 2 = 256: owner rows m / T = 128 / 64 / 32 at T = 2 / 4 / 8 (whole 32-row boxes)
CFG = CONFIGS["tiny"].with_(hidden=256, heads=8, seq_len=128, microbatch=4, n_sub=2)


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _run(monkeypatch, push, cfg, plist, x, dy, T, seq_parallel, two_shot=None, n_sub=2):
    from test_gpu_seqpar import run_sp_group
    monkeypatch.setenv("MERAK_AR_PUSH", push if isinstance(push, str) else ("1" if push else "0"))
    # every row-parallel GEMM pushes at these small shapes (the default K threshold keeps short-K GEMMs on pull)
    monkeypatch.setenv("MERAK_AR_PUSH_MINK", "0")
    if two_shot is not None:
        monkeypatch.setenv("MERAK_AR_TWO_SHOT", "1" if two_shot else "0")
    return run_sp_group(cfg, plist, x, dy, T, n_sub=n_sub, seq_parallel=seq_parallel)


def _assert_identical(a, b, T):
    for r in range(T):
        assert torch.equal(a[r]["y"], b[r]["y"]), (r, "y")
        assert torch.equal(a[r]["dx"], b[r]["dx"]), (r, "dx")
        for k, (ga, gb) in enumerate(zip(a[r]["grads"], b[r]["grads"])):
            for n_ in ga:
                assert torch.equal(ga[n_], gb[n_]), (r, k, n_)


@pytest.mark.parametrize("T", [2, 4, 8])
def test_push_seqpar_chain_bit_identical(T, monkeypatch):
    cfg = CFG.with_(tmp_degree=T)
    K = 3
    plist = [make_params(cfg, layer=k) for k in range(K)]
    x, dy = make_activations(cfg)
    pull = _run(monkeypatch, False, cfg, plist, x, dy, T, True)
    push = _run(monkeypatch, True, cfg, plist, x, dy, T, True)
    _assert_identical(push, pull, T)


@pytest.mark.parametrize("mode", ["1", "2"], ids=["rs", "rs+ag"])
@pytest.mark.parametrize("T", [2, 4, 8])
def test_push_two_shot_chain_bit_identical(T, mode, monkeypatch):
    """Replicated layout, two-shot all-reduce: phase 1 reads the pushed local blocks instead of the peers' slots
    (mode 1); mode 2 also pushes the reduced rows into every rank's all-gather slot, so phase 2 reads locally."""
    cfg = CFG.with_(tmp_degree=T)
    K = 3
    plist = [make_params(cfg, layer=k) for k in range(K)]
    x, dy = make_activations(cfg)
    pull = _run(monkeypatch, False, cfg, plist, x, dy, T, False, two_shot=True)
    push = _run(monkeypatch, mode, cfg, plist, x, dy, T, False, two_shot=True)
    _assert_identical(push, pull, T)
    if T == 4:  # one-shot reference (default pull) too
        one = _run(monkeypatch, False, cfg, plist, x, dy, T, False, two_shot=False)
        _assert_identical(push, one, T)


@pytest.mark.parametrize("T", [2, 4])
def test_push_vs_oracle_n4(T, monkeypatch):
    """n = 4 sub-batches (row offsets r0 = j m in every push map), sequence parallel, vs the fp64 oracle."""
    from gpu_layer_util import compare_to_oracle, oracle_rank_slices
    from oracle import layer_fwd_bwd
    cfg = CFG.with_(tmp_degree=T, microbatch=8, n_sub=4)
    params, x, dy = make_all(cfg, seed=4400 + T)
    y, dx, g = layer_fwd_bwd(params, x, dy, cfg.heads)
    push = _run(monkeypatch, True, cfg, [params], x, dy, T, True, n_sub=4)
    for r in range(T):
        o = {"y": push[r]["y"], "dx": push[r]["dx"], **push[r]["grads"][0]}
        errs, bad = compare_to_oracle(o, y, dx, oracle_rank_slices(g, cfg, T, r), cfg)
        print(r, {k: f"{v:.1e}" for k, v in errs.items()})
        assert not bad, (r, bad)
    pull = _run(monkeypatch, False, cfg, [params], x, dy, T, True, n_sub=4)
    _assert_identical(push, pull, T)


def test_push_ineligible_falls_back(monkeypatch):
    """Owner rows not a whole number of 32-row boxes (m / T = 16): the GEMMs store locally and the all-reduce
    pulls, with the same results."""
    T = 8
    cfg = CFG.with_(tmp_degree=T, seq_len=64)  # m = 128, m / T = 16
    params, x, dy = make_all(cfg, seed=4500)
    pull = _run(monkeypatch, False, cfg, [params], x, dy, T, False, two_shot=True)
    push = _run(monkeypatch, "2", cfg, [params], x, dy, T, False, two_shot=True)
    _assert_identical(push, pull, T)


@pytest.mark.parametrize("T", [2, 4, 8])
def test_push_is_set_up(T, monkeypatch):
    """The bit-identity tests above compare two different code paths only if the push is really on."""
    from paper_2206_04959_b200 import TmpLayer
    for env, want in (("1", True), ("0", False)):
        monkeypatch.setenv("MERAK_AR_PUSH", env)
        ranks = TmpLayer.group(CFG.hidden, CFG.heads, CFG.seq_len, CFG.microbatch, T, n_sub=2,
                               device=torch.cuda.current_device())
        try:
            assert all(r.debug_host()["push"] == want for r in ranks), (T, env)
        finally:
            for r in ranks:
                r.close()


def test_push_mixed_slots_T8(monkeypatch):
    """Realistic T = 8 mix: with the K threshold at 200 the proj GEMM (K T/(T-1) = 96 * 8/7 = 110) keeps the pull
    reduce-scatter while fc2 / fc1 dgrad (439) and QKV dgrad (329) push; the all-gather push covers every slot.
    Bit-identical to the pull layout and within the oracle tolerance."""
    from gpu_layer_util import compare_to_oracle, oracle_rank_slices
    from oracle import layer_fwd_bwd
    T = 8
    cfg = CFG.with_(hidden=768, heads=8, seq_len=128, microbatch=4, n_sub=2, tmp_degree=T)
    params, x, dy = make_all(cfg, seed=4600)
    pull = _run(monkeypatch, False, cfg, [params], x, dy, T, False, two_shot=True)
    monkeypatch.setenv("MERAK_AR_PUSH", "2")
    monkeypatch.setenv("MERAK_AR_PUSH_MINK", "200")
    from test_gpu_seqpar import run_sp_group
    mixed = run_sp_group(cfg, [params], x, dy, T, n_sub=2, seq_parallel=False)
    _assert_identical(mixed, pull, T)
    y, dx, g = layer_fwd_bwd(params, x, dy, cfg.heads)
    for r in range(T):
        o = {"y": mixed[r]["y"], "dx": mixed[r]["dx"], **mixed[r]["grads"][0]}
        errs, bad = compare_to_oracle(o, y, dx, oracle_rank_slices(g, cfg, T, r), cfg)
        assert not bad, (r, bad)
