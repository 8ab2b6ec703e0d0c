"""T > 1 parity on ONE GPU (driver-verifiable): the T ranks of a TMP group as handles of one process
(merak_tmp_init_group, MERAK_COMM_INPROC), each holding its weight shard, every all-reduce summing the
T ranks' bf16 partials in rank order through the same peer kernels (one-shot at T = 2, two-shot at
T >= 4; the cross-rank handshake is the group's event exchange, see merak_tmp.h) -- the method itself: row-parallel partial sums over T ranks with sub-microbatches
overlapping.  Checked per rank against the fp64 oracle's slices (rel. Frobenius <= 2e-2; fp32
check mode <= 1e-5), replicated outputs bit-equal across ranks, n = 1 vs n > 1 bit-identical per rank,
one-shot vs two-shot bit-identical, chained stacks equal to unchained ones."""
import pytest
import torch

from oracle import layer_fwd_bwd
from synth import CONFIGS, make_all

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from gpu_layer_util import TOL_FP32, compare_to_oracle, oracle_chain, oracle_rank_slices, run_gpu_group

TINY = CONFIGS["tiny"]
REPLICATED = ("y", "dx", "ln1_g", "ln1_b", "ln2_g", "ln2_b", "b_o", "b_2")

# (T, name) -> config.  Head splits (reading R8): h320_H5 at T=2 is 3/2, at T=4 2/1/1/1; h640_H10 at T=8
# is 2/2/1/1/1/1/1/1; gpt1.5b at T=2 is the BASELINE config with 13/12 heads.
CASES = {
    (2, "tiny"): TINY.with_(tmp_degree=2),
    (2, "h320_H5_uneven"): TINY.with_(hidden=320, heads=5, seq_len=64, microbatch=4, tmp_degree=2),
    (2, "h384_H4_d96_n4"): TINY.with_(hidden=384, heads=4, seq_len=64, microbatch=4, n_sub=4, tmp_degree=2),
    (4, "h320_H5_uneven"): TINY.with_(hidden=320, heads=5, seq_len=64, microbatch=4, tmp_degree=4),
    (4, "h256_H8_s128_n4"): TINY.with_(hidden=256, heads=8, seq_len=128, microbatch=4, n_sub=4, tmp_degree=4),
    (4, "h320_H4_d80_ragged"): TINY.with_(hidden=320, heads=4, seq_len=208, microbatch=2, tmp_degree=4),
    (8, "h256_H8_d32_s128"): TINY.with_(hidden=256, heads=8, seq_len=128, microbatch=4, tmp_degree=8),
    (8, "h640_H10_uneven"): TINY.with_(hidden=640, heads=10, seq_len=64, microbatch=4, tmp_degree=8),
    (8, "h768_H8_d96_n4"): TINY.with_(hidden=768, heads=8, seq_len=96, microbatch=4, n_sub=4, tmp_degree=8),
}


def _check_ranks(outs, cfg, T, y, dx, g, tol=None):
    failures = []
    for r, out in enumerate(outs):
        kw = {} if tol is None else {"tol": tol}
        errs, bad = compare_to_oracle(out, y, dx, oracle_rank_slices(g, cfg, T, r), cfg, **kw)
        print(f"rank {r}", {k: f"{v:.2e}" for k, v in errs.items()})
        if bad:
            failures.append((r, bad))
    return failures


@pytest.mark.parametrize("key", list(CASES), ids=[f"T{t}-{n}" for t, n in CASES])
def test_group_matches_oracle(key):
    T, _ = key
    cfg = CASES[key]
    params, x, dy = make_all(cfg, seed=3000 + cfg.hidden + T)
    y, dx, g = layer_fwd_bwd(params, x, dy, cfg.heads)
    outs = run_gpu_group(cfg, params, x, dy, T)
    assert not _check_ranks(outs, cfg, T, y, dx, g)
    # replicated outputs (y, dx, LN / row-parallel bias grads) are bit-identical on every rank
    for k in REPLICATED:
        for r in range(1, T):
            assert torch.equal(outs[0][k], outs[r][k]), (k, r)
    # sub-pipelined vs non-sub-pipelined: bit-identical per rank (north_star)
    outs1 = run_gpu_group(cfg, params, x, dy, T, n_sub=1)
    for r in range(T):
        for k in outs[r]:
            assert torch.equal(outs[r][k], outs1[r][k]), (r, k, "n vs n=1")


@pytest.mark.parametrize("T", [2, 4, 8])
def test_group_one_shot_equals_two_shot(T, monkeypatch):
    """The two all-reduce algorithms (one-shot: every rank sums all T partials; two-shot: owner rows
    reduced then gathered) round once at the same point (reading R10): bit-identical."""
    cfg = TINY.with_(hidden=256, heads=8, seq_len=64, microbatch=4, tmp_degree=T)
    params, x, dy = make_all(cfg, seed=3100 + T)
    monkeypatch.setenv("MERAK_AR_TWO_SHOT", "0")
    a = run_gpu_group(cfg, params, x, dy, T)
    monkeypatch.setenv("MERAK_AR_TWO_SHOT", "1")
    b = run_gpu_group(cfg, params, x, dy, T)
    for r in range(T):
        for k in a[r]:
            assert torch.equal(a[r][k], b[r][k]), (r, k)


@pytest.mark.parametrize("T", [2, 4, 8])
def test_group_fp32_check_mode(T):
    """fp32 check mode over the peer all-reduce at T > 1: <= 1e-5 (north_star)."""
    cfg = TINY.with_(hidden=256, heads=8, seq_len=32, microbatch=2, tmp_degree=T)
    params, x, dy = make_all(cfg, seed=3200 + T)
    y, dx, g = layer_fwd_bwd(params, x, dy, cfg.heads)
    outs = run_gpu_group(cfg, params, x, dy, T, precision=1)
    assert not _check_ranks(outs, cfg, T, y, dx, g, tol=TOL_FP32)
    outs1 = run_gpu_group(cfg, params, x, dy, T, precision=1, n_sub=1)
    for r in range(T):
        for k in outs[r]:
            assert torch.equal(outs[r][k], outs1[r][k]), (r, k)


@pytest.mark.parametrize("T", [2, 4])
def test_group_chained_stack(T):
    """K = 3 chained layers (cross-layer overlap) at T > 1: chained == unchained bitwise on every
    rank, and the stack matches the fp64 oracle composed layer by layer."""
    from synth import make_activations, make_params
    cfg = TINY.with_(hidden=256, heads=4, seq_len=128, microbatch=4, n_sub=2, tmp_degree=T)
    plist = [make_params(cfg, layer=k) for k in range(3)]
    x, dy = make_activations(cfg)
    a = run_gpu_group(cfg, None, x, dy, T, chain_params=plist)
    b = run_gpu_group(cfg, None, x, dy, T, chain_params=plist, chain=False)
    y, dxr, gr = oracle_chain(plist, x, dy, cfg.heads)
    for r in range(T):
        for k in ("y", "dx"):
            assert torch.equal(a[r][k], b[r][k]), (r, k)
        for kk in range(3):
            for nm in a[r]["grads"][kk]:
                assert torch.equal(a[r]["grads"][kk][nm], b[r]["grads"][kk][nm]), (r, kk, nm)
        for kk in range(3):
            out = {"y": a[r]["y"], "dx": a[r]["dx"], **a[r]["grads"][kk]}
            errs, bad = compare_to_oracle(out, y, dxr, oracle_rank_slices(gr[kk], cfg, T, r), cfg)
            assert not bad, (r, kk, bad)


@pytest.mark.slow
def test_group_gpt15b_full_T2():
    """BASELINE.json configs[1] at full size: h=1600, H=25 (13/12 heads), s=1024, B=8, T=2, n=2, both ranks
    on one GPU; every tensor of both ranks vs the fp64 oracle, replicated outputs equal, n=1 bit-identical."""
    cfg = CONFIGS["gpt1.5b"]
    params, x, dy = make_all(cfg)
    y, dx, g = layer_fwd_bwd(params, x, dy, cfg.heads)
    outs = run_gpu_group(cfg, params, x, dy, 2)
    assert not _check_ranks(outs, cfg, 2, y, dx, g)
    for k in REPLICATED:
        assert torch.equal(outs[0][k], outs[1][k]), k
    outs1 = run_gpu_group(cfg, params, x, dy, 2, n_sub=1)
    for r in range(2):
        for k in outs[r]:
            assert torch.equal(outs[r][k], outs1[r][k]), (r, k)
