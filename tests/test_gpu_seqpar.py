"""Sequence-parallel layout (seq_parallel = 1): the row-parallel all-reduces become
reduce-scatters (the fused LN / residual epilogues run on each rank's own token rows) and the column-parallel
GEMMs read all-gathered activations.  Checked on ONE GPU with in-process T = 2/4 groups: y / dx (gathered from
the ranks' token shards) and every gradient vs the fp64 oracle; y, dx and the weight / bias gradients
bit-identical to the replicated layout; n = 1 vs n = 2; a chained stack."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from synth import CONFIGS, make_activations, make_all, make_params  # noqa: E402

torch = pytest.importorskip("torch")
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

CFG = CONFIGS["tiny"].with_(hidden=256, heads=8, seq_len=128, microbatch=4, n_sub=2)
WEIGHT_GRADS = ("w_qkv", "b_qkv", "w_o", "b_o", "w_1", "b_1", "w_2", "b_2")


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def run_sp_group(cfg, plist, x, dy, T, n_sub=2, seq_parallel=True):
    """K = len(plist) chained layers on an in-process group; returns per rank: y, dx (full [M, h], the token
    shards scattered back into place) and grads[k]."""
    from paper_2206_04959_b200 import FLAG_CHAIN, PARAM_NAMES, TmpLayer, shard_weights, sp_rows, zero_grads_like
    dev = torch.device("cuda", torch.cuda.current_device())
    M, h = cfg.tokens, cfg.hidden
    ranks = TmpLayer.group(cfg.hidden, cfg.heads, cfg.seq_len, cfg.microbatch, T, n_sub=n_sub, device=dev.index,
                           seq_parallel=seq_parallel)
    K = len(plist)
    X = torch.as_tensor(np.asarray(x).reshape(M, h)).to(dev, torch.bfloat16)
    DY = torch.as_tensor(np.asarray(dy).reshape(M, h)).to(dev, torch.bfloat16)
    rows = [sp_rows(M, n_sub, T, r).to(dev) if seq_parallel else torch.arange(M, device=dev) for r in range(T)]
    ws = [[shard_weights(p, cfg.heads, T, r, dev) for p in plist] for r in range(T)]
    Xr = [X[rows[r]].contiguous() for r in range(T)]
    DYr = [DY[rows[r]].contiguous() for r in range(T)]
    Ys = [[torch.empty_like(Xr[r]) for _ in range(K)] for r in range(T)]
    DXs = [[torch.empty_like(Xr[r]) for _ in range(K)] for r in range(T)]
    grads = [[zero_grads_like(w) for w in ws[r]] for r in range(T)]
    saved = [[ranks[r].new_saved() for _ in range(K)] for r in range(T)]
    streams = [torch.cuda.Stream(device=dev) for _ in range(T)]
    for s in streams:
        s.wait_stream(torch.cuda.current_stream())
    for k in range(K):
        for r in range(T):
            ranks[r].forward(ws[r][k], Xr[r] if k == 0 else Ys[r][k - 1], Ys[r][k], saved[r][k], flags=FLAG_CHAIN,
                             stream=streams[r])
    for k in reversed(range(K)):
        for r in range(T):
            ranks[r].backward(ws[r][k], Xr[r] if k == 0 else Ys[r][k - 1], saved[r][k],
                              DYr[r] if k == K - 1 else DXs[r][k + 1], DXs[r][k], grads[r][k],
                              flags=FLAG_CHAIN if k > 0 else 0, stream=streams[r])
    torch.cuda.synchronize()
    y = torch.empty_like(X)
    dx = torch.empty_like(X)
    for r in range(T):
        y[rows[r]] = Ys[r][K - 1]
        dx[rows[r]] = DXs[r][0]
    outs = [{"y": y.clone(), "dx": dx.clone(), "grads": [{n: g[n].clone() for n in PARAM_NAMES} for g in grads[r]]}
            for r in range(T)]
    for lay in ranks:
        lay.close()
    return outs


@pytest.mark.parametrize("T", [2, 4])
def test_seqpar_vs_oracle_and_replicated(T):
    from gpu_layer_util import compare_to_oracle, oracle_rank_slices
    from oracle import layer_fwd_bwd
    cfg = CFG.with_(tmp_degree=T)
    params, x, dy = make_all(cfg)
    sp = run_sp_group(cfg, [params], x, dy, T)
    rep = run_sp_group(cfg, [params], x, dy, T, seq_parallel=False)
    y, dx, g = layer_fwd_bwd(params, x, dy, cfg.heads)
    for r in range(T):
        o = {"y": sp[r]["y"], "dx": sp[r]["dx"], **sp[r]["grads"][0]}
        errs, bad = compare_to_oracle(o, y, dx, oracle_rank_slices(g, cfg, T, r), cfg)
        print(r, {k: f"{v:.1e}" for k, v in errs.items()})
        assert not bad, (r, bad)
        # every row is computed by the same kernels: y, dx and the weight / bias gradients are bit-identical
        assert torch.equal(sp[r]["y"], rep[r]["y"]) and torch.equal(sp[r]["dx"], rep[r]["dx"])
        for k in WEIGHT_GRADS:
            assert torch.equal(sp[r]["grads"][0][k], rep[r]["grads"][0][k]), (r, k)
        # LN-parameter gradients: same sums in another order
        for k in ("ln1_g", "ln1_b", "ln2_g", "ln2_b"):
            a, b_ = sp[r]["grads"][0][k], rep[r]["grads"][0][k]
            assert (a - b_).norm() <= 1e-5 * b_.norm() + 1e-6, (r, k)


def test_seqpar_n1_vs_n2_and_chain():
    """Sub-pipelined (n = 2) vs n = 1 in the sequence-parallel layout (y, dx and weight gradients bit-identical),
    and a 3-layer chain (cross-layer reuse of the all-gather slot) vs the fp64 oracle."""
    from gpu_layer_util import TOL_BF16, oracle_chain, rel_err
    T = 2
    cfg = CFG.with_(tmp_degree=T)
    params, x, dy = make_all(cfg)
    a = run_sp_group(cfg, [params], x, dy, T, n_sub=2)
    b = run_sp_group(cfg, [params], x, dy, T, n_sub=1)
    for r in range(T):
        assert torch.equal(a[r]["y"], b[r]["y"]) and torch.equal(a[r]["dx"], b[r]["dx"])
        for k in WEIGHT_GRADS:
            assert torch.equal(a[r]["grads"][0][k], b[r]["grads"][0][k]), (r, k)
    K = 3
    plist = [make_params(cfg, layer=k) for k in range(K)]
    xc, dyc = make_activations(cfg)
    outs = run_sp_group(cfg, plist, xc, dyc, T)
    yo, dxo, go = oracle_chain(plist, xc, dyc, cfg.heads)
    M, h = cfg.tokens, cfg.hidden
    assert rel_err(outs[0]["y"].float().cpu().numpy(), yo.reshape(M, h)) <= TOL_BF16
    assert rel_err(outs[0]["dx"].float().cpu().numpy(), dxo.reshape(M, h)) <= TOL_BF16
    from oracle import shard_params
    for r in range(T):
        for k in range(K):
            ref = shard_params(go[k], cfg.heads, T, r)
            for n_, v in ref.items():
                e = rel_err(outs[r]["grads"][k][n_].cpu().numpy(), v)
                assert e <= TOL_BF16, (r, k, n_, e)


def test_seqpar_validation():
    from paper_2206_04959_b200 import MerakError, TmpLayer
    with pytest.raises(MerakError):  # tokens per sub-batch not a multiple of 8 T
        TmpLayer.group(256, 8, 16, 2, 4, n_sub=2, seq_parallel=True)
