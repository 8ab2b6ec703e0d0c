"""Activation recomputation inside the backward: MERAK_FLAG_RECOMPUTE
regenerates every activation the backward reads from x, so the results are bit-identical to a backward on
the forward's own activations -- in a chained stack whose recomputed layers share one scratch buffer, with
the regeneration inside layer_bwd or as a separate early-recompute forward call, at T = 1 and for the
T = 2 / 4 ranks of an in-process group -- and match the fp64 oracle."""
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

CFG = CONFIGS["tiny"].with_(hidden=256, heads=4, seq_len=128, microbatch=4, n_sub=2, tmp_degree=1)


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _same(a, b):
    assert torch.equal(a["y"], b["y"]) and torch.equal(a["dx"], b["dx"])
    for k in range(len(a["grads"])):
        for name in a["grads"][k]:
            assert torch.equal(a["grads"][k][name], b["grads"][k][name]), (k, name)


@pytest.mark.parametrize("n_sub", [1, 2])
@pytest.mark.parametrize("early", [False, True])
def test_recompute_chain_bit_identical_and_oracle(n_sub, early):
    from gpu_layer_util import TOL_BF16, oracle_chain, rel_err, run_gpu_chain
    cfg = CFG.with_(n_sub=n_sub)
    K = 3
    params = [make_params(cfg, layer=k) for k in range(K)]
    x, dy = make_activations(cfg)
    ref = run_gpu_chain(cfg, params, x, dy)
    rc = run_gpu_chain(cfg, params, x, dy, recompute=[True, False, True], early=early)
    _same(ref, rc)
    allrc = run_gpu_chain(cfg, params, x, dy, recompute=[True] * K, early=early)
    _same(ref, allrc)
    y, dx, g = oracle_chain(params, x, dy, cfg.heads)
    M, h = cfg.tokens, cfg.hidden
    errs = {"y": rel_err(rc["y"].float().cpu().numpy(), y.reshape(M, h)),
            "dx": rel_err(rc["dx"].float().cpu().numpy(), dx.reshape(M, h))}
    for k in range(K):
        for name, r in g[k].items():
            errs[f"{k}.{name}"] = rel_err(rc["grads"][k][name].cpu().numpy(), r)
    bad = {k: v for k, v in errs.items() if not v <= TOL_BF16}
    assert not bad, bad


@pytest.mark.parametrize("T", [2, 4])
def test_recompute_group_bit_identical(T):
    """T ranks of an in-process group: each rank's backward on a garbage-filled scratch with
    MERAK_FLAG_RECOMPUTE equals its backward on the forward's activations, bit for bit."""
    from gpu_layer_util import compare_to_oracle, oracle_rank_slices
    from oracle import layer_fwd_bwd
    from paper_2206_04959_b200 import FLAG_RECOMPUTE, PARAM_NAMES, TmpLayer, shard_weights, zero_grads_like
    cfg = CFG.with_(tmp_degree=T, heads=8, hidden=256)
    params, x, dy = make_all(cfg)
    dev = torch.device("cuda", torch.cuda.current_device())
    M, h = cfg.tokens, cfg.hidden
    X = torch.as_tensor(np.asarray(x).reshape(M, h)).to(dev, torch.bfloat16)
    DY = torch.as_tensor(np.asarray(dy).reshape(M, h)).to(dev, torch.bfloat16)
    outs = {}
    for mode in ("saved", "recompute"):
        ranks = TmpLayer.group(cfg.hidden, cfg.heads, cfg.seq_len, cfg.microbatch, T, n_sub=2, device=dev.index)
        ws = [shard_weights(params, cfg.heads, T, r, dev) for r in range(T)]
        Y = [torch.empty_like(X) for _ in range(T)]
        DX = [torch.empty_like(X) for _ in range(T)]
        G = [zero_grads_like(w) for w in ws]
        S = [lay.new_saved() for lay in ranks]
        st = [torch.cuda.Stream(device=dev) for _ in range(T)]
        for s in st:
            s.wait_stream(torch.cuda.current_stream())
        for r in range(T):
            ranks[r].forward(ws[r], X, Y[r], S[r], stream=st[r])
        torch.cuda.synchronize()
        flags = 0
        if mode == "recompute":
            for s_ in S:
                s_.fill_(0xFF)
            flags = FLAG_RECOMPUTE
        for r in range(T):
            ranks[r].backward(ws[r], X, S[r], DY, DX[r], G[r], flags=flags, stream=st[r])
        torch.cuda.synchronize()
        outs[mode] = [{"y": Y[r], "dx": DX[r], **{k: G[r][k] for k in PARAM_NAMES}} for r in range(T)]
        for lay in ranks:
            lay.close()
    y, dx, g = layer_fwd_bwd(params, x, dy, cfg.heads)
    for r in range(T):
        a, b = outs["saved"][r], outs["recompute"][r]
        for k in a:
            assert torch.equal(a[k], b[k]), (r, k)
        _, bad = compare_to_oracle(b, y, dx, oracle_rank_slices(g, cfg, T, r), cfg)
        assert not bad, (r, bad)


def test_recompute_rejected_in_fp32_mode():
    from paper_2206_04959_b200 import FLAG_RECOMPUTE, MERAK_FP32_CHECK, MerakError, TmpLayer, shard_weights, zero_grads_like
    cfg = CONFIGS["tiny"].with_(tmp_degree=1)
    params, x, dy = make_all(cfg)
    dev = torch.device("cuda", torch.cuda.current_device())
    lay = TmpLayer(cfg.hidden, cfg.heads, cfg.seq_len, cfg.microbatch, precision=MERAK_FP32_CHECK, device=dev.index)
    w = shard_weights(params, cfg.heads, 1, 0, dev, dtype=torch.float32)
    X = torch.as_tensor(np.asarray(x).reshape(cfg.tokens, cfg.hidden)).to(dev, torch.float32)
    S = lay.new_saved()
    with pytest.raises(MerakError):
        lay.backward(w, X, S, X, torch.empty_like(X), zero_grads_like(w), flags=FLAG_RECOMPUTE)
    lay.close()
