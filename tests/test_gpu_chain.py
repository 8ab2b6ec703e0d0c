"""K stacked layers with MERAK_FLAG_CHAIN (cross-layer overlap, the bench's mode) vs the fp64 oracle
composed layer by layer, and chained vs unchained bit-identity (same kernels and per-element order;
exercises the cross-layer workspace hazards of the multi-stream schedule)."""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from synth import CONFIGS, make_activations, make_params  # noqa: E402

torch = pytest.importorskip("torch")

CFG = CONFIGS["tiny"].with_(hidden=256, heads=4, seq_len=128, microbatch=4, n_sub=2, tmp_degree=1)


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


@pytest.mark.parametrize("n_sub", [1, 2, 4])
def test_chained_layers_vs_oracle_and_unchained(n_sub):
    from gpu_layer_util import TOL_BF16, oracle_chain, rel_err, run_gpu_chain
    cfg = CFG.with_(n_sub=n_sub)
    K = 3
    params = [make_params(cfg, layer=k) for k in range(K)]
    x, dy = make_activations(cfg)
    a = run_gpu_chain(cfg, params, x, dy, chain=True)
    b = run_gpu_chain(cfg, params, x, dy, chain=False)
    assert torch.equal(a["y"], b["y"]) and torch.equal(a["dx"], b["dx"])
    for k in range(K):
        for name in a["grads"][k]:
            assert torch.equal(a["grads"][k][name], b["grads"][k][name]), (k, name)
    y, dx, g = oracle_chain(params, x, dy, cfg.heads)
    M, h = cfg.tokens, cfg.hidden
    errs = {"y": rel_err(a["y"].float().cpu().numpy(), y.reshape(M, h)),
            "dx": rel_err(a["dx"].float().cpu().numpy(), dx.reshape(M, h))}
    for k in range(K):
        for name, ref in g[k].items():
            errs[f"{k}.{name}"] = rel_err(a["grads"][k][name].cpu().numpy(), ref)
    print({k: f"{v:.1e}" for k, v in errs.items()})
    bad = {k: v for k, v in errs.items() if not v <= TOL_BF16}
    assert not bad, bad


def test_chained_ln1_fused_into_ar2(monkeypatch):
    """in a chain, layer k+1's LN1 is computed by layer k's AR#2 epilogue kernel (launched
    by the next call; opt-in MERAK_FUSE_LN1=1).  The fused LN1 uses the row engine's arithmetic on the stored
    bf16 y, so the stack is bit-identical to MERAK_FUSE_LN1=0 (separate LN1 kernels), and the LN kernel
    launches drop by (K-1) n."""
    import numpy as np
    from gpu_layer_util import run_gpu_chain
    from paper_2206_04959_b200 import FLAG_CHAIN, TmpLayer, shard_weights
    K, n = 3, 2
    cfg = CFG.with_(n_sub=n)
    params = [make_params(cfg, layer=k) for k in range(K)]
    x, dy = make_activations(cfg)
    monkeypatch.setenv("MERAK_FUSE_LN1", "1")
    fused = run_gpu_chain(cfg, params, x, dy, chain=True)
    monkeypatch.setenv("MERAK_FUSE_LN1", "0")
    plain = run_gpu_chain(cfg, params, x, dy, chain=True)
    assert torch.equal(fused["y"], plain["y"]) and torch.equal(fused["dx"], plain["dx"])
    for k in range(K):
        for name in fused["grads"][k]:
            assert torch.equal(fused["grads"][k][name], plain["grads"][k][name]), (k, name)
    # LN launches of a chained forward stack, per setting (profiling counts launches per kernel class)
    dev = torch.device("cuda", torch.cuda.current_device())
    M, h = cfg.tokens, cfg.hidden
    X = torch.as_tensor(np.asarray(x).reshape(M, h)).to(dev, torch.bfloat16)
    counts = {}
    for env in ("1", "0"):
        monkeypatch.setenv("MERAK_FUSE_LN1", env)
        lay = TmpLayer(cfg.hidden, cfg.heads, cfg.seq_len, cfg.microbatch, n_sub=n, device=dev.index)
        ws = [shard_weights(p, cfg.heads, 1, 0, dev) for p in params]
        Ys = [torch.empty_like(X) for _ in range(K)]
        sv = [lay.new_saved() for _ in range(K)]
        lay.set_profiling(True)
        for k in range(K):
            lay.forward(ws[k], X if k == 0 else Ys[k - 1], Ys[k], sv[k], flags=FLAG_CHAIN)
        lay.join()
        counts[env] = lay.get_profile()["layernorm"]["launches"]
        torch.cuda.synchronize()
        assert torch.equal(Ys[K - 1], fused["y"])
        lay.close()
    assert counts["0"] - counts["1"] == (K - 1) * n, counts
