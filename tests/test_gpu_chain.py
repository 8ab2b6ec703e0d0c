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
