"""fp32 check mode (MERAK_FP32_CHECK) vs the fp64 oracle: relative Frobenius error <= 1e-5 on every
output and gradient (north_star), and n_sub > 1 bit-identical to n_sub = 1 (SURVEY §8(c) rules)."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from oracle import layer_fwd_bwd  # noqa: E402
from synth import CONFIGS, make_all  # noqa: E402

torch = pytest.importorskip("torch")

TINY = CONFIGS["tiny"].with_(tmp_degree=1)
CASES = {
    "tiny": TINY,
    "h320_d64_s64_n2": TINY.with_(hidden=320, heads=5, seq_len=64, microbatch=4, n_sub=2),
    "h256_d32_s128_n4": TINY.with_(hidden=256, heads=8, seq_len=128, microbatch=4, n_sub=4),
    "h320_d80_s48": TINY.with_(hidden=320, heads=4, seq_len=48, microbatch=2, n_sub=2),
    "h384_d96_s32": TINY.with_(hidden=384, heads=4, seq_len=32, microbatch=2, n_sub=2),
    "h256_d128_s80": TINY.with_(hidden=256, heads=2, seq_len=80, microbatch=2, n_sub=2),
}


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


@pytest.mark.parametrize("name", list(CASES))
def test_fp32_check_mode_vs_oracle(name):
    from gpu_layer_util import TOL_FP32, compare_to_oracle, oracle_rank_slices, run_gpu_layer
    cfg = CASES[name]
    params, x, dy = make_all(cfg, seed=4000 + cfg.hidden)
    out = run_gpu_layer(cfg, params, x, dy, precision=1)
    y, dx, g = layer_fwd_bwd(params, x, dy, cfg.heads)
    errs, bad = compare_to_oracle(out, y, dx, oracle_rank_slices(g, cfg, 1, 0), cfg, tol=TOL_FP32)
    print(name, {k: f"{v:.1e}" for k, v in errs.items()})
    assert not bad, bad


@pytest.mark.parametrize("name", ["h320_d64_s64_n2", "h256_d32_s128_n4"])
def test_fp32_check_mode_subbatch_bit_identity(name):
    from gpu_layer_util import run_gpu_layer
    cfg = CASES[name]
    params, x, dy = make_all(cfg, seed=4100 + cfg.hidden)
    a = run_gpu_layer(cfg, params, x, dy, precision=1)
    b = run_gpu_layer(cfg, params, x, dy, precision=1, n_sub=1)
    for k in a:
        assert torch.equal(a[k], b[k]), k
