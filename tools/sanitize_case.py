"""One tiny layer fwd+bwd for compute-sanitizer runs: T = 1 (one handle), or an in-process T = 2 group
(MERAK_COMM_INPROC) when argv[1] == "group".  Exit 0 = ran and matched the fp64 oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from gpu_layer_util import compare_to_oracle, oracle_rank_slices, run_gpu_group, run_gpu_layer  # noqa: E402
from oracle import layer_fwd_bwd  # noqa: E402
from synth import CONFIGS, make_all  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "single"
cfg = CONFIGS["tiny"].with_(hidden=128, heads=2, seq_len=64, microbatch=2, tmp_degree=2 if mode == "group" else 1)
params, x, dy = make_all(cfg, seed=5)
y, dx, g = layer_fwd_bwd(params, x, dy, cfg.heads)
outs = run_gpu_group(cfg, params, x, dy, 2) if mode == "group" else [run_gpu_layer(cfg, params, x, dy)]
bad = {}
for r, o in enumerate(outs):
    _, b = compare_to_oracle(o, y, dx, oracle_rank_slices(g, cfg, cfg.tmp_degree, r), cfg)
    bad.update(b)
print("sanitize case", mode, "ok" if not bad else bad)
sys.exit(1 if bad else 0)
