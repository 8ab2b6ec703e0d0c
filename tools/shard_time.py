"""Per-rank compute of the TMP = 8 shards on one GPU (MERAK_COMM_LOCAL, rank 0 of 8) under environment variants:
TFLOP/s per GPU of 4 chained layers, interleaved repetitions.  One JSON line per (config, variant, rep).
Usage: python tools/shard_time.py [VAR=VALUE,VAR=VALUE ...]   (each argument is one variant; "" = defaults)"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import Stack, layer_flops  # noqa: E402
from paper_2206_04959_b200 import MERAK_COMM_LOCAL  # noqa: E402
from synth import CONFIGS  # noqa: E402


def timed(st, n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        st.step()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def main():
    variants = sys.argv[1:] or [""]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    L, T = 4, 8
    for rep in range(2):
        for name in ("gpt20b", "gpt8.3b"):
            cfg = CONFIGS[name]
            for var in variants:
                env = dict(kv.split("=", 1) for kv in var.split(",") if kv)
                old = {k: os.environ.get(k) for k in env}
                os.environ.update(env)  # kept for the whole run: some switches are read per launch
                try:
                    st = Stack(cfg, L, T, 0, dev, None, cfg.n_sub, comm=MERAK_COMM_LOCAL)
                    for _ in range(3):
                        st.step()
                    ms = timed(st, 8)
                    st.close()
                finally:
                    for k, v in old.items():
                        if v is None:
                            os.environ.pop(k, None)
                        else:
                            os.environ[k] = v
                fl = L * layer_flops(cfg) / T
                print(json.dumps({"config": name, "variant": var or "default", "rep": rep, "ms_per_step": ms,
                                  "tflops_per_gpu": fl / (ms * 1e-3) / 1e12}), flush=True)


if __name__ == "__main__":
    main()
