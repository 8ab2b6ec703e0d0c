"""Host enqueue cost of a bench step vs its GPU time (one GPU, T = 1): if the host needs longer to issue a
step's ~180 launches (tensor-map encodes, events, ctypes) than the GPU needs to run them, the step is
host-bound.  Prints one JSON line per config."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from synth import CONFIGS  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    for name in sys.argv[1:] or ["gpt1.5b", "gpt20b"]:
        cfg = CONFIGS[name].with_(tmp_degree=1)
        st = bench.Stack(cfg, 4, 1, 0, dev, None, cfg.n_sub)
        for _ in range(3):
            st.step()
        torch.cuda.synchronize()
        n = 10
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t0 = time.perf_counter()
        for _ in range(n):
            st.step()
        t_host = (time.perf_counter() - t0) / n
        e1.record()
        torch.cuda.synchronize()
        t_gpu = e0.elapsed_time(e1) / n * 1e-3
        launches = st.layer.launch_count()
        st.close()
        print(json.dumps({"config": name, "host_ms_per_step": t_host * 1e3, "gpu_ms_per_step": t_gpu * 1e3,
                          "host_bound": t_host > t_gpu}), flush=True)


if __name__ == "__main__":
    main()
