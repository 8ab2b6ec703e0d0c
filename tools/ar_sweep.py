"""All-reduce cost vs message size (torchrun, T = WORLD_SIZE): handshake alone, forward and backward
epilogue all-reduces through merak_tmp_bench_allreduce.  Prints one JSON line (rank 0)."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_04959_b200 import TmpLayer  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    h = int(os.environ.get("H", 1600))
    layer = TmpLayer(h, 25 if h == 1600 else 32, 1024, 8, tmp_degree=world, tmp_rank=rank, n_sub=1,
                     group=dist.group.WORLD)
    res = {}
    for rows in (16, 512, 2048, 4096, 8192):
        r = {"hs_us": layer.bench_allreduce(2, rows, 50) * 1e3,
             "fwd_us": layer.bench_allreduce(0, rows, 30) * 1e3,
             "bwd_us": layer.bench_allreduce(1, rows, 30) * 1e3}
        res[rows] = {k: round(v, 2) for k, v in r.items()}
    # per-kernel timeline of a few small all-reduces (events around each launch on the comm stream)
    layer.set_profiling(True)
    layer.bench_allreduce(0, 16, 4)
    tl = layer.get_timeline()
    layer.set_profiling(False)
    layer.close()
    if rank == 0:
        t0 = tl[-12][2] if len(tl) >= 12 else 0.0
        print(json.dumps({"timeline_us": [(c, round((a - t0) * 1e3, 2), round((b - t0) * 1e3, 2)) for c, _, a, b in tl[-12:]]}))
        print(json.dumps({"T": world, "h": h, "two_shot_env": os.environ.get("MERAK_AR_TWO_SHOT"), "res": res}))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
