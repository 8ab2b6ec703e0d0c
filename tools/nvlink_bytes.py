"""NVLink hardware byte counters around the all-reduce (torchrun, T = WORLD_SIZE; NVLink evidence that ncu cannot
give for a multi-rank kernel).  Each rank reads its GPU's NVML NVLink counters (data TX / RX per link, summed over
the links) before and after `iters` all-reduces of one gpt20b sub-batch partial (rows x h bf16) through
merak_tmp_bench_allreduce, and the bytes per all-reduce are compared with the algorithm's bytes per GPU and
direction: one-shot (T-1) x msg, two-shot 2 (T-1)/T x msg.  Rank 0 prints one JSON line.
Env: H (hidden, default 6144), ROWS (default 4096), ITERS (default 50), MERAK_AR_TWO_SHOT / MERAK_AR_PUSH as for
the library."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_04959_b200 import TmpLayer  # noqa: E402


def nvlink_counters(dev_index):
    """Summed NVLink data TX / RX counters of one GPU (KiB throughput fields, else byte counters); None if absent."""
    try:
        import pynvml as nv
    except ImportError:
        return None
    nv.nvmlInit()
    hdl = nv.nvmlDeviceGetHandleByIndex(dev_index)
    out = {}
    for name, fid, scale in (("tx", nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, 1024),
                             ("rx", nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, 1024)):
        tot, ok = 0, False
        for link in range(18):
            try:
                v = nv.nvmlDeviceGetFieldValues(hdl, [(fid, link)])[0]
            except Exception:  # noqa: BLE001
                continue
            if v.nvmlReturn != 0:
                continue
            ok = True
            tot += int(v.value.ullVal) * scale
        out[name] = tot if ok else None
    return out


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    h = int(os.environ.get("H", 6144))
    rows = int(os.environ.get("ROWS", 4096))
    iters = int(os.environ.get("ITERS", 50))
    layer = TmpLayer(h, h // 96, 2048, 4, tmp_degree=world, tmp_rank=rank, n_sub=2, group=dist.group.WORLD)
    two = layer.debug_host()["two_shot"]
    push = layer.debug_host()["push"]
    msg = rows * h * 2
    algo = (2 * (world - 1) / world if two else (world - 1)) * msg
    phys = os.environ.get("CUDA_VISIBLE_DEVICES")
    nvml_index = int(phys.split(",")[local]) if phys else local
    res = {}
    for which, name in ((0, "fwd"), (1, "bwd")):
        layer.bench_allreduce(which, rows, 5)
        torch.cuda.synchronize()
        dist.barrier()
        c0 = nvlink_counters(nvml_index)
        ms = layer.bench_allreduce(which, rows, iters)
        torch.cuda.synchronize()
        c1 = nvlink_counters(nvml_index)
        r = {"us": ms * 1e3}
        if c0 and c1:
            for k in ("tx", "rx"):
                if c0[k] is not None and c1[k] is not None:
                    # merak_tmp_bench_allreduce runs 3 untimed warm-up all-reduces before the timed `iters`
                    r[f"{k}_bytes_per_ar"] = (c1[k] - c0[k]) / (iters + 3)
        gathered = [None] * world
        dist.all_gather_object(gathered, r)
        res[name] = gathered
    layer.close()
    if rank == 0:
        print(json.dumps({"T": world, "h": h, "rows": rows, "msg_bytes": msg, "two_shot": two, "push": push,
                          "algorithmic_bytes_per_gpu_direction": algo, "per_rank": res,
                          "note": "NVML NVLink data TX/RX counters (KiB fields x 1024) summed over links, "
                                  "difference over the iters + 3 (warm-up) all-reduces of the call; includes the "
                                  "handshake flag traffic"}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
