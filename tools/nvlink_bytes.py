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


def _nvml_fields(dev_index):
    """Summed NVLink TX / RX bytes over the links from NVML field values; tries the byte counters first, then the
    KiB data-throughput fields.  Returns ({"tx": bytes, "rx": bytes, "source": name}, diagnostics)."""
    try:
        import pynvml as nv
    except ImportError:
        return None, "no pynvml"
    nv.nvmlInit()
    hdl = nv.nvmlDeviceGetHandleByIndex(dev_index)
    diag = {}
    for src, ftx, frx, scale in (("COUNT_BYTES", nv.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES,
                                  nv.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES, 1),
                                 ("THROUGHPUT_DATA_KiB", nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
                                  nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, 1024)):
        out, ok = {}, True
        for name, fid in (("tx", ftx), ("rx", frx)):
            tot, n = 0, 0
            for link in range(18):
                try:
                    v = nv.nvmlDeviceGetFieldValues(hdl, [(fid, link)])[0]
                except Exception as e:  # noqa: BLE001
                    diag[f"{src}/{name}/{link}"] = repr(e)[:80]
                    continue
                if v.nvmlReturn != 0:
                    diag[f"{src}/{name}/{link}"] = int(v.nvmlReturn)
                    continue
                tot += int(v.value.ullVal) * scale
                n += 1
            ok = ok and n > 0
            out[name] = tot
        if ok:
            out["source"] = "NVML " + src
            return out, None
    return None, dict(list(diag.items())[:6])


def _smi(dev_index):
    """`nvidia-smi nvlink -gt d -i N`: per-link 'Data Tx / Rx' counters in KiB, summed."""
    import re
    import subprocess
    try:
        txt = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(dev_index)], capture_output=True,
                             text=True, timeout=30).stdout
    except Exception as e:  # noqa: BLE001
        return None, repr(e)[:80]
    tx = sum(int(v) for v in re.findall(r"Tx:\s*(\d+)\s*KiB", txt))
    rx = sum(int(v) for v in re.findall(r"Rx:\s*(\d+)\s*KiB", txt))
    if not re.search(r"Tx:\s*\d+", txt):
        return None, txt[:200]
    return {"tx": tx * 1024, "rx": rx * 1024, "source": "nvidia-smi nvlink -gt d"}, None


def nvlink_counters(dev_index):
    c, d1 = _nvml_fields(dev_index)
    if c:
        return c, None
    c, d2 = _smi(dev_index)
    return c, {"nvml": d1, "smi": d2}


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
    push = layer.debug_host()["push"] and two and (rows // world) % 32 == 0
    msg = rows * h * 2
    # bench_allreduce zeroes the slot and runs the all-reduce alone: with the push, the reduce-scatter half would
    # travel inside the GEMM, so only the all-gather half moves here
    algo = ((world - 1) / world if push else 2 * (world - 1) / world if two else (world - 1)) * msg
    phys = os.environ.get("CUDA_VISIBLE_DEVICES")
    nvml_index = int(phys.split(",")[local]) if phys else local
    res = {}
    for which, name in ((0, "fwd"), (1, "bwd")):
        layer.bench_allreduce(which, rows, 5)
        torch.cuda.synchronize()
        dist.barrier()
        c0, diag = nvlink_counters(nvml_index)
        ms = layer.bench_allreduce(which, rows, iters)
        torch.cuda.synchronize()
        c1, _ = nvlink_counters(nvml_index)
        r = {"us": ms * 1e3}
        if c0 and c1:
            r["source"] = c0["source"]
            for k in ("tx", "rx"):
                # merak_tmp_bench_allreduce runs 3 untimed warm-up all-reduces before the timed `iters`
                r[f"{k}_bytes_per_ar"] = (c1[k] - c0[k]) / (iters + 3)
        else:
            r["counters_unavailable"] = diag
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
