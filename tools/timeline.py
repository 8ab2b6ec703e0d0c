"""Two-stream timeline of one chained K-layer step (the fig:pipedtp(b) analog).

torchrun --nproc-per-node T tools/timeline.py   (or plain python for T = 1)
Prints per-stream busy time, all-reduce time overlapped with compute, and an ASCII Gantt of
rank 0; writes gpurun_out/timeline_T{T}_n{n}.json.  Event timestamps bracket each launch on its own
stream (cudaEventRecord), so a bracket includes any wait for SM resources."""
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2206_04959_b200 import FLAG_CHAIN, TmpLayer, shard_weights, zero_grads_like  # noqa: E402
from synth import CONFIGS, make_activations, make_params  # noqa: E402


def union(iv):
    iv = sorted(iv)
    out = []
    for a, b in iv:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def overlap(a, b):
    tot, j = 0.0, 0
    for x0, x1 in a:
        for y0, y1 in b:
            tot += max(0.0, min(x1, y1) - max(x0, y0))
    return tot


def main():
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD
    n = int(os.environ.get("NSUB", 2))
    K = int(os.environ.get("K", 4))
    cfg = CONFIGS[os.environ.get("CFG", "gpt1.5b")].with_(tmp_degree=world, n_sub=n)
    x, dy = make_activations(cfg)
    ws = [shard_weights(make_params(cfg, layer=k), cfg.heads, world, rank, dev) for k in range(K)]
    M, h = cfg.tokens, cfg.hidden
    X = torch.as_tensor(x.reshape(M, h)).to(dev, torch.bfloat16)
    DY = torch.as_tensor(dy.reshape(M, h)).to(dev, torch.bfloat16)
    Ys = [torch.empty_like(X) for _ in range(K)]
    DXs = [torch.empty_like(X) for _ in range(K)]
    grads = [zero_grads_like(w) for w in ws]
    layer = TmpLayer(cfg.hidden, cfg.heads, cfg.seq_len, cfg.microbatch, tmp_degree=world, tmp_rank=rank, n_sub=n,
                     device=rank, group=group)
    saved = [layer.new_saved() for _ in range(K)]

    def step():
        for k in range(K):
            layer.forward(ws[k], X if k == 0 else Ys[k - 1], Ys[k], saved[k], flags=FLAG_CHAIN)
        for k in reversed(range(K)):
            layer.backward(ws[k], X if k == 0 else Ys[k - 1], saved[k], DY if k == K - 1 else DXs[k + 1], DXs[k],
                           grads[k], flags=FLAG_CHAIN if k > 0 else 0)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    layer.set_profiling(True)
    step()
    tl = layer.get_timeline()
    layer.set_profiling(False)
    comp = union([[a, b] for c, s, a, b in tl if s in ("comp", "wgrad")])
    comm = union([[a, b] for c, s, a, b in tl if s == "comm" and c == "allreduce"])
    span = max(b for _, _, _, b in tl)
    busy_comp = sum(b - a for a, b in comp)
    busy_comm = sum(b - a for a, b in comm)
    ov = overlap(comm, comp)
    res = {"rank": rank, "T": world, "n_sub": n, "K": K, "step_ms": span, "compute_busy_ms": busy_comp,
           "allreduce_busy_ms": busy_comm, "allreduce_overlapped_ms": ov, "allreduce_exposed_ms": busy_comm - ov,
           "compute_idle_ms": span - busy_comp, "launches": len(tl)}
    if rank == 0:
        print(json.dumps(res))
        # ASCII Gantt of the first layer's forward (both streams)
        width = 160
        end = max(b for c, s, a, b in tl[: len(tl) // (2 * K)] if True) if tl else 1.0
        for name in ("comp", "wgrad", "comm"):
            row = [" "] * width
            for c, s, a, b in tl:
                if s != name or a > end:
                    continue
                ch = {"gemm": "G", "attn_fwd": "A", "attn_bwd": "a", "layernorm": "L", "allreduce": "R",
                      "reduce": "r"}[c]
                for i in range(int(a / end * (width - 1)), min(width, int(b / end * (width - 1)) + 1)):
                    row[i] = ch
            print(f"{name:>5} |" + "".join(row) + "|")
        print(f"        0 ms{' ' * (width - 16)}{end:.3f} ms  (first layer forward, rank 0)")
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        json.dump({"summary": res, "timeline": tl}, open(os.path.join(ROOT, "gpurun_out",
                                                                     f"timeline_T{world}_n{n}.json"), "w"))
    layer.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
