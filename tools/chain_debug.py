"""Debug helper (torchrun, T = WORLD_SIZE): K chained layers with host copies, sync + print per phase."""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_04959_b200 import FLAG_CHAIN, TmpLayer, shard_weights, zero_grads_like  # noqa: E402
from synth import CONFIGS, make_activations, make_params  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    cfg = CONFIGS[os.environ.get("CFG", "gpt1.5b")].with_(tmp_degree=world)
    K = int(os.environ.get("K", 4))
    x, dy = make_activations(cfg)
    ws = [shard_weights(make_params(cfg, layer=k), cfg.heads, world, rank, dev) for k in range(K)]
    M, h = cfg.tokens, cfg.hidden
    X = torch.as_tensor(x.reshape(M, h)).to(dev, torch.bfloat16)
    DY = torch.as_tensor(dy.reshape(M, h)).to(dev, torch.bfloat16)
    Ys = [torch.empty_like(X) for _ in range(K)]
    DXs = [torch.empty_like(X) for _ in range(K)]
    grads = [zero_grads_like(w) for w in ws]
    layer = TmpLayer(cfg.hidden, cfg.heads, cfg.seq_len, cfg.microbatch, tmp_degree=world, tmp_rank=rank,
                     n_sub=cfg.n_sub, device=rank, group=dist.group.WORLD)
    saved = [layer.new_saved() for _ in range(K)]

    def say(m):
        print(f"[rank {rank}] {time.time():.2f} {m}", flush=True)

    def step(xi, dyi, chain=True, extra=0):
        for k in range(K):
            layer.forward(ws[k], xi if k == 0 else Ys[k - 1], Ys[k], saved[k],
                          flags=(FLAG_CHAIN if chain else 0) | extra)
        for k in reversed(range(K)):
            layer.backward(ws[k], xi if k == 0 else Ys[k - 1], saved[k], dyi if k == K - 1 else DXs[k + 1], DXs[k],
                           grads[k], flags=(FLAG_CHAIN if (chain and k > 0) else 0) | extra)

    for i in range(3):
        step(X, DY)
        torch.cuda.synchronize()
        say(f"plain step {i} ok")
    for i in range(2):
        step(X, DY, extra=2)
        torch.cuda.synchronize()
        say(f"no-comm step {i} ok")
    step(X, DY)
    torch.cuda.synchronize()
    say("plain after no-comm ok")
    layer.set_subbatches(1)
    for i in range(2):
        step(X, DY)
        torch.cuda.synchronize()
        say(f"n=1 step {i} ok")
    layer.set_subbatches(cfg.n_sub)
    for i in range(2):
        step(X, DY)
        torch.cuda.synchronize()
        say(f"back to n={cfg.n_sub} step {i} ok")
    hx, hdy = X.cpu().pin_memory(), DY.cpu().pin_memory()
    hy, hdx = torch.empty_like(hx).pin_memory(), torch.empty_like(hx).pin_memory()
    Xe, DYe = torch.empty_like(X), torch.empty_like(DY)
    for i in range(3):
        Xe.copy_(hx, non_blocking=True)
        DYe.copy_(hdy, non_blocking=True)
        step(Xe, DYe)
        hy.copy_(Ys[K - 1], non_blocking=True)
        hdx.copy_(DXs[0], non_blocking=True)
        torch.cuda.synchronize()
        say(f"copy step {i} ok")
    for i in range(3):
        Xe.copy_(hx, non_blocking=True)
        DYe.copy_(hdy, non_blocking=True)
        step(Xe, DYe)
        hy.copy_(Ys[K - 1], non_blocking=True)
        hdx.copy_(DXs[0], non_blocking=True)
        say(f"copy step (no sync) {i} issued")
    torch.cuda.synchronize()
    say("all ok")
    layer.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
