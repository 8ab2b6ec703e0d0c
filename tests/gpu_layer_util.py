"""Helpers for layer-level GPU parity tests: run the C-ABI layer on seeded inputs and compare with
the fp64 oracle.  Test infrastructure only."""
from __future__ import annotations

import numpy as np
import torch

from paper_2206_04959_b200 import PARAM_NAMES, TmpLayer, shard_weights, zero_grads_like

TOL_BF16 = 2e-2  # north_star: relative Frobenius error <= 2e-2 for bf16 with fp32 accumulation
TOL_FP32 = 1e-5  # north_star: <= 1e-5 for the fp32 check mode


def rel_err(gpu, ref) -> float:
    g = np.asarray(gpu, dtype=np.float64)
    r = np.asarray(ref, dtype=np.float64)
    return float(np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-300))


def run_gpu_layer(cfg, params, x, dy, T=1, rank=0, n_sub=None, group=None, reps=1, flags=0, device=None, comm=0,
                  precision=0):
    """Forward + backward through merak_tmp_layer_fwd/bwd.  Returns dict of torch tensors on device:
    y, dx and the rank's fp32 gradient shards.  precision=1: MERAK_FP32_CHECK (fp32 tensors)."""
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    n = cfg.n_sub if n_sub is None else n_sub
    layer = TmpLayer(cfg.hidden, cfg.heads, cfg.seq_len, cfg.microbatch, tmp_degree=T, tmp_rank=rank, n_sub=n,
                     device=dev.index, group=group, comm=comm, precision=precision)
    dt = torch.float32 if precision == 1 else torch.bfloat16
    w = shard_weights(params, cfg.heads, T, rank, dev, dtype=dt)
    M, h = cfg.tokens, cfg.hidden
    X = torch.as_tensor(np.asarray(x).reshape(M, h)).to(dev, dt)
    DY = torch.as_tensor(np.asarray(dy).reshape(M, h)).to(dev, dt)
    Y = torch.empty_like(X)
    DX = torch.empty_like(X)
    saved = layer.new_saved()
    out = None
    for _ in range(reps):
        grads = zero_grads_like(w)
        layer.forward(w, X, Y, saved, flags=flags)
        layer.backward(w, X, saved, DY, DX, grads, flags=flags)
        torch.cuda.synchronize()
        out = {"y": Y.clone(), "dx": DX.clone(), **{k: grads[k].clone() for k in PARAM_NAMES}}
    layer.close()
    return out


def oracle_rank_slices(grads_global, cfg, T, rank):
    """Slice the oracle's global fp64 gradients to rank `rank`'s shard using the oracle's own partition."""
    from oracle import shard_params
    return shard_params(grads_global, cfg.heads, T, rank)


def compare_to_oracle(out, y_ref, dx_ref, grads_ref_rank, cfg, tol=TOL_BF16):
    """Relative Frobenius error per tensor; b_qkv compared as one packed tensor (its k-slice is 0)."""
    M, h = cfg.tokens, cfg.hidden
    errs = {"y": rel_err(out["y"].float().cpu().numpy(), np.asarray(y_ref).reshape(M, h)),
            "dx": rel_err(out["dx"].float().cpu().numpy(), np.asarray(dx_ref).reshape(M, h))}
    for k in PARAM_NAMES:
        errs[k] = rel_err(out[k].cpu().numpy(), grads_ref_rank[k])
    bad = {k: v for k, v in errs.items() if not (v <= tol)}
    return errs, bad


def run_gpu_chain(cfg, params_list, x, dy, T=1, rank=0, group=None, chain=True, n_sub=None, recompute=None,
                  early=False):
    """K stacked layers through the C ABI: forward 0..K-1, backward K-1..0.  chain=True passes
    MERAK_FLAG_CHAIN on every call but the last backward (cross-layer overlap, the bench's mode), so
    the library's cross-layer event hazards (workspace reuse between layers) are exercised.
    recompute: per-layer bools -- those layers write their forward activations into ONE shared scratch
    buffer and regenerate them in the backward (MERAK_FLAG_RECOMPUTE); early=True runs the regeneration as
    a separate forward call (MERAK_FLAG_RECOMPUTE on layer_fwd) just before the layer's backward.
    Returns dict: y (last layer), dx (first layer), grads[k]."""
    from paper_2206_04959_b200 import FLAG_CHAIN, FLAG_RECOMPUTE
    dev = torch.device("cuda", torch.cuda.current_device())
    K = len(params_list)
    n = cfg.n_sub if n_sub is None else n_sub
    layer = TmpLayer(cfg.hidden, cfg.heads, cfg.seq_len, cfg.microbatch, tmp_degree=T, tmp_rank=rank, n_sub=n,
                     device=dev.index, group=group)
    ws = [shard_weights(p, cfg.heads, T, rank, dev) for p in params_list]
    M, h = cfg.tokens, cfg.hidden
    X = torch.as_tensor(np.asarray(x).reshape(M, h)).to(dev, torch.bfloat16)
    DY = torch.as_tensor(np.asarray(dy).reshape(M, h)).to(dev, torch.bfloat16)
    Ys = [torch.empty_like(X) for _ in range(K)]
    DXs = [torch.empty_like(X) for _ in range(K)]
    grads = [zero_grads_like(w) for w in ws]
    rc = list(recompute) if recompute is not None else [False] * K
    scratch = layer.new_saved() if any(rc) else None
    saved = [scratch if rc[k] else layer.new_saved() for k in range(K)]
    f = FLAG_CHAIN if chain else 0
    for k in range(K):
        layer.forward(ws[k], X if k == 0 else Ys[k - 1], Ys[k], saved[k], flags=f)
    if scratch is not None:  # nothing may depend on what the forwards left in the scratch buffer
        layer.join()  # a chained forward's AR#2 epilogue (reads its saved x1) is launched by the next call / join
        torch.cuda.synchronize()
        scratch.fill_(0xFF)
    for k in reversed(range(K)):
        xin = X if k == 0 else Ys[k - 1]
        bf = f if k > 0 else 0
        if rc[k] and early:
            layer.forward(ws[k], xin, None, saved[k], flags=f | FLAG_RECOMPUTE)
        elif rc[k]:
            bf |= FLAG_RECOMPUTE
        layer.backward(ws[k], xin, saved[k], DY if k == K - 1 else DXs[k + 1], DXs[k], grads[k], flags=bf)
    torch.cuda.synchronize()
    out = {"y": Ys[K - 1].clone(), "dx": DXs[0].clone(), "grads": [{k: g[k].clone() for k in PARAM_NAMES}
                                                                  for g in grads]}
    layer.close()
    return out


def oracle_chain(params_list, x, dy, heads):
    """fp64 composition of the oracle layer: forward through all layers, backward in reverse."""
    from oracle.layer import layer_backward, layer_forward
    caches, h_in = [], x
    for p in params_list:
        h_in, c = layer_forward(p, h_in, heads)
        caches.append(c)
    y = h_in
    grads = [None] * len(params_list)
    g = dy
    for k in reversed(range(len(params_list))):
        g, grads[k] = layer_backward(params_list[k], caches[k], g, heads)
    return y, g, grads


def run_gpu_group(cfg, params, x, dy, T, n_sub=None, precision=0, flags=0, chain_params=None, chain=True):
    """The T ranks of a TMP group as handles of this process on one GPU (merak_tmp_init_group,
    MERAK_COMM_INPROC): each rank holds its own weight shard and outputs, every all-reduce sums the T
    ranks' partials through the peer kernels.  Each rank issues its calls on its own caller stream (the
    library defers each call until every rank made it, then issues the set together).  chain_params: list of per-layer params -> K chained layers (MERAK_FLAG_CHAIN on every
    call but the last backward; chain=False: no chaining), else one layer with `params`.
    Returns [per-rank dict]: y, dx and the rank's gradient shards (grads[k] per layer when chained)."""
    from paper_2206_04959_b200 import FLAG_CHAIN
    dev = torch.device("cuda", torch.cuda.current_device())
    n = cfg.n_sub if n_sub is None else n_sub
    ranks = TmpLayer.group(cfg.hidden, cfg.heads, cfg.seq_len, cfg.microbatch, T, n_sub=n, device=dev.index,
                           precision=precision)
    dt = torch.float32 if precision == 1 else torch.bfloat16
    plist = chain_params if chain_params is not None else [params]
    K = len(plist)
    ws = [[shard_weights(p, cfg.heads, T, r, dev, dtype=dt) for p in plist] for r in range(T)]
    M, h = cfg.tokens, cfg.hidden
    X = torch.as_tensor(np.asarray(x).reshape(M, h)).to(dev, dt)
    DY = torch.as_tensor(np.asarray(dy).reshape(M, h)).to(dev, dt)
    Ys = [[torch.empty_like(X) for _ in range(K)] for _ in range(T)]
    DXs = [[torch.empty_like(X) for _ in range(K)] for _ in range(T)]
    grads = [[zero_grads_like(w) for w in ws[r]] for r in range(T)]
    saved = [[ranks[r].new_saved() for _ in range(K)] for r in range(T)]
    streams = [torch.cuda.Stream(device=dev) for _ in range(T)]
    for s in streams:
        s.wait_stream(torch.cuda.current_stream())
    cf = FLAG_CHAIN if chain_params is not None and chain else 0
    for k in range(K):
        for r in range(T):
            ranks[r].forward(ws[r][k], X if k == 0 else Ys[r][k - 1], Ys[r][k], saved[r][k], flags=flags | cf,
                             stream=streams[r])
    for k in reversed(range(K)):
        for r in range(T):
            ranks[r].backward(ws[r][k], X if k == 0 else Ys[r][k - 1], saved[r][k],
                              DY if k == K - 1 else DXs[r][k + 1], DXs[r][k], grads[r][k],
                              flags=flags | (cf if k > 0 else 0), stream=streams[r])
    torch.cuda.synchronize()
    outs = []
    for r in range(T):
        o = {"y": Ys[r][K - 1].clone(), "dx": DXs[r][0].clone()}
        if chain_params is None:
            o.update({k: grads[r][0][k].clone() for k in PARAM_NAMES})
        else:
            o["grads"] = [{k: g[k].clone() for k in PARAM_NAMES} for g in grads[r]]
        outs.append(o)
    for lay in ranks:
        lay.close()
    return outs
