"""fp64 emulation of the *method's dataflow*: Megatron TMP sharding plus
sub-microbatch splitting, for the two invariants north_star fixes:

  (1) summing the row-parallel partial outputs across TMP ranks equals the
      unsharded layer ("divides weight matrices along row or column
      dimension with additional AllReduce operations"; P:558 two AllReduces in
      FP and two in BP);
  (2) splitting into sub-microbatches leaves every output and gradient
      unchanged ("evenly split each microbatch ... into two
      sub-microbatches, whose procedures are independent of each other").

TEST INFRASTRUCTURE ONLY (see oracle/layer.py header).  The partition rule is
this package's own implementation of DESIGN.md reading R8 (whole heads, ranks
r < H mod T take one extra head) and R9 (contiguous equal batch slices).
"""
from __future__ import annotations

import numpy as np

from .layer import (causal_attention, causal_attention_backward, gelu, gelu_grad, layer_norm,
                    layer_norm_backward)


def head_partition(H: int, T: int):
    """Reading R8: rank r owns H_r = H//T + (r < H % T) whole heads, contiguous, in rank order.
    Returns [(first_head, n_heads)] for r = 0..T-1."""
    if H < T:
        raise ValueError("H < T")
    out, start = [], 0
    for r in range(T):
        n = H // T + (1 if r < H % T else 0)
        out.append((start, n))
        start += n
    return out


def shard_params(params, heads: int, T: int, r: int):
    """Rank r's weight shard (SURVEY §8(b) layout):
      w_qkv_r = [q rows of its heads; k rows; v rows]  ([3 h_r, h]), b_qkv_r likewise;
      w_o_r = w_o[:, its head columns] ([h, h_r]);
      w_1_r = w_1[r f_r:(r+1) f_r, :], b_1_r likewise;  w_2_r = w_2[:, r f_r:(r+1) f_r];
      LN params, b_o, b_2 replicated."""
    h = params["w_o"].shape[0]
    f = params["w_1"].shape[0]
    d = h // heads
    if f % T:
        raise ValueError("f % T != 0")
    e0, ne = head_partition(heads, T)[r]
    cs = slice(e0 * d, (e0 + ne) * d)
    fr = f // T
    fs = slice(r * fr, (r + 1) * fr)
    wqkv, bqkv = params["w_qkv"], params["b_qkv"]
    out = dict(params)
    out["w_qkv"] = np.concatenate([wqkv[0 * h:1 * h][cs], wqkv[1 * h:2 * h][cs], wqkv[2 * h:3 * h][cs]], 0)
    out["b_qkv"] = np.concatenate([bqkv[0 * h:1 * h][cs], bqkv[1 * h:2 * h][cs], bqkv[2 * h:3 * h][cs]], 0)
    out["w_o"] = params["w_o"][:, cs]
    out["w_1"] = params["w_1"][fs]
    out["b_1"] = params["b_1"][fs]
    out["w_2"] = params["w_2"][:, fs]
    return out


def unshard_grads(rank_grads, heads: int, T: int):
    """Inverse of shard_params for gradients: place each rank's shard in the global tensor.
    Replicated grads (LN, b_o, b_2) are taken from rank 0 (they are identical on every rank)."""
    g0 = rank_grads[0]
    h = g0["w_o"].shape[0]
    d = h // heads
    out = {k: np.array(g0[k]) for k in ("ln1_g", "ln1_b", "ln2_g", "ln2_b", "b_o", "b_2")}
    fr = g0["w_1"].shape[0]
    f = fr * T
    wqkv = np.zeros((3 * h, h)); bqkv = np.zeros(3 * h)
    wo = np.zeros((h, h)); w1 = np.zeros((f, h)); b1 = np.zeros(f); w2 = np.zeros((h, f))
    for r, (e0, ne) in enumerate(head_partition(heads, T)):
        g = rank_grads[r]
        hr = ne * d
        cs = slice(e0 * d, (e0 + ne) * d)
        for blk in range(3):
            wqkv[blk * h:(blk + 1) * h][cs] = g["w_qkv"][blk * hr:(blk + 1) * hr]
            bqkv[blk * h:(blk + 1) * h][cs] = g["b_qkv"][blk * hr:(blk + 1) * hr]
        wo[:, cs] = g["w_o"]
        w1[r * fr:(r + 1) * fr] = g["w_1"]
        b1[r * fr:(r + 1) * fr] = g["b_1"]
        w2[:, r * fr:(r + 1) * fr] = g["w_2"]
    out.update(w_qkv=wqkv, b_qkv=bqkv, w_o=wo, w_1=w1, b_1=b1, w_2=w2)
    return out


def _allreduce(parts):
    """Sum in fixed rank order 0..T-1 (reading R10)."""
    acc = np.zeros_like(parts[0])
    for p in parts:
        acc = acc + p
    return acc


def sharded_fwd_bwd(params, x, dy, heads: int, T: int, n_sub: int):
    """The method's dataflow in fp64: for each sub-microbatch j (batch slice, R9) and each
    rank r, the column-parallel GEMMs/attention/GeLU on rank r's shard, the row-parallel
    partial products, and the all-reduce (rank-order sum) followed by the replicated
    bias/residual/LayerNorm work.  Backward mirrors it with the two backward all-reduces
    (fc1 dgrad, QKV dgrad).  Returns (y, dx, global grads, per-rank grads)."""
    x = np.asarray(x, np.float64)
    dy = np.asarray(dy, np.float64)
    p = {k: np.asarray(v, np.float64) for k, v in params.items()}
    B = x.shape[0]
    if B % n_sub:
        raise ValueError("B % n_sub != 0")
    b = B // n_sub
    shards = [shard_params(p, heads, T, r) for r in range(T)]
    parts = head_partition(heads, T)
    y = np.empty_like(x)
    dx = np.empty_like(x)
    rg = [{k: np.zeros_like(v) for k, v in s.items()} for s in shards]
    for j in range(n_sub):
        xs, dys = x[j * b:(j + 1) * b], dy[j * b:(j + 1) * b]
        # ---- forward: attention block
        u, xh1, rho1 = layer_norm(xs, p["ln1_g"], p["ln1_b"])
        caches, pa = [], []
        for r in range(T):
            s_ = shards[r]
            hr = parts[r][1] * (p["w_o"].shape[0] // heads)
            qkv = u @ s_["w_qkv"].T + s_["b_qkv"]
            q, k, v = qkv[..., :hr], qkv[..., hr:2 * hr], qkv[..., 2 * hr:]
            c, P = causal_attention(q, k, v, parts[r][1])
            caches.append(dict(q=q, k=k, v=v, c=c, P=P, hr=hr))
            pa.append(c @ s_["w_o"].T)                       # row-parallel partial (no bias)
        x1 = xs + _allreduce(pa) + p["b_o"]                  # AR#1 + bias + residual
        u2, xh2, rho2 = layer_norm(x1, p["ln2_g"], p["ln2_b"])
        pf = []
        for r in range(T):
            s_ = shards[r]
            z = u2 @ s_["w_1"].T + s_["b_1"]
            g = gelu(z)
            caches[r].update(z=z, g=g)
            pf.append(g @ s_["w_2"].T)
        y[j * b:(j + 1) * b] = x1 + _allreduce(pf) + p["b_2"]   # AR#2 + bias + residual
        # ---- backward: FFN block
        pd = []
        for r in range(T):
            s_, c_ = shards[r], caches[r]
            dz = (dys @ s_["w_2"]) * gelu_grad(c_["z"])
            rg[r]["w_2"] += dys.reshape(-1, dys.shape[-1]).T @ c_["g"].reshape(-1, c_["g"].shape[-1])
            rg[r]["w_1"] += dz.reshape(-1, dz.shape[-1]).T @ u2.reshape(-1, u2.shape[-1])
            rg[r]["b_1"] += dz.sum(axis=(0, 1))
            rg[r]["b_2"] += dys.sum(axis=(0, 1))
            pd.append(dz @ s_["w_1"])
        du2 = _allreduce(pd)                                  # AR#3
        dln2, dg2, db2 = layer_norm_backward(du2, xh2, rho2, p["ln2_g"])
        dx1 = dys + dln2
        pq = []
        for r in range(T):
            s_, c_ = shards[r], caches[r]
            rg[r]["ln2_g"] += dg2
            rg[r]["ln2_b"] += db2
            rg[r]["w_o"] += dx1.reshape(-1, dx1.shape[-1]).T @ c_["c"].reshape(-1, c_["c"].shape[-1])
            rg[r]["b_o"] += dx1.sum(axis=(0, 1))
            dc = dx1 @ s_["w_o"]
            dq, dk, dv = causal_attention_backward(dc, c_["q"], c_["k"], c_["v"], c_["P"], parts[r][1])
            dqkv = np.concatenate([dq, dk, dv], -1)
            rg[r]["w_qkv"] += dqkv.reshape(-1, dqkv.shape[-1]).T @ u.reshape(-1, u.shape[-1])
            rg[r]["b_qkv"] += dqkv.sum(axis=(0, 1))
            pq.append(dqkv @ s_["w_qkv"])
        du = _allreduce(pq)                                   # AR#4
        dln1, dg1, db1 = layer_norm_backward(du, xh1, rho1, p["ln1_g"])
        for r in range(T):
            rg[r]["ln1_g"] += dg1
            rg[r]["ln1_b"] += db1
        dx[j * b:(j + 1) * b] = dx1 + dln1
    return y, dx, unshard_grads(rg, heads, T), rg
