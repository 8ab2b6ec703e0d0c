"""Pins for the fp64 oracle (CPU, -m "not gpu").

The oracle is checked against things other than itself:
  * brute-force central finite differences on the tiny config (every gradient);
  * torch fp64 autograd over library routines (F.layer_norm, SDPA is_causal, gelu tanh);
  * closed forms (position-0 attention, uniform attention, zero weights, d b_k == 0,
    LN-backward row sums, GeLU special values and the erf-GeLU bound);
  * the two invariants north_star fixes (sharded sum == unsharded; sub-batching).
A plausible slip (dropped term, wrong sign/index, transposed operand) fails one of these.
"""
import math

import numpy as np
import pytest
import scipy.special

from oracle import (causal_attention, gelu, gelu_grad, head_partition, layer_backward, layer_forward, layer_fwd_bwd,
                    layer_norm, layer_norm_backward, shard_params, sharded_fwd_bwd)
from synth import CONFIGS, make_all

TINY = CONFIGS["tiny"]


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def tiny():
    params, x, dy = make_all(TINY)
    params = {k: v.astype(np.float64) for k, v in params.items()}
    return params, x.astype(np.float64), dy.astype(np.float64)


def _loss(params, x, dy, heads):
    y, _ = layer_forward(params, x, heads)
    return float((y * dy).sum())


# ----------------------------------------------------------------------------- finite differences
def test_fd_directional_all_tensors(tiny):
    """<grad, v> vs (L(theta+eps v) - L(theta-eps v)) / 2 eps for random directions v,
    for x and each of the 12 parameter tensors (L = sum y * dy so grad = backward(dy))."""
    params, x, dy = tiny
    H = TINY.heads
    _, dx, grads = layer_fwd_bwd(params, x, dy, H)
    rng = np.random.default_rng(7)
    eps = 1e-6
    names = ["x"] + list(params)
    for name in names:
        for _ in range(3):
            base = x if name == "x" else params[name]
            v = rng.standard_normal(base.shape)
            g = dx if name == "x" else grads[name]
            an = float((g * v).sum())

            def L(sign):
                if name == "x":
                    return _loss(params, x + sign * eps * v, dy, H)
                p2 = dict(params)
                p2[name] = params[name] + sign * eps * v
                return _loss(p2, x, dy, H)

            fd = (L(+1) - L(-1)) / (2 * eps)
            assert abs(fd - an) <= 1e-6 * abs(an) + 1e-7, (name, fd, an)


def test_fd_per_coordinate_sample(tiny):
    """Per-coordinate central differences on a random sample of coordinates of every tensor
    (catches a wrong index that a random direction could average out)."""
    params, x, dy = tiny
    H = TINY.heads
    _, dx, grads = layer_fwd_bwd(params, x, dy, H)
    rng = np.random.default_rng(11)
    eps = 1e-5  # |L| ~ 50: roundoff ~ 1e-14 |L| / eps, truncation ~ eps^2
    for name in ["x"] + list(params):
        base = x if name == "x" else params[name]
        g = dx if name == "x" else grads[name]
        flat_idx = rng.choice(base.size, size=min(base.size, 24), replace=False)
        for fi in flat_idx:
            idx = np.unravel_index(fi, base.shape)

            def L(sign):
                b2 = base.copy()
                b2[idx] += sign * eps
                if name == "x":
                    return _loss(params, b2, dy, H)
                p2 = dict(params)
                p2[name] = b2
                return _loss(p2, x, dy, H)

            fd = (L(+1) - L(-1)) / (2 * eps)
            assert abs(fd - g[idx]) <= 1e-5 * abs(g[idx]) + 5e-8, (name, idx, fd, g[idx])


# ----------------------------------------------------------------------------- independent library
def _torch_layer(params, x, dy, heads):
    import torch
    import torch.nn.functional as F
    P = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in params.items()}
    X = torch.tensor(x, dtype=torch.float64, requires_grad=True)
    B, s, h = x.shape
    d = h // heads
    u = F.layer_norm(X, (h,), P["ln1_g"], P["ln1_b"], eps=1e-5)
    qkv = F.linear(u, P["w_qkv"], P["b_qkv"])
    q, k, v = qkv.split(h, dim=-1)
    sh = lambda t: t.view(B, s, heads, d).transpose(1, 2)
    c = F.scaled_dot_product_attention(sh(q), sh(k), sh(v), is_causal=True)
    c = c.transpose(1, 2).reshape(B, s, h)
    x1 = X + F.linear(c, P["w_o"], P["b_o"])
    u2 = F.layer_norm(x1, (h,), P["ln2_g"], P["ln2_b"], eps=1e-5)
    g = F.gelu(F.linear(u2, P["w_1"], P["b_1"]), approximate="tanh")
    y = x1 + F.linear(g, P["w_2"], P["b_2"])
    y.backward(torch.tensor(dy, dtype=torch.float64))
    return (y.detach().numpy(), X.grad.numpy(), {k: t.grad.numpy() for k, t in P.items()})


@pytest.mark.parametrize("shape", [(2, 16, 64, 2), (2, 40, 96, 3), (1, 128, 256, 4)])
def test_torch_fp64_autograd(shape):
    B, s, h, H = shape
    cfg = TINY.with_(hidden=h, heads=H, seq_len=s, microbatch=B)
    params, x, dy = make_all(cfg, seed=1234 + h)
    y, dx, grads = layer_fwd_bwd(params, x, dy, H)
    ty, tdx, tg = _torch_layer(params, x, dy, H)
    assert rel(y, ty) < 1e-12
    assert rel(dx, tdx) < 1e-12
    for k in grads:
        if k == "b_qkv":
            continue
        assert rel(grads[k], tg[k]) < 1e-10, k
    # b_qkv: its k-slice is identically zero (shift invariance), compare the packed tensor absolutely
    assert np.abs(grads["b_qkv"] - tg["b_qkv"]).max() < 1e-10 * np.abs(tg["b_qkv"]).max()


# ----------------------------------------------------------------------------- closed forms
def test_attention_position0_and_uniform():
    rng = np.random.default_rng(3)
    B, s, H, d = 2, 12, 3, 8
    q = rng.standard_normal((B, s, H * d))
    k = rng.standard_normal((B, s, H * d))
    v = rng.standard_normal((B, s, H * d))
    c, P = causal_attention(q, k, v, H)
    # position 0 attends only to itself -> c[:,0] == v[:,0] exactly
    assert np.array_equal(c[:, 0], v[:, 0])
    # masked probabilities are exactly zero; rows sum to 1
    assert np.all(P[..., np.triu_indices(s, 1)[0], np.triu_indices(s, 1)[1]] == 0)
    assert np.allclose(P.sum(-1), 1.0, atol=1e-14)
    # k == 0 -> uniform causal average c[i] = mean_{j<=i} v[j]
    c0, _ = causal_attention(q, np.zeros_like(k), v, H)
    expect = np.cumsum(v, axis=1) / np.arange(1, s + 1)[None, :, None]
    assert np.allclose(c0, expect, rtol=0, atol=1e-13)


def test_key_bias_grad_is_zero(tiny):
    """softmax is shift-invariant per row, so d b_k == 0 (q_i . b_k is constant over keys)."""
    params, x, dy = tiny
    _, _, g = layer_fwd_bwd(params, x, dy, TINY.heads)
    h = TINY.hidden
    dbq, dbk = g["b_qkv"][:h], g["b_qkv"][h:2 * h]
    assert np.abs(dbk).max() <= 1e-12 * np.abs(dbq).max()
    assert np.abs(dbq).max() > 1e-4


def test_layer_norm_closed_forms():
    rng = np.random.default_rng(5)
    x = rng.standard_normal((7, 33)) * 3 + 1.5
    u, xhat, rho = layer_norm(x, np.ones(33), np.zeros(33))
    var = x.var(axis=-1)  # numpy biased variance: an independent routine
    assert np.allclose(rho[:, 0], 1 / np.sqrt(var + 1e-5), rtol=1e-14)
    assert np.allclose(u.mean(-1), 0, atol=1e-14)
    assert np.allclose(u.var(-1), var / (var + 1e-5), rtol=1e-12)
    du = rng.standard_normal(x.shape)
    dx, dg, db = layer_norm_backward(du, xhat, rho, rng.uniform(0.5, 1.5, 33))
    assert np.abs(dx.sum(-1)).max() < 1e-13 * np.abs(dx).max() * 33  # rows of dx sum to 0
    assert np.allclose(db, du.sum(0)) and np.allclose(dg, (du * xhat).sum(0))


def test_gelu_special_values():
    assert gelu(np.array(0.0)) == 0.0
    assert gelu_grad(np.array(0.0)) == 0.5
    z = np.array([8.0, 12.0])
    assert np.allclose(gelu(z), z, rtol=1e-12) and np.allclose(gelu_grad(z), 1.0, atol=1e-12)
    assert np.allclose(gelu(-z), 0.0, atol=1e-12)
    # tanh approximation vs the exact erf GeLU (scipy): |diff| < 5e-4 over [-6, 6]
    t = np.linspace(-6, 6, 2001)
    exact = 0.5 * t * (1 + scipy.special.erf(t / math.sqrt(2)))
    assert np.abs(gelu(t) - exact).max() < 5e-4
    # derivative vs central differences
    e = 1e-6
    assert np.allclose(gelu_grad(t), (gelu(t + e) - gelu(t - e)) / (2 * e), atol=1e-8)


def test_zero_output_weights(tiny):
    """W_o = W_2 = 0  =>  y = x + b_o + b_2 and dx = dy exactly."""
    params, x, dy = tiny
    p = dict(params)
    p["w_o"] = np.zeros_like(p["w_o"])
    p["w_2"] = np.zeros_like(p["w_2"])
    y, dx, g = layer_fwd_bwd(p, x, dy, TINY.heads)
    assert np.array_equal(y, x + p["b_o"] + p["b_2"])
    assert np.array_equal(dx, dy)
    assert np.all(g["w_1"] == 0) and np.all(g["w_qkv"] == 0)


# ----------------------------------------------------------------------------- invariants
def test_head_partition():
    assert head_partition(25, 2) == [(0, 13), (13, 12)]
    assert head_partition(25, 8) == [(0, 4), (4, 3), (7, 3), (10, 3), (13, 3), (16, 3), (19, 3), (22, 3)]
    assert head_partition(32, 4) == [(0, 8), (8, 8), (16, 8), (24, 8)]
    with pytest.raises(ValueError):
        head_partition(2, 4)


@pytest.mark.parametrize("T,n,h,H", [(1, 1, 80, 5), (2, 1, 80, 5), (2, 2, 80, 5), (4, 2, 80, 5), (3, 4, 96, 6),
                                     (4, 4, 96, 6), (3, 2, 120, 5)])
def test_invariant_sharded_equals_unsharded(T, n, h, H):
    """(1) sum of row-parallel partials over ranks == unsharded layer, incl. uneven head
    splits (H=5 at T=2: 3/2, T=4: 2/1/1/1; H=6 at T=4: 2/2/1/1; H=5 at T=3: 2/2/1);
    (2) sub-batching leaves outputs and grads unchanged."""
    cfg = TINY.with_(hidden=h, heads=H, seq_len=12, microbatch=4)
    assert cfg.ffn % T == 0 and cfg.hidden % cfg.heads == 0
    params, x, dy = make_all(cfg, seed=99)
    y, dx, g = layer_fwd_bwd(params, x, dy, cfg.heads)
    ys, dxs, gs, _ = sharded_fwd_bwd(params, x, dy, cfg.heads, T, n)
    assert rel(ys, y) < 1e-14
    assert rel(dxs, dx) < 1e-14
    for k in g:
        tol = 1e-13 if k != "b_qkv" else None
        if tol:
            assert rel(gs[k], g[k]) < tol, k
        else:
            assert np.abs(gs[k] - g[k]).max() < 1e-13 * np.abs(g[k]).max()


def test_sub_batching_forward_per_sample_exact():
    """Samples are independent: the forward of sample i does not depend on others."""
    cfg = TINY.with_(microbatch=4)
    params, x, dy = make_all(cfg, seed=5)
    y, _ = layer_forward(params, x, cfg.heads)
    for i in range(4):
        yi, _ = layer_forward(params, x[i:i + 1], cfg.heads)
        assert np.allclose(yi[0], y[i], rtol=0, atol=1e-14)


def test_shard_params_layout():
    cfg = TINY.with_(hidden=80, heads=5)
    params, _, _ = make_all(cfg, seed=2)
    s = shard_params(params, 5, 2, 1)  # rank 1 owns heads 3,4 -> columns 48..80
    h, d = 80, 16
    assert s["w_qkv"].shape == (3 * 32, 80)
    assert np.array_equal(s["w_qkv"][32:64], params["w_qkv"][h + 48:h + 80])
    assert np.array_equal(s["w_o"], params["w_o"][:, 48:80])
    assert np.array_equal(s["w_1"], params["w_1"][160:320])


def test_layer_flops_pin():
    """oracle.layer_flops against an independent tally: every GEMM of the layer enumerated by its
    (M, N, K) (forward QKV / proj / fc1 / fc2, each also as dgrad and wgrad in the backward), and the
    causal attention products counted pair by pair (key j <= query i, diagonal included, reading R4):
    QK^T and PV forward, dV, dP, dQ, dK backward, d multiply-adds each.  Also the closed form
    72 B s h^2 + 6 B h s (s+1) at the BASELINE shapes (the per-GPU values SURVEY §8 tabulates x T)."""
    from oracle import layer_flops
    for (B, s, h, H) in [(2, 16, 64, 2), (3, 20, 96, 6), (1, 33, 80, 5)]:
        f, M, d = 4 * h, B * s, h // H
        fwd = [(M, 3 * h, h), (M, h, h), (M, f, h), (M, h, f)]
        gemm = sum(2 * m * nn * k for (m, nn, k) in fwd) * 3  # fwd + dgrad + wgrad: same M*N*K each
        pairs = sum(1 for i in range(s) for j in range(s) if j <= i)
        attn = 2 * d * pairs * (2 + 4) * H * B
        assert layer_flops(B, s, h, H) == gemm + attn, (B, s, h, H)
    for (B, s, h, H, T, per_gpu_tf) in [(8, 1024, 1600, 25, 2, 0.795), (8, 1024, 2560, 32, 4, 0.999),
                                        (8, 1024, 3072, 32, 8, 0.715), (4, 2048, 6144, 64, 8, 2.861)]:
        closed = 72.0 * B * s * h * h + 6.0 * B * h * s * (s + 1)
        assert layer_flops(B, s, h, H) == closed
        assert abs(closed / T / 1e12 - per_gpu_tf) < 6e-4, (h, closed / T / 1e12)
