"""CPU fp64 oracle of one GPT decoder layer, forward and backward.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  The product path
(paper_2206_04959_b200/) never imports, links or executes anything here, and
this package imports nothing from it.

What it computes (plain definition):
Sub-pipelined TMP is an exact reformulation of the plain layer:
  * Megatron TMP ("divides weight matrices along row or column dimension
    with additional AllReduce operations") is exact by linearity: the
    row-parallel partial products sum to the full product;
  * sub-microbatches are independent ("whose procedures are independent
    of each other").
So the oracle of the whole path is the unsharded, unsplit layer, here in fp64
with numpy (BLAS dgemm is the only library primitive).  The GPT block details
the paper leaves open ("attention block and FFN block"; P:623 GPT
"transformer decoder"; P:636 HF Transformers 4.15 GPT-2) follow the DESIGN.md
readings:
  R1 pre-LN GPT-2 block;  R2 tanh GeLU;  R3 LN eps=1e-5, biased variance;
  R4 causal mask incl. diagonal, masked prob exactly 0, scale 1/sqrt(d);
  R5 dropout off;  R6 biases on all four GEMMs;  R7 f = 4h.

Notation (per sample; tokens are rows):
  u  = LN1(x)                          (step 1)
  q,k,v = u Wq^T+bq, u Wk^T+bk, u Wv^T+bv, head e = columns e*d..e*d+d-1 (step 2)
  S_e = q_e k_e^T / sqrt(d) (+causal mask), P_e = softmax(S_e), c_e = P_e v_e  (step 3)
  x1 = x + c Wo^T + bo                 (step 4)
  u2 = LN2(x1); z = u2 W1^T + b1; g = gelu(z)   (step 5)
  y  = x1 + g W2^T + b2                (step 6)
Backward (step 7) uses the explicit chain-rule formulas written out below.

Parity: pinned by tests/test_oracle_pins.py (finite differences, torch fp64
autograd of library routines, closed forms, invariants).  The *choice* of the
GPT block details R1-R7 is a documented reading the paper does not pin.
"""
from __future__ import annotations

import math

import numpy as np

LN_EPS = 1e-5  # R3
GELU_C = math.sqrt(2.0 / math.pi)  # R2: gelu(z) = z/2 (1 + tanh(c (z + 0.044715 z^3)))
GELU_A = 0.044715


# ----------------------------------------------------------------------------- elementwise
def gelu(z):
    """tanh-approximation GeLU (R2)."""
    return 0.5 * z * (1.0 + np.tanh(GELU_C * (z + GELU_A * z ** 3)))


def gelu_grad(z):
    """d gelu / dz for the tanh approximation:
    1/2 (1 + t) + 1/2 z (1 - t^2) c (1 + 3a z^2),  t = tanh(c (z + a z^3))."""
    t = np.tanh(GELU_C * (z + GELU_A * z ** 3))
    return 0.5 * (1.0 + t) + 0.5 * z * (1.0 - t * t) * GELU_C * (1.0 + 3.0 * GELU_A * z * z)


# ----------------------------------------------------------------------------- LayerNorm (R3)
def layer_norm(x, gamma, beta, eps=LN_EPS):
    """u = (x - mu) * rho * gamma + beta, mu = mean_h x, var biased, rho = 1/sqrt(var + eps).
    Returns (u, xhat, rho)."""
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    rho = 1.0 / np.sqrt(var + eps)
    xhat = (x - mu) * rho
    return xhat * gamma + beta, xhat, rho


def layer_norm_backward(du, xhat, rho, gamma):
    """dx = rho (dxhat - mean(dxhat) - xhat mean(dxhat * xhat)), dxhat = du * gamma;
    dgamma = sum_tok du * xhat, dbeta = sum_tok du."""
    dxhat = du * gamma
    m1 = dxhat.mean(axis=-1, keepdims=True)
    m2 = (dxhat * xhat).mean(axis=-1, keepdims=True)
    dx = rho * (dxhat - m1 - xhat * m2)
    red = tuple(range(du.ndim - 1))
    return dx, (du * xhat).sum(axis=red), du.sum(axis=red)


# ----------------------------------------------------------------------------- attention (R4)
def causal_attention(q, k, v, heads):
    """q, k, v: [B, s, H*d].  Per (sample, head): S = q k^T / sqrt(d), S[i, j] = -inf for j > i,
    P = softmax_j(S), c = P v.  Returns (c [B, s, H*d], P [B, H, s, s])."""
    B, s, hd = q.shape
    d = hd // heads
    scale = 1.0 / math.sqrt(d)
    mask = np.triu(np.ones((s, s), dtype=bool), k=1)
    c = np.empty_like(q)
    P = np.empty((B, heads, s, s))
    for b in range(B):
        for e in range(heads):
            sl = slice(e * d, (e + 1) * d)
            S = (q[b, :, sl] @ k[b, :, sl].T) * scale
            S[mask] = -np.inf
            S = S - S.max(axis=1, keepdims=True)
            E = np.exp(S)  # exp(-inf) = 0 exactly: masked probabilities are exactly 0
            Pe = E / E.sum(axis=1, keepdims=True)
            P[b, e] = Pe
            c[b, :, sl] = Pe @ v[b, :, sl]
    return c, P


def causal_attention_backward(dc, q, k, v, P, heads):
    """Per (sample, head), with D = rowsum(dc * c) = rowsum(dP * P):
    dV = P^T dc;  dP = dc V^T;  dS = P * (dP - rowsum(dP * P));  dQ = dS K / sqrt(d);  dK = dS^T Q / sqrt(d)."""
    B, s, hd = q.shape
    d = hd // heads
    scale = 1.0 / math.sqrt(d)
    dq, dk, dv = np.empty_like(q), np.empty_like(k), np.empty_like(v)
    for b in range(B):
        for e in range(heads):
            sl = slice(e * d, (e + 1) * d)
            Pe = P[b, e]
            dv[b, :, sl] = Pe.T @ dc[b, :, sl]
            dP = dc[b, :, sl] @ v[b, :, sl].T
            dS = Pe * (dP - (dP * Pe).sum(axis=1, keepdims=True))
            dq[b, :, sl] = (dS @ k[b, :, sl]) * scale
            dk[b, :, sl] = (dS.T @ q[b, :, sl]) * scale
    return dq, dk, dv


# ----------------------------------------------------------------------------- the layer
def _f64(params):
    return {k: np.asarray(v, dtype=np.float64) for k, v in params.items()}


def layer_forward(params, x, heads):
    """Steps 1-6.  x: [B, s, h].  Returns (y, cache)."""
    p = _f64(params)
    x = np.asarray(x, dtype=np.float64)
    h = x.shape[-1]
    u, xhat1, rho1 = layer_norm(x, p["ln1_g"], p["ln1_b"])                 # step 1
    qkv = u @ p["w_qkv"].T + p["b_qkv"]                                     # step 2
    q, k, v = qkv[..., :h], qkv[..., h:2 * h], qkv[..., 2 * h:]
    c, P = causal_attention(q, k, v, heads)                                 # step 3
    x1 = x + c @ p["w_o"].T + p["b_o"]                                      # step 4
    u2, xhat2, rho2 = layer_norm(x1, p["ln2_g"], p["ln2_b"])               # step 5
    z = u2 @ p["w_1"].T + p["b_1"]
    g = gelu(z)
    y = x1 + g @ p["w_2"].T + p["b_2"]                                      # step 6
    cache = dict(x=x, u=u, xhat1=xhat1, rho1=rho1, q=q, k=k, v=v, c=c, P=P,
                 x1=x1, u2=u2, xhat2=xhat2, rho2=rho2, z=z, g=g)
    return y, cache


def layer_backward(params, cache, dy, heads):
    """Step 7.  Returns (dx, grads) with grads keyed like params."""
    p = _f64(params)
    dy = np.asarray(dy, dtype=np.float64)
    C = cache
    red = (0, 1)

    def wgrad(dout, inp):  # sum over tokens of dout^T inp  -> [out, in]
        return dout.reshape(-1, dout.shape[-1]).T @ inp.reshape(-1, inp.shape[-1])

    gr = {}
    # FFN block
    gr["w_2"] = wgrad(dy, C["g"])
    gr["b_2"] = dy.sum(axis=red)
    dz = (dy @ p["w_2"]) * gelu_grad(C["z"])
    gr["w_1"] = wgrad(dz, C["u2"])
    gr["b_1"] = dz.sum(axis=red)
    du2 = dz @ p["w_1"]
    dln2, gr["ln2_g"], gr["ln2_b"] = layer_norm_backward(du2, C["xhat2"], C["rho2"], p["ln2_g"])
    dx1 = dy + dln2
    # attention block
    gr["w_o"] = wgrad(dx1, C["c"])
    gr["b_o"] = dx1.sum(axis=red)
    dc = dx1 @ p["w_o"]
    dq, dk, dv = causal_attention_backward(dc, C["q"], C["k"], C["v"], C["P"], heads)
    dqkv = np.concatenate([dq, dk, dv], axis=-1)
    gr["w_qkv"] = wgrad(dqkv, C["u"])
    gr["b_qkv"] = dqkv.sum(axis=red)
    du = dqkv @ p["w_qkv"]
    dln1, gr["ln1_g"], gr["ln1_b"] = layer_norm_backward(du, C["xhat1"], C["rho1"], p["ln1_g"])
    dx = dx1 + dln1
    return dx, gr


def layer_fwd_bwd(params, x, dy, heads):
    """Unsharded, unsplit layer forward + backward in fp64: (y, dx, grads)."""
    y, cache = layer_forward(params, x, heads)
    dx, grads = layer_backward(params, cache, dy, heads)
    return y, dx, grads


def layer_flops(B, s, h, heads, ffn_mult=4):
    """Algorithmic fwd+bwd FLOPs of one layer (SURVEY.md §8 / DESIGN.md §5):
    GEMMs 2*3*(4h^2 + 2*f*h)*tokens = 72 B s h^2 (f=4h) plus causal attention
    (QK^T and PV, fwd 2x2 B h s(s+1)/2 FLOP, bwd twice that) = 6 B h s (s+1)."""
    f = ffn_mult * h
    gemm = 6.0 * B * s * (3 * h * h + h * h + 2 * f * h)
    attn = 6.0 * B * h * s * (s + 1)
    return gemm + attn
