"""Kernel-level numerics (GPU): each sm_100a kernel vs a plain PyTorch fp32 reference of the same op
on the same bf16 inputs, through the testing entry points of libmerak_tmp.so (merak_tmp_testing.h)."""
import ctypes
import math

import pytest
import torch

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2206_04959_b200.binding import lib


def P(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def S():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def rel(a, b):
    a, b = a.double(), b.double()
    return ((a - b).norm() / b.norm().clamp_min(1e-30)).item()


def gelu_ref(z):
    return torch.nn.functional.gelu(z, approximate="tanh")


def gelu_grad_ref(z):
    c = math.sqrt(2 / math.pi)
    t = torch.tanh(c * (z + 0.044715 * z ** 3))
    return 0.5 * (1 + t) + 0.5 * z * (1 - t * t) * c * (1 + 3 * 0.044715 * z * z)


def run_gemm(A, B, M, N, K, a_mn, b_mn, epi, bias=None, aux=None, out32=None, max_ctas=0, db32=None, ldb=None):
    dev = A.device
    out = torch.zeros(M, N, dtype=torch.bfloat16, device=dev)
    out2 = torch.zeros(M, N, dtype=torch.bfloat16, device=dev)
    ld32 = N - 1 if db32 is not None else N
    err = lib().merak_test_gemm(P(A), P(B), M, N, K, A.shape[1], ldb or B.shape[1], int(a_mn), int(b_mn), epi,
                                P(out), N, P(out2), N, P(bias), P(aux), N, P(out32), ld32, P(db32), max_ctas, S())
    assert err == 0, err
    torch.cuda.synchronize()
    return out, out2


GEMM_SHAPES = [(16, 96, 64), (128, 128, 64), (256, 384, 320), (300, 200, 96), (520, 264, 1600), (4096, 4800, 1600),
               (4096, 1600, 6400)]


@pytest.mark.parametrize("dyn", [0, 1])
@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
def test_gemm_forward_epilogues(M, N, K, dyn, monkeypatch):
    monkeypatch.setenv("MERAK_GEMM_DYN", str(dyn))  # static vs dynamic (atomic) tile schedule
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
    bias = (torch.randn(N, device="cuda", generator=g) * 0.1).bfloat16()
    ref = A.float() @ B.float().T
    out, _ = run_gemm(A, B, M, N, K, False, False, 0)
    assert rel(out, ref) < 5e-3
    out, _ = run_gemm(A, B, M, N, K, False, False, 1, bias=bias)
    assert rel(out, ref + bias.float()) < 5e-3
    z, gl = run_gemm(A, B, M, N, K, False, False, 2, bias=bias)
    assert rel(z, ref + bias.float()) < 5e-3
    assert rel(gl, gelu_ref(ref + bias.float())) < 5e-3


@pytest.mark.parametrize("dyn", [0, 1])
@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
def test_gemm_dgrad(M, N, K, dyn, monkeypatch):
    """dgrad: B stored [K, N] (the weight [out, in] read MN-major)."""
    monkeypatch.setenv("MERAK_GEMM_DYN", str(dyn))
    g = torch.Generator(device="cuda").manual_seed(M + 3 * N)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    Bs = (torch.randn(K, N, device="cuda", generator=g) * 0.05).bfloat16()
    z = torch.randn(M, N, device="cuda", generator=g).bfloat16()
    ref = A.float() @ Bs.float()
    out, _ = run_gemm(A, Bs, M, N, K, False, True, 0)
    assert rel(out, ref) < 5e-3
    out, _ = run_gemm(A, Bs, M, N, K, False, True, 3, aux=z)
    assert rel(out, ref * gelu_grad_ref(z.float())) < 5e-3


@pytest.mark.parametrize("M,N,K", [(96, 64, 16), (256, 320, 128), (1600, 3200, 4096), (200, 136, 48)])
def test_gemm_wgrad_accumulate_and_split_bit_identity(M, N, K):
    """wgrad: C[M,N] (fp32, preloaded) += A_s^T B_s with A_s [K, M], B_s [K, N] (tokens = K).
    Splitting K at a multiple of 16 in two accumulating calls is bit-identical to one call."""
    g = torch.Generator(device="cuda").manual_seed(K + M)
    As = torch.randn(K, M, device="cuda", generator=g).bfloat16()
    Bs = torch.randn(K, N, device="cuda", generator=g).bfloat16()
    C0 = torch.randn(M, N, device="cuda", generator=g)
    C = C0.clone()
    run_gemm(As, Bs, M, N, K, True, True, 4, out32=C)
    ref = C0.double() + As.double().T @ Bs.double()
    assert rel(C, ref) < 1e-5
    if K % 32 == 0:
        C2 = C0.clone()
        k1 = K // 2
        run_gemm(As[:k1], Bs[:k1], M, N, k1, True, True, 4, out32=C2)
        run_gemm(As[k1:], Bs[k1:], M, N, K - k1, True, True, 4, out32=C2)
        assert torch.equal(C, C2)


@pytest.mark.parametrize("M,N,K", [(64, 64, 32), (1600, 1600, 4096), (1600, 6400, 256), (96, 136, 48)])
def test_gemm_wgrad_ones_column_bias_grad(M, N, K):
    """wgrad with the ones column: B_s [K, N+8] whose column N is 1 (the saved-activation pad) gives
    dW += A_s^T B_s[:, :N] and db += A_s^T 1 = column sums of A_s, split bit-identically."""
    g = torch.Generator(device="cuda").manual_seed(K * 3 + N)
    As = torch.randn(K, M, device="cuda", generator=g).bfloat16()
    Bp = torch.zeros(K, N + 8, device="cuda").bfloat16()
    Bp[:, :N] = torch.randn(K, N, device="cuda", generator=g).bfloat16()
    Bp[:, N] = 1.0
    C0 = torch.randn(M, N, device="cuda", generator=g)
    d0 = torch.randn(M, device="cuda", generator=g)
    C, d = C0.clone(), d0.clone()
    run_gemm(As, Bp, M, N + 1, K, True, True, 4, out32=C, db32=d, ldb=N + 8)
    assert rel(C, C0.double() + As.double().T @ Bp[:, :N].double()) < 1e-5
    assert rel(d, d0.double() + As.double().sum(0)) < 1e-5
    if K % 32 == 0:
        C2, d2 = C0.clone(), d0.clone()
        k1 = K // 2
        run_gemm(As[:k1], Bp[:k1], M, N + 1, k1, True, True, 4, out32=C2, db32=d2, ldb=N + 8)
        run_gemm(As[k1:], Bp[k1:], M, N + 1, K - k1, True, True, 4, out32=C2, db32=d2, ldb=N + 8)
        assert torch.equal(C, C2) and torch.equal(d, d2)


def test_gemm_reduction_order_independent_of_m():
    """Bit-identity rule (i): the value of an output row does not depend on M or the grid."""
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn(1024, 640, device="cuda", generator=g).bfloat16()
    B = (torch.randn(512, 640, device="cuda", generator=g) * 0.05).bfloat16()
    full, _ = run_gemm(A, B, 1024, 512, 640, False, False, 0)
    half, _ = run_gemm(A[512:].contiguous(), B, 512, 512, 640, False, False, 0, max_ctas=7)
    assert torch.equal(full[512:], half)


def test_gemm_dynamic_schedule_bit_identical_to_static(monkeypatch):
    """The dynamic tile order changes which cluster computes a tile, never a tile's K order; repeated
    launches also check that the kernel leaves its counter at 0."""
    g = torch.Generator(device="cuda").manual_seed(2)
    A = torch.randn(4096, 1600, device="cuda", generator=g).bfloat16()
    B = (torch.randn(4800, 1600, device="cuda", generator=g) * 0.05).bfloat16()
    monkeypatch.setenv("MERAK_GEMM_DYN", "0")
    ref, _ = run_gemm(A, B, 4096, 4800, 1600, False, False, 0)
    monkeypatch.setenv("MERAK_GEMM_DYN", "1")
    for mc in (0, 0, 20, 7, 0):
        out, _ = run_gemm(A, B, 4096, 4800, 1600, False, False, 0, max_ctas=mc)
        assert torch.equal(out, ref), mc


# ------------------------------------------------------------------------------------------- attention
def attn_ref(qkv, b, s, H, d):
    hr = H * d
    q, k, v = qkv.float().view(b, s, 3, H, d).permute(2, 0, 3, 1, 4)
    S_ = (q @ k.transpose(-1, -2)) / math.sqrt(d)
    mask = torch.triu(torch.ones(s, s, dtype=torch.bool, device=qkv.device), 1)
    S_ = S_.masked_fill(mask, float("-inf"))
    Pm = torch.softmax(S_, -1)
    o = Pm @ v
    return o.permute(0, 2, 1, 3).reshape(b * s, hr)


@pytest.mark.parametrize("b,s,H,d", [(2, 16, 2, 32), (2, 100, 3, 64), (1, 256, 2, 80), (2, 1024, 2, 96),
                                     (1, 192, 2, 128), (4, 1024, 4, 64), (2, 208, 5, 64), (1, 2048, 2, 96),
                                     (3, 144, 3, 128), (2, 272, 2, 32)])
def test_attention_fwd_bwd(b, s, H, d):
    g = torch.Generator(device="cuda").manual_seed(s * d + H)
    hr = H * d
    qkv = torch.randn(b * s, 3 * hr, device="cuda", generator=g).bfloat16()
    ctx = torch.zeros(b * s, hr, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(b, H, s, device="cuda")
    assert lib().merak_test_attn_fwd(P(qkv), P(ctx), P(lse), b, s, H, d, S()) == 0
    torch.cuda.synchronize()
    q = qkv.float().requires_grad_(True)
    ref = attn_ref(q, b, s, H, d)
    assert rel(ctx, ref) < 1e-2
    dctx = torch.randn(b * s, hr, device="cuda", generator=g).bfloat16()
    ref.backward(dctx.float())
    dqkv = torch.zeros_like(qkv)
    ws = torch.zeros(lib().merak_test_attn_bwd_ws_bytes(b, s, H, d), device="cuda", dtype=torch.uint8)
    assert lib().merak_test_attn_bwd(P(qkv), P(ctx), P(lse), P(dctx), P(dqkv), P(ws), b, s, H, d, S()) == 0
    torch.cuda.synchronize()
    gq = q.grad.view(b * s, 3, hr)
    dq = dqkv.view(b * s, 3, hr)
    for i in range(3):
        assert rel(dq[:, i], gq[:, i]) < 2e-2, i
    # deterministic (ordered dQ accumulation, counters left at zero): a second call is bit-identical
    dqkv2 = torch.zeros_like(qkv)
    assert lib().merak_test_attn_bwd(P(qkv), P(ctx), P(lse), P(dctx), P(dqkv2), P(ws), b, s, H, d, S()) == 0
    torch.cuda.synchronize()
    assert torch.equal(dqkv, dqkv2)


# ------------------------------------------------------------------------------------------- LN / AR
@pytest.mark.parametrize("m,h", [(16, 64), (300, 1600), (64, 6144)])
def test_layernorm_fwd(m, h):
    g = torch.Generator(device="cuda").manual_seed(h)
    x = (torch.randn(m, h, device="cuda", generator=g) * 2 + 0.5).bfloat16()
    ga = (torch.rand(h, device="cuda", generator=g) + 0.5).bfloat16()
    be = (torch.randn(h, device="cuda", generator=g) * 0.1).bfloat16()
    u = torch.zeros_like(x)
    mean = torch.zeros(m, device="cuda")
    rstd = torch.zeros(m, device="cuda")
    assert lib().merak_test_ln_fwd(P(x), P(ga), P(be), P(u), P(mean), P(rstd), m, h, 1e-5, S()) == 0
    torch.cuda.synchronize()
    ref = torch.nn.functional.layer_norm(x.float(), (h,), ga.float(), be.float(), 1e-5)
    assert rel(u, ref) < 5e-3
    assert torch.allclose(mean, x.float().mean(-1), rtol=1e-4, atol=1e-5)


def _ptr_array(ts):
    return (ctypes.c_void_p * len(ts))(*[t.data_ptr() for t in ts])


@pytest.mark.parametrize("T,m,h", [(1, 32, 64), (2, 256, 1600), (4, 128, 2560), (8, 64, 6144)])
def test_allreduce_fwd_fake_peers(T, m, h):
    """AR#1 data path with T ranks emulated as T buffers on one device (no handshake)."""
    g = torch.Generator(device="cuda").manual_seed(T * h)
    parts = [(torch.randn(m, h, device="cuda", generator=g) * 0.3).bfloat16() for _ in range(T)]
    x = torch.randn(m, h, device="cuda", generator=g).bfloat16()
    bias = (torch.randn(h, device="cuda", generator=g) * 0.02).bfloat16()
    ga = (torch.rand(h, device="cuda", generator=g) + 0.5).bfloat16()
    be = (torch.randn(h, device="cuda", generator=g) * 0.1).bfloat16()
    out, u2 = torch.zeros_like(x), torch.zeros_like(x)
    mean, rstd = torch.zeros(m, device="cuda"), torch.zeros(m, device="cuda")
    arr = _ptr_array(parts)
    assert lib().merak_test_ar_fwd(arr, T, m, h, P(x), P(bias), P(out), 1, P(ga), P(be), P(u2), P(mean), P(rstd),
                                   1e-5, 0, S()) == 0
    torch.cuda.synchronize()
    ref = sum(p.float() for p in parts) + bias.float() + x.float()
    assert rel(out, ref) < 5e-3
    lnref = torch.nn.functional.layer_norm(out.float(), (h,), ga.float(), be.float(), 1e-5)
    assert rel(u2, lnref) < 5e-3


@pytest.mark.parametrize("T,m,h", [(1, 32, 64), (2, 256, 1600), (4, 64, 6144)])
def test_allreduce_bwd_fake_peers(T, m, h):
    g = torch.Generator(device="cuda").manual_seed(T + h)
    parts = [(torch.randn(m, h, device="cuda", generator=g) * 0.3).bfloat16() for _ in range(T)]
    x = (torch.randn(m, h, device="cuda", generator=g) * 1.5).bfloat16()
    ga = (torch.rand(h, device="cuda", generator=g) + 0.5).bfloat16()
    dres = torch.randn(m, h, device="cuda", generator=g).bfloat16()
    xf = x.float()
    mean = xf.mean(-1)
    rstd = torch.rsqrt(xf.var(-1, unbiased=False) + 1e-5)
    dx = torch.zeros_like(x)
    dg = torch.randn(h, device="cuda", generator=g)
    db = torch.randn(h, device="cuda", generator=g)
    dg0, db0 = dg.clone(), db.clone()
    G = 8
    ws = torch.zeros(2 * (m // G) * h + 2 * m * h, device="cuda")
    arr = _ptr_array(parts)
    s = 32 if m % 32 == 0 else m  # rows per sample
    assert lib().merak_test_ar_bwd(arr, T, m, s, h, P(x), P(mean), P(rstd), P(ga), P(dres), P(dx), P(dg), P(db),
                                   P(ws), 0, S()) == 0
    torch.cuda.synchronize()
    # the all-reduced gradient is the fp32 rank-ordered sum rounded once to bf16 (reading R10)
    du = sum(p.float() for p in parts).bfloat16().float()
    xr = xf.clone().requires_grad_(True)
    gr = ga.float().clone().requires_grad_(True)
    br = torch.zeros(h, device="cuda", requires_grad=True)
    y = torch.nn.functional.layer_norm(xr, (h,), gr, br, 1e-5)
    y.backward(du)
    assert rel(dx, dres.float() + xr.grad) < 5e-3
    assert rel(dg - dg0, gr.grad) < 1e-4
    assert rel(db - db0, br.grad) < 1e-4


def test_colsum_fixed_order_bit_identity():
    g = torch.Generator(device="cuda").manual_seed(5)
    X = torch.randn(512, 320, device="cuda", generator=g).bfloat16()
    g1 = torch.randn(320, device="cuda", generator=g)
    g2 = g1.clone()
    ref = g1.double() + X.double().sum(0)
    ws = torch.zeros(2 * 512 // 64 * 320, device="cuda")
    assert lib().merak_test_colsum(P(X), 320, 512, 64, 320, P(g1), P(ws), S()) == 0
    for j in range(4):  # the same 8 samples of 64 rows in four sub-batches
        assert lib().merak_test_colsum(P(X[j * 128:]), 320, 128, 64, 320, P(g2), P(ws), S()) == 0
    torch.cuda.synchronize()
    assert torch.equal(g1, g2)
    assert rel(g1, ref) < 1e-6
