"""Run attention fwd+bwd cases (b s H d ...) through the test entry points and check vs torch autograd.

env MERAK_ATTN_BWD_TC=1 selects the tcgen05 backward, MERAK_ATTN_TC=1 the tcgen05 forward."""
import ctypes, math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_04959_b200.binding import lib  # noqa: E402

P = lambda t: ctypes.c_void_p(t.data_ptr())
st = lambda: ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
args = list(map(int, sys.argv[1:]))
for i in range(0, len(args), 4):
    b, s, H, d = args[i:i + 4]
    hr = H * d
    g = torch.Generator(device="cuda").manual_seed(s * d + H)
    qkv = torch.randn(b * s, 3 * hr, device="cuda", generator=g).bfloat16()
    ctx = torch.zeros(b * s, hr, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(b, H, s, device="cuda")
    assert lib().merak_test_attn_fwd(P(qkv), P(ctx), P(lse), b, s, H, d, st()) == 0
    dctx = torch.randn(b * s, hr, device="cuda", generator=g).bfloat16()
    dqkv = torch.zeros_like(qkv)
    delta = torch.zeros(b, H, s, device="cuda")
    assert lib().merak_test_attn_bwd(P(qkv), P(ctx), P(lse), P(dctx), P(dqkv), P(delta), b, s, H, d, st()) == 0
    torch.cuda.synchronize()
    q = qkv.float().requires_grad_(True)
    qq, k, v = q.view(b, s, 3, H, d).permute(2, 0, 3, 1, 4)
    S_ = (qq @ k.transpose(-1, -2)) / math.sqrt(d)
    S_ = S_.masked_fill(torch.triu(torch.ones(s, s, dtype=torch.bool, device="cuda"), 1), float("-inf"))
    ref = (torch.softmax(S_, -1) @ v).permute(0, 2, 1, 3).reshape(b * s, hr)
    ref.backward(dctx.float())
    gq = q.grad.view(b * s, 3, hr)
    dq = dqkv.float().view(b * s, 3, hr)
    errs = [((dq[:, j] - gq[:, j]).norm() / gq[:, j].norm()).item() for j in range(3)]
    fe = ((ctx.float() - ref).norm() / ref.norm()).item()
    print(f"case b{b} s{s} H{H} d{d}: fwd {fe:.2e} dq {errs[0]:.2e} dk {errs[1]:.2e} dv {errs[2]:.2e}", flush=True)
