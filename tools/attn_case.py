"""Run one attention forward case (b s H d) through the test entry point and check vs torch."""
import ctypes, math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_04959_b200.binding import lib  # noqa: E402
b, s, H, d = map(int, sys.argv[1:5])
hr = H * d
g = torch.Generator(device="cuda").manual_seed(s * d + H)
qkv = torch.randn(b * s, 3 * hr, device="cuda", generator=g).bfloat16()
ctx = torch.zeros(b * s, hr, device="cuda", dtype=torch.bfloat16)
lse = torch.zeros(b, H, s, device="cuda")
P = lambda t: ctypes.c_void_p(t.data_ptr())
assert lib().merak_test_attn_fwd(P(qkv), P(ctx), P(lse), b, s, H, d, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0
torch.cuda.synchronize()
q, k, v = qkv.float().view(b, s, 3, H, d).permute(2, 0, 3, 1, 4)
S_ = (q @ k.transpose(-1, -2)) / math.sqrt(d)
S_ = S_.masked_fill(torch.triu(torch.ones(s, s, dtype=torch.bool, device="cuda"), 1), float("-inf"))
ref = (torch.softmax(S_, -1) @ v).permute(0, 2, 1, 3).reshape(b * s, hr)
err = ((ctx.float() - ref).norm() / ref.norm()).item()
print(f"case b{b} s{s} H{H} d{d}: rel err {err:.2e}", flush=True)
