"""Attention microbenchmark (CUDA events around back-to-back launches of the C-ABI test entry points).
Prints one JSON line per shape: forward / backward us and TFLOP/s (causal FLOPs: fwd 2*b*hr*s(s+1),
bwd twice that)."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_04959_b200.binding import lib  # noqa: E402

SHAPES = [(2, 2048, 64, 96), (4, 1024, 25, 64), (4, 1024, 32, 80), (4, 1024, 32, 96), (2, 2048, 8, 128)]


def main():
    shapes = SHAPES
    if len(sys.argv) > 1:  # b,s,H,d[:b,s,H,d...]
        shapes = [tuple(int(v) for v in x.split(",")) for x in sys.argv[1].split(":")]
    L = lib()
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for (b, s, H, d) in shapes:
        hr = H * d
        qkv = torch.randn(b * s, 3 * hr, device="cuda").bfloat16()
        ctx = torch.empty(b * s, hr, device="cuda", dtype=torch.bfloat16)
        lse = torch.empty(b, H, s, device="cuda")
        dctx = torch.randn(b * s, hr, device="cuda").bfloat16()
        dqkv = torch.empty_like(qkv)
        ws = torch.zeros(L.merak_test_attn_bwd_ws_bytes(b, s, H, d), device="cuda", dtype=torch.uint8)
        res = {"b": b, "s": s, "H": H, "d": d}
        for name, fn in (("fwd", lambda: L.merak_test_attn_fwd(P(qkv), P(ctx), P(lse), b, s, H, d, st)),
                         ("bwd", lambda: L.merak_test_attn_bwd(P(qkv), P(ctx), P(lse), P(dctx), P(dqkv), P(ws),
                                                               b, s, H, d, st))):
            for _ in range(3):
                assert fn() == 0
            n = 20
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(n):
                fn()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / n * 1e3
            fl = 2.0 * b * hr * s * (s + 1) * (1 if name == "fwd" else 2)
            res[name + "_us"] = us
            res[name + "_tflops"] = fl / (us * 1e-6) / 1e12
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
