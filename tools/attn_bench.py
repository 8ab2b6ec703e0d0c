"""Microbenchmark of the attention kernels (CUDA events).  env MERAK_ATTN_TC=1 selects the tcgen05 forward."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_04959_b200.binding import lib  # noqa: E402


def P(t):
    return ctypes.c_void_p(t.data_ptr())


def main():
    res = {}
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for (b, s, H, d) in [(4, 1024, 25, 64), (4, 1024, 8, 80), (4, 1024, 4, 96), (2, 2048, 8, 96)]:
        hr = H * d
        qkv = torch.randn(b * s, 3 * hr, device="cuda").bfloat16()
        ctx = torch.empty(b * s, hr, device="cuda").bfloat16()
        lse = torch.empty(b, H, s, device="cuda")
        dctx = torch.randn(b * s, hr, device="cuda").bfloat16()
        dqkv = torch.empty_like(qkv)
        delta = torch.empty(b, H, s, device="cuda")
        fl = 2.0 * b * hr * s * (s + 1)

        def t(fn):
            for _ in range(3):
                fn()
            ts = []
            for _ in range(10):
                a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                fn()
                e.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(e))
            return sorted(ts)[5]
        tf = t(lambda: lib().merak_test_attn_fwd(P(qkv), P(ctx), P(lse), b, s, H, d, st))
        tb = t(lambda: lib().merak_test_attn_bwd(P(qkv), P(ctx), P(lse), P(dctx), P(dqkv), P(delta), b, s, H, d, st))
        res[f"b{b}_s{s}_H{H}_d{d}"] = {"fwd_us": round(tf * 1e3, 1), "fwd_tflops": round(fl / tf / 1e9, 1),
                                       "bwd_us": round(tb * 1e3, 1), "bwd_tflops": round(2 * fl / tb / 1e9, 1)}
    print(json.dumps({"fwd_tc": os.environ.get("MERAK_ATTN_TC", "0"), "bwd_tc": os.environ.get("MERAK_ATTN_BWD_TC", "1"), "res": res}))


if __name__ == "__main__":
    main()
