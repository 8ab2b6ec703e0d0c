"""Where a tcgen05 attention-backward CTA spends its time (per-CTA clock stamps, see
attention_bwd_tc.cu dbg layout).  Prints one JSON summary."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_04959_b200.binding import lib  # noqa: E402

P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731


def main():
    b, s, H, d = (int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (4, 1024, 25, 64)))
    hr = H * d
    L = lib()
    L.merak_test_attn_bwd_dbg.argtypes = [ctypes.c_void_p] * 6 + [ctypes.c_int] * 4 + [ctypes.c_void_p, ctypes.c_void_p]
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    qkv = torch.randn(b * s, 3 * hr, device="cuda").bfloat16()
    ctx = torch.empty(b * s, hr, device="cuda").bfloat16()
    lse = torch.empty(b, H, s, device="cuda")
    dctx = torch.randn(b * s, hr, device="cuda").bfloat16()
    dqkv = torch.empty_like(qkv)
    delta = torch.empty(b, H, s, device="cuda")
    assert L.merak_test_attn_fwd(P(qkv), P(ctx), P(lse), b, s, H, d, st) == 0
    nq = (s + 127) // 128
    ncta = nq * H * b
    dbg = torch.zeros(2 * ncta * 64, dtype=torch.int64, device="cuda")
    for _ in range(3):
        assert L.merak_test_attn_bwd_dbg(P(qkv), P(ctx), P(lse), P(dctx), P(dqkv), P(delta), b, s, H, d, P(dbg), st) == 0
    torch.cuda.synchronize()
    # one merged launch, grid (H, b, 2 x tiles): role = z & 1 (even: dQ, odd: dK/dV)
    A = dbg.cpu().numpy().astype(np.int64).reshape(2 * nq, H * b, 64)
    D = [A[0::2].reshape(-1, 64), A[1::2].reshape(-1, 64)]
    out = {}
    for k, name in enumerate(("dq", "dkdv")):
        X = D[k]
        ns = (X[:, 57] - X[:, 56]).astype(np.float64)
        cyc = (X[:, 61] - X[:, 0]).astype(np.float64)
        ghz = float(np.median(cyc / np.maximum(ns, 1)))
        n_it = X[:, 63]
        pro = (X[:, 1] - X[:, 0]) / ghz / 1e3
        first = (X[:, 2] - X[:, 1]) / ghz / 1e3
        its = []
        for c in range(ncta):
            n = int(min(n_it[c], 54))
            if n > 1:
                its.extend(list(np.diff(X[c, 2:2 + n]) / ghz / 1e3))
        epi = (X[:, 61] - X[:, 60]) / ghz / 1e3
        tot = cyc / ghz / 1e3
        t0 = min(D[0][:, 56].min(), D[1][:, 56].min())
        span = (X[:, 57].max() - t0) / 1e3
        out[name] = {"ctas": ncta, "kernel_span_us": round(span, 1), "clock_ghz": round(ghz, 3),
                     "cta_total_us": {"mean": round(float(tot.mean()), 2), "max": round(float(tot.max()), 2)},
                     "prologue_us_mean": round(float(pro.mean()), 2), "first_scores_us_mean": round(float(first.mean()), 2),
                     "iter_us": {"mean": round(float(np.mean(its)), 3), "p50": round(float(np.median(its)), 3),
                                 "p90": round(float(np.percentile(its, 90)), 3)},
                     "epilogue_us_mean": round(float(epi.mean()), 2),
                     "iters_mean": round(float(n_it.mean()), 2),
                     "sum_cta_us_per_sm": round(float(tot.sum()) / 148, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
