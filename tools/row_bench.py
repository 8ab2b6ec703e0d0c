"""HBM roofline of the replicated row kernels (LayerNorm forward, all-reduce forward / backward epilogues) at a
gpt20b sub-batch (m = 4096 rows, h = 6144) through the test entry points (fake peers on one device, no handshake):
mean device time over `iters` launches (CUDA events) and GB/s of algorithmic bytes (every input row read once,
every output row written once).  One JSON line per kernel.  MERAK_LIB selects an alternative build (A/B)."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_04959_b200.binding import lib  # noqa: E402


def P(t):
    return ctypes.c_void_p(t.data_ptr())


def timeit(fn, iters=30):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e-3


def main():
    m, h = int(os.environ.get("M", 4096)), int(os.environ.get("H", 6144))
    S = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    g = torch.Generator(device="cuda").manual_seed(1)
    rnd = lambda: (torch.randn(m, h, device="cuda", generator=g)).bfloat16()  # noqa: E731
    x, dres, out, u = rnd(), rnd(), torch.empty(m, h, device="cuda", dtype=torch.bfloat16), \
        torch.empty(m, h, device="cuda", dtype=torch.bfloat16)
    parts = [rnd() for _ in range(2)]
    ga = (torch.rand(h, device="cuda", generator=g) + 0.5).bfloat16()
    be = (torch.randn(h, device="cuda", generator=g) * 0.1).bfloat16()
    mean, rstd = torch.zeros(m, device="cuda"), torch.ones(m, device="cuda")
    dg, db = torch.zeros(h, device="cuda"), torch.zeros(h, device="cuda")
    ws = torch.zeros(2 * (m // 8) * h + 2 * (m // 2048 if m >= 2048 else 1) * h + 2 * m * h, device="cuda")
    arr1 = (ctypes.c_void_p * 1)(parts[0].data_ptr())
    arr2 = (ctypes.c_void_p * 2)(parts[0].data_ptr(), parts[1].data_ptr())
    row = m * h * 2
    cases = {
        "ln_fwd": (lambda: lib().merak_test_ln_fwd(P(x), P(ga), P(be), P(u), P(mean), P(rstd), m, h, 1e-5, S),
                   2 * row),
        "ar_fwd_T1": (lambda: lib().merak_test_ar_fwd(arr1, 1, m, h, P(x), P(be), P(out), 0, P(ga), P(be), P(u),
                                                      P(mean), P(rstd), 1e-5, 0, S), 3 * row),
        "ar_fwd_T1_ln": (lambda: lib().merak_test_ar_fwd(arr1, 1, m, h, P(x), P(be), P(out), 1, P(ga), P(be), P(u),
                                                         P(mean), P(rstd), 1e-5, 0, S), 4 * row),
        "ar_fwd_T2_ln": (lambda: lib().merak_test_ar_fwd(arr2, 2, m, h, P(x), P(be), P(out), 1, P(ga), P(be), P(u),
                                                         P(mean), P(rstd), 1e-5, 0, S), 5 * row),
        # includes the per-sample LN-gradient reduction kernels of the test entry point (s = 2048 rows per sample)
        "ar_bwd_T1": (lambda: lib().merak_test_ar_bwd(arr1, 1, m, 2048, h, P(x), P(mean), P(rstd), P(ga), P(dres),
                                                      P(out), P(dg), P(db), P(ws), 0, S), 4 * row),
    }
    for name, (fn, nbytes) in cases.items():
        assert fn() == 0, name
        t = timeit(fn)
        print(json.dumps({"kernel": name, "m": m, "h": h, "us": t * 1e6, "alg_bytes": nbytes,
                          "GBps": nbytes / t / 1e9, "lib": os.path.basename(os.environ.get("MERAK_LIB", "default"))}),
              flush=True)


if __name__ == "__main__":
    main()
