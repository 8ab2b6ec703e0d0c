"""Microbenchmark of the tcgen05 GEMM at the layer's shapes (CUDA events, L2 flushed between reps).
Usage: python tools/gemm_bench.py   (env MERAK_GEMM_CG=1|2 selects the cta_group; T, M_TOK)"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_04959_b200.binding import lib  # noqa: E402


def P(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def shapes(h, f, hr, m):
    # (name, M, N, K, a_mn, b_mn, epi)
    return [("qkv", m, 3 * hr, h, 0, 0, 1), ("proj", m, h, hr, 0, 0, 0), ("fc1", m, f, h, 0, 0, 2),
            ("fc2", m, h, f, 0, 0, 0), ("fc2_dgrad", m, f, h, 0, 1, 3), ("fc1_dgrad", m, h, f, 0, 1, 0),
            ("proj_dgrad", m, hr, h, 0, 1, 0), ("qkv_dgrad", m, h, 3 * hr, 0, 1, 0),
            ("w2_wgrad", h, f + 1, m, 1, 1, 4), ("w1_wgrad", f, h + 1, m, 1, 1, 4),
            ("wo_wgrad", h, hr + 1, m, 1, 1, 4), ("wqkv_wgrad", 3 * hr, h + 1, m, 1, 1, 4)]


def main():
    h, T, m = int(os.environ.get("H", 1600)), int(os.environ.get("T", 1)), int(os.environ.get("M_TOK", 4096))
    f = 4 * h // T
    hr = 832 if (T == 2 and h == 1600) else h // T
    flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
    out = {}
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for name, M, N, K, amn, bmn, epi in shapes(h, f, hr, m):
        A = torch.randn(K if amn else M, M if amn else K, device="cuda").bfloat16()
        B = torch.randn(K if bmn else N, (N + 63) // 64 * 64 if bmn else K, device="cuda").bfloat16()
        o = torch.empty(M, N, device="cuda").bfloat16()
        o2 = torch.empty(M, N, device="cuda").bfloat16()
        bias = torch.randn(N, device="cuda").bfloat16()
        o32 = torch.zeros(M, N, device="cuda")
        db = torch.zeros(M, device="cuda")
        ldb = B.shape[1]

        def run():
            e = lib().merak_test_gemm(P(A), P(B), M, N, K, A.shape[1], ldb, amn, bmn, epi, P(o), N, P(o2), N, P(bias),
                                      P(o2), N, P(o32), N - 1 if epi == 4 else N, P(db) if epi == 4 else None, 0, st)
            assert e == 0, e
        for _ in range(3):
            run()
        ts = []
        for _ in range(10):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            run()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        t = ts[len(ts) // 2]
        out[name] = {"M": M, "N": N, "K": K, "us": round(t * 1e3, 2), "tflops": round(2 * M * N * K / (t * 1e-3) / 1e12, 1)}
        if os.environ.get("CUBLAS") and not amn and not bmn:
            Bt = B[:N, :K]
            def cb():
                torch.matmul(A, Bt.T, out=o)
            for _ in range(3):
                cb()
            ts = []
            for _ in range(10):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                cb()
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ts.sort()
            out[name]["cublas_tflops"] = round(2 * M * N * K / (ts[len(ts) // 2] * 1e-3) / 1e12, 1)
    tot_f = sum(2 * v["M"] * v["N"] * v["K"] for v in out.values())
    tot_t = sum(v["us"] for v in out.values()) * 1e-6
    print(json.dumps({"cg": os.environ.get("MERAK_GEMM_CG", "2"), "bn": os.environ.get("MERAK_GEMM_BN", "auto"),
                      "h": h, "T": T, "m": m, "total_tflops": tot_f / tot_t / 1e12,
                      "total_us": tot_t * 1e6, "gemms": out}))


if __name__ == "__main__" and not os.environ.get("VARIANTS"):
    main()


def variants():
    """qkv shape: default vs 6-stage (192 KB) vs no-store epilogue vs cuBLAS (torch.matmul)."""
    M, N, K = int(os.environ.get("VM", 4096)), int(os.environ.get("VN", 4800)), int(os.environ.get("VK", 1600))
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(N, K, device="cuda").bfloat16()
    o = torch.empty(M, N, device="cuda").bfloat16()
    flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    res = {}

    def tm(fn):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(10):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        t = ts[len(ts) // 2]
        return {"us": round(t * 1e3, 2), "tflops": round(2 * M * N * K / (t * 1e-3) / 1e12, 1)}
    for name, epi in (("default_bn256", 6 if False else 0), ("stages192KB", 6), ("no_store", 5)):
        def run(epi=epi):
            e = lib().merak_test_gemm(P(A), P(B), M, N, K, K, K, 0, 0, epi, P(o), N, None, N, None, None, N, None, N,
                                      None, 0, st)
            assert e == 0, e
        res[name] = tm(run)
    res["cublas"] = tm(lambda: torch.matmul(A, B.T, out=o))
    print(json.dumps({"M": M, "N": N, "K": K, "variants": res}))


if __name__ == "__main__" and os.environ.get("VARIANTS"):
    variants()
