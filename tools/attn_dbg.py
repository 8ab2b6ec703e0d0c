"""Per-CTA clock stamps of the attention backward (AttnArgs::dbg, 192 x u64 per CTA): time per half-block
of the MMA issuer (q_full / p_full acquisition), prologue, epilogue, CTA spans (diagnostics only)."""
import ctypes, json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_04959_b200.binding import lib  # noqa: E402

b, s, H, d = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "2,2048,64,96").split(","))
L = lib()
L.merak_test_attn_bwd_dbg.argtypes = [ctypes.c_void_p] * 6 + [ctypes.c_int] * 4 + [ctypes.c_void_p, ctypes.c_void_p]
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
hr = H * d
qkv = torch.randn(b * s, 3 * hr, device="cuda").bfloat16()
ctx = torch.empty(b * s, hr, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(b, H, s, device="cuda")
dctx = torch.randn(b * s, hr, device="cuda").bfloat16()
dqkv = torch.empty_like(qkv)
ws = torch.zeros(L.merak_test_attn_bwd_ws_bytes(b, s, H, d), device="cuda", dtype=torch.uint8)
nkt = (s + 127) // 128
ncta = b * H * nkt
dbg = torch.zeros(ncta * 192, dtype=torch.int64, device="cuda")
assert L.merak_test_attn_fwd(P(qkv), P(ctx), P(lse), b, s, H, d, st) == 0
for _ in range(3):
    assert L.merak_test_attn_bwd_dbg(P(qkv), P(ctx), P(lse), P(dctx), P(dqkv), P(ws), b, s, H, d, P(dbg), st) == 0
torch.cuda.synchronize()
D = dbg.view(ncta, 192).cpu().tolist()
t0 = min(r[76] for r in D)
t1 = max(r[78] for r in D)
per_it, gaps_q, gaps_p, prol, epi = [], [], [], [], []
for r in D:
    ni = r[77]
    prol.append(r[1] - r[0])
    if ni >= 4:
        q = [r[2 + i] for i in range(min(ni, 36))]
        pp = [r[38 + i] for i in range(min(ni, 36))]
        per_it.append((q[-1] - q[1]) / (len(q) - 2))
        gaps_q += [pp[i] - q[i] for i in range(len(q))]
        gaps_p += [q[i + 1] - pp[i] for i in range(len(q) - 1)]
    epi.append(r[75] - r[74])
med = lambda v: sorted(v)[len(v) // 2]  # noqa: E731
print(json.dumps({"shape": [b, s, H, d], "kernel_span_us": (t1 - t0) / 1e3, "ctas": ncta,
                  "cta_span_us_median": med([(r[78] - r[76]) / 1e3 for r in D]),
                  "clk_per_halfblock_median": med(per_it), "prologue_clk_median": med(prol),
                  "q_to_p_clk_median": med(gaps_q), "p_to_nextq_clk_median": med(gaps_p),
                  "epilogue_clk_median": med(epi),
                  "kvdone_after_lastissue_clk": med([r[70] - r[74] for r in D if r[77] <= 32]),
                  "dkdv_store_clk": med([r[71] - r[70] for r in D if r[77] <= 32]),
                  "bulk0_end_after_lastissue_clk": med([r[72] - r[74] for r in D if r[77] <= 32]),
                  "bulk1_end_after_lastissue_clk": med([r[73] - r[74] for r in D if r[77] <= 32 and r[77] > 1]),
                  "last_dqfull_after_lastissue_clk": med([r[88] - r[74] for r in D]),
                  "ew_busy_clk": med([r[128 + j] - r[96 + j] for r in D if r[77] >= 8 for j in range(1, (min(r[77], 32) + 1) // 2 - 1)]),
                  "grads_to_dqfree_wait_clk": med([r[144 + j] - r[38 + 2 * j] for r in D if r[77] >= 8 for j in range(1, (min(r[77], 32) - 2) // 2)]),
                  "dqfree_wait_clk": med([r[160 + j] - r[144 + j] for r in D if r[77] >= 8 for j in range(1, (min(r[77], 32) - 2) // 2)]),
                  "grads_issue_clk": med([r[112 + j] - r[38 + 2 * j] for r in D if r[77] >= 8 for j in range(1, (min(r[77], 32) - 2) // 2)]),
                  "sdone_after_grads_issue_clk": med([r[96 + j + 1] - r[38 + 2 * j] for r in D if r[77] >= 8 for j in range(1, (min(r[77], 32) - 2) // 2)]),
                  "next_scores_issue_after_grads_clk": med([r[2 + 2 * j + 2] - r[38 + 2 * j] for r in D if r[77] >= 8 for j in range(1, (min(r[77], 32) - 2) // 2)]),
                  "ew_idle_clk": med([r[96 + j + 1] - r[128 + j] for r in D if r[77] >= 8 for j in range(1, (min(r[77], 32) + 1) // 2 - 1)]),
                  "last_block_thread": (lambda L: {"staged_after_lastissue": med([r[80 + 4 * (L(r))] - r[74] for r in D]),
                                                   "counter_wait": med([r[81 + 4 * L(r)] - r[80 + 4 * L(r)] for r in D]),  # (now before staging)
                                                   "read": med([r[82 + 4 * L(r)] - r[81 + 4 * L(r)] for r in D]),
                                                   "complete": med([r[83 + 4 * L(r)] - r[82 + 4 * L(r)] for r in D])})(
                      lambda r: (r[77] - 1) & 1),
                  "sum_cta_span_over_148_us": sum((r[78] - r[76]) for r in D) / 148 / 1e3}))
