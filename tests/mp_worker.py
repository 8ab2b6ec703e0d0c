"""Multi-rank worker (launched by torchrun from tests/test_gpu_multi.py): the TMP layer on T = WORLD_SIZE
GPUs through the C ABI, each rank holding its shard; checks vs the fp64 oracle's slices, cross-rank
bit equality of the replicated outputs, bit-identity of n = 1 vs n = 2 at T > 1, and of the one-shot vs
two-shot all-reduce.
Exit code 0 = all checks passed."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from gpu_layer_util import TOL_FP32, compare_to_oracle, oracle_rank_slices, run_gpu_layer  # noqa: E402
from oracle import layer_fwd_bwd  # noqa: E402
from synth import CONFIGS  # noqa: E402
from synth import make_all  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    backend = os.environ.get("MERAK_TEST_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group("gloo")
    group = dist.group.WORLD
    T = world
    tiny = CONFIGS["tiny"]
    cases = {
        "tiny": tiny.with_(tmp_degree=T),
        "h320_H5_uneven": tiny.with_(hidden=320, heads=5, seq_len=64, microbatch=4, tmp_degree=T),
        "h256_H8_s128_n4": tiny.with_(hidden=256, heads=8, seq_len=128, microbatch=4, n_sub=4, tmp_degree=T),
        "h320_H4_d80": tiny.with_(hidden=320, heads=4, seq_len=96, microbatch=2, tmp_degree=T),
        "h384_H4_d96": tiny.with_(hidden=384, heads=4, seq_len=64, microbatch=4, n_sub=2, tmp_degree=T),
    }
    if os.environ.get("MERAK_TEST_FULL", "0") == "1":
        cases["gpt1.5b"] = CONFIGS["gpt1.5b"].with_(tmp_degree=T)
    failures = []
    for name, cfg in cases.items():
        if cfg.heads < T or cfg.ffn % T:
            continue
        params, x, dy = make_all(cfg, seed=2000 + cfg.hidden)
        out = run_gpu_layer(cfg, params, x, dy, T=T, rank=rank, group=group)
        y, dx, g = layer_fwd_bwd(params, x, dy, cfg.heads)
        errs, bad = compare_to_oracle(out, y, dx, oracle_rank_slices(g, cfg, T, rank), cfg)
        print(f"[rank {rank}] {name} T={T}", {k: f"{v:.2e}" for k, v in errs.items()}, flush=True)
        if bad:
            failures.append((name, bad))
        # replicated outputs must be bit-identical on every rank
        for k in ("y", "dx", "ln1_g", "ln1_b", "ln2_g", "ln2_b", "b_o", "b_2"):
            t = out[k].contiguous()
            gathered = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(gathered, t)
            if not all(torch.equal(gathered[0], q) for q in gathered):
                failures.append((name, f"{k} differs across ranks"))
        # sub-pipelined vs non-sub-pipelined bit-identity at T > 1
        out1 = run_gpu_layer(cfg, params, x, dy, T=T, rank=rank, group=group, n_sub=1)
        for k in out:
            if not torch.equal(out[k], out1[k]):
                failures.append((name, f"{k}: n={cfg.n_sub} vs n=1 not bit-identical"))
        # one-shot vs two-shot all-reduce (default: two-shot at T >= 4) must be bit-identical
        os.environ["MERAK_AR_TWO_SHOT"] = "0" if T >= 4 else "1"
        try:
            out2 = run_gpu_layer(cfg, params, x, dy, T=T, rank=rank, group=group)
        finally:
            del os.environ["MERAK_AR_TWO_SHOT"]
        for k in out:
            if not torch.equal(out[k], out2[k]):
                failures.append((name, f"{k}: one-shot vs two-shot all-reduce not bit-identical"))
        # fused GEMM -> reduce-scatter push (MERAK_AR_PUSH=1, two-shot): row-parallel GEMM epilogues store their
        # boxes into the owners' slots over NVLink (peer TMA maps); same sums, so bit-identical
        for mode in ("1", "2"):  # 2: the reduced rows are pushed into every rank's all-gather slot as well
            os.environ["MERAK_AR_PUSH"] = mode
            os.environ["MERAK_AR_TWO_SHOT"] = "1"
            os.environ["MERAK_AR_PUSH_MINK"] = "0"  # every row-parallel GEMM pushes at these shapes
            try:
                outq = run_gpu_layer(cfg, params, x, dy, T=T, rank=rank, group=group)
            finally:
                del os.environ["MERAK_AR_PUSH"]
                del os.environ["MERAK_AR_TWO_SHOT"]
                del os.environ["MERAK_AR_PUSH_MINK"]
            for k in out:
                if not torch.equal(out[k], outq[k]):
                    failures.append((name, f"{k}: pushed reduce-scatter (mode {mode}) not bit-identical"))
        # programmatic dependent launch along the all-reduce chain (opt-in) must not change a bit
        os.environ["MERAK_AR_PDL"] = "1"
        try:
            outp = run_gpu_layer(cfg, params, x, dy, T=T, rank=rank, group=group)
        finally:
            del os.environ["MERAK_AR_PDL"]
        for k in out:
            if not torch.equal(out[k], outp[k]):
                failures.append((name, f"{k}: PDL all-reduce chain not bit-identical"))
        # fp32 check mode over the peer all-reduce (tolerance 1e-5)
        if cfg.hidden <= 320:
            out32 = run_gpu_layer(cfg, params, x, dy, T=T, rank=rank, group=group, precision=1)
            errs, bad = compare_to_oracle(out32, y, dx, oracle_rank_slices(g, cfg, T, rank), cfg, tol=TOL_FP32)
            print(f"[rank {rank}] {name} T={T} fp32", {k: f"{v:.1e}" for k, v in errs.items()}, flush=True)
            if bad:
                failures.append((name + "/fp32", bad))
        # NCCL baseline (MERAK_COMM_NCCL): same kernels, ncclAllReduce instead of the peer kernel
        outn = run_gpu_layer(cfg, params, x, dy, T=T, rank=rank, group=group, comm=1)
        errs, bad = compare_to_oracle(outn, y, dx, oracle_rank_slices(g, cfg, T, rank), cfg)
        print(f"[rank {rank}] {name} T={T} nccl", {k: f"{v:.2e}" for k, v in errs.items()}, flush=True)
        if bad:
            failures.append((name + "/nccl", bad))
        # NVLS in-switch reduction (MERAK_COMM_NVLS) where every device supports multicast:
        # oracle parity, replicated outputs equal on every rank, run-to-run determinism of the switch's sum,
        # and n = 1 vs n = 2 bit-identity
        from paper_2206_04959_b200 import MERAK_COMM_NVLS, MerakError
        try:
            outv = run_gpu_layer(cfg, params, x, dy, T=T, rank=rank, group=group, comm=MERAK_COMM_NVLS)
        except MerakError as e:
            if e.status != -3:
                raise
            print(f"[rank {rank}] {name} T={T} nvls: unsupported here ({e})", flush=True)
            continue
        errs, bad = compare_to_oracle(outv, y, dx, oracle_rank_slices(g, cfg, T, rank), cfg)
        print(f"[rank {rank}] {name} T={T} nvls", {k: f"{v:.2e}" for k, v in errs.items()}, flush=True)
        if bad:
            failures.append((name + "/nvls", bad))
        for k in ("y", "dx", "ln1_g", "ln1_b", "ln2_g", "ln2_b", "b_o", "b_2"):
            t = outv[k].contiguous()
            gathered = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(gathered, t)
            if not all(torch.equal(gathered[0], q) for q in gathered):
                failures.append((name, f"nvls: {k} differs across ranks"))
        outv2 = run_gpu_layer(cfg, params, x, dy, T=T, rank=rank, group=group, comm=MERAK_COMM_NVLS, reps=2)
        outv1 = run_gpu_layer(cfg, params, x, dy, T=T, rank=rank, group=group, comm=MERAK_COMM_NVLS, n_sub=1)
        for k in outv:
            if not torch.equal(outv[k], outv2[k]):
                failures.append((name, f"nvls: {k} not run-to-run deterministic"))
            if not torch.equal(outv[k], outv1[k]):
                failures.append((name, f"nvls: {k}: n={cfg.n_sub} vs n=1 not bit-identical"))
    # sequence-parallel layout across processes (NEXT-2): y / dx / weight gradients bit-identical to the replicated
    # layout (each rank's token shard), LN gradients within 1e-5
    from paper_2206_04959_b200 import FLAG_CHAIN as _FC, PARAM_NAMES, TmpLayer, shard_weights, sp_rows, zero_grads_like
    scfg = tiny.with_(hidden=256, heads=8, seq_len=128, microbatch=4, n_sub=2, tmp_degree=T)
    sparams, sx, sdy = make_all(scfg, seed=77)
    ref = run_gpu_layer(scfg, sparams, sx, sdy, T=T, rank=rank, group=group)
    dev = torch.device("cuda", torch.cuda.current_device())
    lay = TmpLayer(scfg.hidden, scfg.heads, scfg.seq_len, scfg.microbatch, tmp_degree=T, tmp_rank=rank, n_sub=2,
                   device=dev.index, group=group, seq_parallel=True)
    rows = sp_rows(scfg.tokens, 2, T, rank).to(dev)
    X = torch.as_tensor(np.asarray(sx).reshape(scfg.tokens, scfg.hidden)).to(dev, torch.bfloat16)[rows].contiguous()
    DY = torch.as_tensor(np.asarray(sdy).reshape(scfg.tokens, scfg.hidden)).to(dev, torch.bfloat16)[rows].contiguous()
    w = shard_weights(sparams, scfg.heads, T, rank, dev)
    G = zero_grads_like(w)
    Y, DX, SV = torch.empty_like(X), torch.empty_like(X), lay.new_saved()
    lay.forward(w, X, Y, SV)
    lay.backward(w, X, SV, DY, DX, G)
    torch.cuda.synchronize()
    lay.close()
    if not (torch.equal(Y, ref["y"][rows]) and torch.equal(DX, ref["dx"][rows])):
        failures.append(("seqpar", "y / dx differ from the replicated layout"))
    for k in PARAM_NAMES:
        if k.startswith("ln"):
            if (G[k] - ref[k]).norm() > 1e-5 * ref[k].norm() + 1e-6:
                failures.append(("seqpar", f"{k} off"))
        elif not torch.equal(G[k], ref[k]):
            failures.append(("seqpar", f"{k} not bit-identical to the replicated layout"))
    print(f"[rank {rank}] seqpar T={T} done", flush=True)
    # chained stack (cross-layer overlap + workspace hazards across ranks): chained == unchained bitwise
    from gpu_layer_util import run_gpu_chain
    from synth import make_activations, make_params
    ccfg = tiny.with_(hidden=256, heads=4, seq_len=128, microbatch=4, n_sub=2, tmp_degree=T)
    cparams = [make_params(ccfg, layer=k) for k in range(3)]
    cx, cdy = make_activations(ccfg)
    ca = run_gpu_chain(ccfg, cparams, cx, cdy, T=T, rank=rank, group=group, chain=True)
    cb = run_gpu_chain(ccfg, cparams, cx, cdy, T=T, rank=rank, group=group, chain=False)
    if not (torch.equal(ca["y"], cb["y"]) and torch.equal(ca["dx"], cb["dx"]) and
            all(torch.equal(ca["grads"][k][nm], cb["grads"][k][nm]) for k in range(3) for nm in ca["grads"][k])):
        failures.append(("chain", "chained vs unchained not bit-identical"))
    print(f"[rank {rank}] chain T={T} done", flush=True)
    dist.barrier()
    if failures:
        print(f"[rank {rank}] FAIL {failures}", flush=True)
    ok = torch.tensor([0 if failures else 1], device="cuda")
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    dist.destroy_process_group()
    sys.exit(0 if ok.item() == 1 else 1)


if __name__ == "__main__":
    main()
