#!/usr/bin/env python
"""Benchmark of the sub-pipelined TMP transformer layer (Merak §6.3) on B200.

python bench.py --gpus N --steps K --warmup W            (N > 1: launched by torchrun, one rank per GPU)
python bench.py --impl reference ...                      (the fp64 CPU oracle as the reference arm)

One step = forward + backward of a stack of L (default 4) chained layers with distinct weights (every
SURVEY §8(a) row: LN1, QKV, attention, proj, AR#1 + LN2, fc1 + GeLU, fc2, AR#2, and the backward mirror
with AR#3 / AR#4 and all weight gradients), so the all-reduce of one layer overlaps the next layer's first
sub-batch, over one microbatch of the headline workload: the GPT-20B-shaped layer of
BASELINE.json configs[4] (h=6144, H=64, s=2048, B=4, n=2 sub-batches), the largest configuration, which
fits one GPU at T = 1.  The TMP degree is T = N (rank r holds shard r; strong scaling, the model is fixed).
Inputs are synthetic (synth/, seeded), resident in HBM; the per-step working set (weights, gradients,
saved activations: > 10 GB at T = 1) is far larger than the 126 MB L2, so no flush is needed.
value = algorithmic TFLOP/s PER GPU of the layer ((72Bsh^2 + 6Bhs(s+1)) x L FLOPs per step / N / device
time, max over ranks), as BASELINE.json's metric states.  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TMP layer fwd+bwd TFLOP/s/GPU at TMP=1/2/4/8; exposed all-reduce ms/layer"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--layers", type=int, default=4, help="L chained layers per step (distinct weights)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="merak", choices=["merak", "reference"])
    ap.add_argument("--config", default="gpt20b")
    ap.add_argument("--n-sub", type=int, default=None)
    ap.add_argument("--comm-ctas", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the n=1 / no-comm / e2e / side-workload / profiling passes")
    return ap.parse_args()


def layer_flops(cfg):
    """Algorithmic fwd+bwd FLOPs of one unsharded layer: 72 B s h^2 (GEMMs, f = 4h) + 6 B h s (s+1)
    (causal attention) -- DESIGN.md §5, pinned in tests/test_oracle_pins.py::test_layer_flops_pin."""
    B, s, h = cfg.microbatch, cfg.seq_len, cfg.hidden
    f = cfg.ffn
    return 6.0 * B * s * (4 * h * h + 2 * f * h) + 6.0 * B * h * s * (s + 1)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("bf16_tflops", 1590.0), d.get("bf16_tflops_sustained", 1400.0), "measured"
    return 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock, power and clock-event (throttle) reasons sampled every ~5 ms through NVML from a
    background thread while the timed region runs."""

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = None
        self._t = None

    def __enter__(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.index]) if vis and vis.split(",")[self.index].isdigit() else self.index
            h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self._max = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception:
            return self
        self._stop = threading.Event()
        flags = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                 "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                 "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                 "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}

        def run():
            while not self._stop.is_set():
                try:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
                    self.rows.append((sm, [k for k, f in flags.items() if rs & f], pw))
                except Exception:
                    pass
                self._stop.wait(0.005)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        if self._t:
            self._stop.set()
            self._t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        reasons = sorted({r for row in self.rows for r in row[1]})
        return {"sm_mhz": statistics.median([r[0] for r in self.rows]), "sm_max_mhz": float(self._max),
                "reasons": reasons, "samples": len(self.rows), "power_w_max": max(r[2] for r in self.rows),
                "source": "NVML, ~5 ms period, timed region only"}


def _use_host_cores():
    """torchrun sets OMP_NUM_THREADS=1; the oracle is timed on all of the host cores this process may use."""
    try:
        import numpy  # noqa: F401  (load the BLAS first, then raise its thread limit)
        from threadpoolctl import threadpool_limits
        threadpool_limits(len(os.sched_getaffinity(0)))
    except Exception:
        pass


def _blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads") or 1 for i in threadpool_info()] or [1])
    except Exception:
        return os.cpu_count()


_SAMPLES = {}


def oracle_sample(cfg, tokens):
    """The bounded oracle sample: ONE sample of the workload's layer (full h, H, weights), restricted to its
    first `tokens` positions.  Attention is causal, so these positions' outputs do not depend on later ones:
    the sample is exactly a prefix of the workload's computation.  Returns (seconds, FLOPs)."""
    _use_host_cores()
    from oracle import layer_flops as oflops, layer_fwd_bwd
    from synth import make_all
    sub = cfg.with_(microbatch=1, seq_len=tokens)
    key = (sub.name, sub.hidden, tokens)
    if key not in _SAMPLES:  # drawing a full-h layer's weights takes ~20 s: once per sample shape
        _SAMPLES[key] = make_all(sub)
    params, x, dy = _SAMPLES[key]
    t0 = time.perf_counter()
    layer_fwd_bwd(params, x, dy, sub.heads)
    dt = time.perf_counter() - t0
    return dt, oflops(1, tokens, sub.hidden, sub.heads)


def cpu_oracle_baseline(cfg, tokens=512):
    dt, fl = oracle_sample(cfg, tokens)
    return {"value": fl / dt / 1e12, "unit": "TFLOP/s", "cores": _blas_threads(), "kind": "oracle",
            "sample": f"1 of the {cfg.microbatch} samples of the {cfg.name} layer (h={cfg.hidden}, H={cfg.heads}), "
                      f"its first {tokens} of {cfg.seq_len} positions (a causal prefix), fwd+bwd, unsharded, fp64 "
                      f"numpy: {dt:.2f} s, {fl / 1e9:.0f} GFLOP",
            "seconds": dt, "host_cores_visible": len(os.sched_getaffinity(0))}


def arm_config(cfg, L, T, n_sub):
    """The workload both arms report (the reference arm times a bounded sample of it)."""
    return {"workload": f"{cfg.name} layer fwd+bwd x {L} chained layers: h={cfg.hidden}, H={cfg.heads}, "
                        f"s={cfg.seq_len}, B={cfg.microbatch}, TMP={T}, n_sub={n_sub}",
            "layers": L, "tmp_degree": T, "n_sub": n_sub, "hidden": cfg.hidden, "heads": cfg.heads,
            "seq_len": cfg.seq_len, "microbatch": cfg.microbatch,
            "l2": "not flushed: the per-step working set (weights, fp32 grads, saved activations) is >> 126 MB L2"}


def run_reference(args, cfg, rank, world):
    """--impl reference: the CPU oracle as it stands; each step a bounded sample of the workload (one sample,
    a causal prefix of 128 positions, full h).  Rank 0 only; other ranks exit without work."""
    if rank != 0:
        return
    tokens = 128
    for _ in range(args.warmup):
        oracle_sample(cfg, tokens)
    tot, fl = 0.0, 0.0
    for _ in range(args.steps):
        dt, f = oracle_sample(cfg, tokens)
        tot += dt
        fl += f
    v = fl / tot / 1e12
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": arm_config(cfg, args.layers, world, cfg.n_sub),
            "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": _blas_threads(), "kind": "oracle",
                             "sample": f"bounded sample: each step = 1 of the {cfg.microbatch} samples of one "
                                       f"{cfg.name} layer, its first {tokens} positions (causal prefix), fwd+bwd, "
                                       f"unsharded, fp64 numpy"},
            "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


class Stack:
    """L chained layers of one rank (weights, grads, saved activations, outputs) on one TmpLayer handle."""

    def __init__(self, cfg, L, T, rank, dev, group, n_sub, comm=0, comm_ctas=0, streams1=False, seq_parallel=False):
        import torch

        from paper_2206_04959_b200 import TmpLayer, shard_weights, sp_rows, zero_grads_like
        from synth import make_activations_torch, make_params_torch
        self.cfg, self.L, self.T, self.dev = cfg, L, T, dev
        self.X, self.DY = make_activations_torch(cfg, dev)
        if seq_parallel:  # this rank's token shard (merak_tmp.h, sequence-parallel layout)
            rows = sp_rows(cfg.tokens, n_sub, T, rank).to(dev)
            self.X, self.DY = self.X[rows].contiguous(), self.DY[rows].contiguous()
        self.ws = [shard_weights(make_params_torch(cfg, dev, layer=k), cfg.heads, T, rank, dev) for k in range(L)]
        self.Ys = [torch.empty_like(self.X) for _ in range(L)]
        self.DXs = [torch.empty_like(self.X) for _ in range(L)]
        self.grads = [zero_grads_like(w) for w in self.ws]
        if streams1:
            os.environ["MERAK_STREAMS"] = "1"
        try:
            self.layer = TmpLayer(cfg.hidden, cfg.heads, cfg.seq_len, cfg.microbatch, tmp_degree=T, tmp_rank=rank,
                                  n_sub=n_sub, comm=comm, comm_ctas=comm_ctas, device=dev.index, group=group,
                                  seq_parallel=seq_parallel)
        finally:
            if streams1:
                del os.environ["MERAK_STREAMS"]
        self.saved = [self.layer.new_saved() for _ in range(L)]

    def step(self, flags=0, X=None, DY=None, recompute=None):
        """L layers forward, then backward in reverse (overlap across layers): every call but the last
        backward passes MERAK_FLAG_CHAIN, so layer k+1's sub-batch 0 starts while layer k's last all-reduce is
        in flight; the last backward joins the caller stream.  recompute: per-layer bools -- those layers keep
        no activations (their forward writes a shared scratch buffer) and regenerate them inside the backward
        (MERAK_FLAG_RECOMPUTE)."""
        from paper_2206_04959_b200 import FLAG_CHAIN, FLAG_RECOMPUTE
        X = self.X if X is None else X
        DY = self.DY if DY is None else DY
        L, lay = self.L, self.layer
        rc = list(recompute) if recompute is not None else [False] * L
        if any(rc) and getattr(self, "scratch", None) is None:
            self.scratch = lay.new_saved()
        sv = [self.scratch if rc[k] else self.saved[k] for k in range(L)]
        for k in range(L):
            lay.forward(self.ws[k], X if k == 0 else self.Ys[k - 1], self.Ys[k], sv[k], flags=flags | FLAG_CHAIN)
        for k in reversed(range(L)):
            lay.backward(self.ws[k], X if k == 0 else self.Ys[k - 1], sv[k],
                         DY if k == L - 1 else self.DXs[k + 1], self.DXs[k], self.grads[k],
                         flags=flags | (FLAG_CHAIN if k > 0 else 0) | (FLAG_RECOMPUTE if rc[k] else 0))

    def close(self):
        self.layer.close()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    from synth import CONFIGS
    cfg = CONFIGS[args.config]
    T = world
    n_sub = args.n_sub or cfg.n_sub
    cfg = cfg.with_(tmp_degree=T, n_sub=n_sub)
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import torch
    import torch.distributed as dist

    from paper_2206_04959_b200 import FLAG_NO_COMM

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD
    L = args.layers
    stack = Stack(cfg, L, T, rank, dev, group, n_sub, comm_ctas=args.comm_ctas)
    stream = torch.cuda.current_stream()
    t_start = time.time()

    def stage(msg):  # progress markers on stderr (multi-rank runs: evidence if a run ever stalls)
        if world > 1 or os.environ.get("MERAK_BENCH_TRACE"):
            print(f"[rank {rank} +{time.time() - t_start:.1f}s] {msg}", file=sys.stderr, flush=True)

    import faulthandler
    faulthandler.dump_traceback_later(int(os.environ.get("MERAK_BENCH_TRACE_S", "300")), exit=False)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def timed(st, nsteps, flags=0, prof=False, recompute=None):
        """nsteps back-to-back steps between one pair of CUDA events on the caller stream, bracketed by
        synchronize + barrier; returns (max-over-ranks ms per step, kernel launches, profile)."""
        if prof:
            st.layer.set_profiling(True)
        l0 = st.layer.launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        for _ in range(nsteps):
            st.step(flags, recompute=recompute)
        e1.record(stream)
        barrier()
        launches = st.layer.launch_count() - l0
        prof_d = st.layer.get_profile() if prof else None
        if prof:
            st.layer.set_profiling(False)
        return max_over_ranks(e0.elapsed_time(e1) / nsteps), launches, prof_d

    for _ in range(args.warmup):
        stack.step()
    barrier()
    stage("warmup done")
    with ClockSampler(local) as clk:
        ms_step, launches, _ = timed(stack, args.steps)
    clocks = clk.summary()
    stage("timed done")
    fl = L * layer_flops(cfg)
    value = fl / world / (ms_step * 1e-3) / 1e12  # per GPU (BASELINE.json metric)

    extras = {}
    if not args.no_extras:
        nx = max(3, args.steps // 2)
        # exposed communication: same kernels with every all-reduce reading only the local partial
        if T > 1:
            ms_nc, _, _ = timed(stack, nx, flags=FLAG_NO_COMM)
            extras["exposed_allreduce_ms_per_layer"] = (ms_step - ms_nc) / L
            extras["exposed_allreduce_frac"] = (ms_step - ms_nc) / ms_step
            extras["no_comm_ms_per_step"] = ms_nc
            stage("no-comm done")
            rows = cfg.tokens // n_sub
            dh = stack.layer.debug_host()
            two, push = dh["two_shot"], dh["push"] and dh["two_shot"] and (rows // T) % 32 == 0
            t_f = stack.layer.bench_allreduce(0, rows, 20)
            t_b = stack.layer.bench_allreduce(1, rows, 20)
            t_h = stack.layer.bench_allreduce(0, rows // 2, 20)
            msg = rows * cfg.hidden * 2
            # bytes each GPU moves over NVLink per AR in the timed kernels (pull: loads from the peers; push: the
            # reduce-scatter half travels inside the GEMM epilogue, the timed part stores the all-gather half)
            nvl = ((T - 1) / T if push else 2 * (T - 1) / T if two else (T - 1)) * msg
            alg = "two-shot, reduce-scatter pushed by the GEMM epilogue (not timed here)" if push else \
                "two-shot" if two else "one-shot"
            extras["allreduce"] = {"algorithm": alg, "rows": rows, "msg_bytes": msg,
                                   "nvlink_bytes_in_per_gpu": nvl, "fwd_ar_us": t_f * 1e3, "bwd_ar_us": t_b * 1e3,
                                   "achieved_GBps": nvl / (t_f * 1e-3) / 1e9, "peak_GBps": 900.0,
                                   "frac": nvl / (t_f * 1e-3) / 900e9,
                                   "marginal_GBps": (nvl / 2) / ((t_f - t_h) * 1e-3) / 1e9 if t_f > t_h else None,
                                   "fixed_us": (2 * t_h - t_f) * 1e3,
                                   "note": "forward AR#2 alone on the comm stream incl. handshake kernel(s); "
                                           "peak = NVLink 5 per direction"}
            stage("allreduce bench done")
        else:
            extras["exposed_allreduce_ms_per_layer"] = 0.0
        # n = 1 (Megatron-style, no sub-pipelining) with the same kernels: fig:ablation_pipetp analog
        if n_sub != 1:
            stack.layer.set_subbatches(1)
            stack.step()
            ms_n1, _, _ = timed(stack, nx)
            stack.layer.set_subbatches(n_sub)
            stack.step()
            extras["n1_ms_per_step"] = ms_n1
            extras["subpipelining_speedup_vs_n1"] = ms_n1 / ms_step
            stage("n=1 done")
        extras["e2e"] = e2e_pass(stack, nx, world, rank, dev, fl, dist, barrier, max_over_ranks)
        stage("e2e done")
        extras["roofline"], extras["serialized_ms_per_step"] = roofline_pass(cfg, L, T, rank, dev, group, n_sub, args,
                                                                             timed, value)
        stage("profiling pass done")
        extras["recompute"] = recompute_pass(cfg, L, stack, timed, ms_step, nx)
        stage("recompute pass done")
        extras["side_workloads"] = side_workloads(args, T, rank, dev, group, timed, stack)
        stage("side workloads done")
        if world > 1:
            def guarded(name, fn, *a):
                # side passes are deterministic across ranks: a failure on one is a failure on all, so it is
                # recorded in the line instead of losing the measured headline
                try:
                    extras[name] = fn(*a)
                except Exception as e:  # noqa: BLE001
                    extras[name] = {"error": f"{type(e).__name__}: {e}"[:300]}
                stage(f"{name} pass done")
            guarded("nvls", nvls_pass, args, cfg, L, T, rank, dev, group, n_sub, timed, ms_step)
            guarded("seq_parallel", seqpar_pass, args, cfg, L, T, rank, dev, group, n_sub, timed, ms_step)
            guarded("push", push_pass, args, cfg, L, T, rank, dev, group, n_sub, timed, ms_step)
            guarded("pipeline", pipeline_pass, args, rank, world, dev, barrier, max_over_ranks)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded, synth/)",
                "config": arm_config(cfg, L, T, n_sub), "flops_per_step": fl, "ms_per_layer": ms_step / L,
                "value_whole_job": value * world, "tokens_per_s": L * cfg.tokens / (ms_step * 1e-3),
                "gpu_launches": launches, "clocks": clocks}
        for k in ("roofline", "e2e"):
            if k in extras:
                line[k] = extras[k]
        line.update({k: v for k, v in extras.items() if k not in ("roofline", "e2e")})
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_oracle_baseline(cfg)
        print(json.dumps(line), flush=True)
    stack.close()
    faulthandler.cancel_dump_traceback_later()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def e2e_pass(stack, ne, world, rank, dev, fl, dist, barrier, max_over_ranks):
    """The same metric through the public API with HOST buffers: every step uploads its x and dy from pinned
    host memory and downloads y and dx (all inside the timed region, on copy streams), double-buffered as an
    input pipeline would be.  x, dy, y, dx are replicated on the T ranks: each rank moves its 1/T row slice
    over PCIe and the slices are all-gathered over NVLink (NCCL)."""
    import torch

    from paper_2206_04959_b200 import FLAG_CHAIN
    X, DY, L = stack.X, stack.DY, stack.L
    M = X.shape[0]
    rows = M // world
    r0 = rank * rows
    hx = X[r0:r0 + rows].cpu().pin_memory()
    hdy = DY[r0:r0 + rows].cpu().pin_memory()
    hy = torch.empty_like(hx).pin_memory()
    hdx = torch.empty_like(hx).pin_memory()
    Xb, DYb = [torch.empty_like(X) for _ in range(2)], [torch.empty_like(DY) for _ in range(2)]
    stream = torch.cuda.current_stream()

    def upload(bi_):
        if world == 1:
            Xb[bi_].copy_(hx, non_blocking=True)
            DYb[bi_].copy_(hdy, non_blocking=True)
            return
        Xb[bi_][r0:r0 + rows].copy_(hx, non_blocking=True)
        DYb[bi_][r0:r0 + rows].copy_(hdy, non_blocking=True)
        dist.all_gather_into_tensor(Xb[bi_], Xb[bi_][r0:r0 + rows])
        dist.all_gather_into_tensor(DYb[bi_], DYb[bi_][r0:r0 + rows])
    cp = torch.cuda.Stream(device=dev)    # uploads (H2D copy engine)
    cpo = torch.cuda.Stream(device=dev)   # downloads (D2H copy engine)
    lay, ws, Ys, DXs, saved, grads = stack.layer, stack.ws, stack.Ys, stack.DXs, stack.saved, stack.grads
    barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    cp.wait_stream(stream)
    ev_in, ev_free, ev_y, ev_dx = [None, None], [None, None], None, None
    with torch.cuda.stream(cp):
        upload(0)
    ev_in[0] = cp.record_event()
    for i in range(ne):
        bb = i & 1
        stream.wait_event(ev_in[bb])
        if i + 1 < ne:  # prefetch the next step's inputs once their buffer's last use (step i-1) is done
            if ev_free[1 - bb] is not None:
                cp.wait_event(ev_free[1 - bb])
            with torch.cuda.stream(cp):
                upload(1 - bb)
            ev_in[1 - bb] = cp.record_event()
        if ev_y is not None:
            stream.wait_event(ev_y)  # the previous y download has read Ys[L-1]
        for k in range(L):
            # the last forward joins the caller stream, so y is complete when the copy stream reads it
            lay.forward(ws[k], Xb[bb] if k == 0 else Ys[k - 1], Ys[k], saved[k], flags=FLAG_CHAIN if k < L - 1 else 0)
        cpo.wait_stream(stream)
        with torch.cuda.stream(cpo):
            hy.copy_(Ys[L - 1][r0:r0 + rows], non_blocking=True)
        ev_y = cpo.record_event()
        if ev_dx is not None:
            stream.wait_event(ev_dx)  # the previous dx download has read DXs[0]
        for k in reversed(range(L)):
            lay.backward(ws[k], Xb[bb] if k == 0 else Ys[k - 1], saved[k], DYb[bb] if k == L - 1 else DXs[k + 1],
                         DXs[k], grads[k], flags=FLAG_CHAIN if k > 0 else 0)
        ev_free[bb] = stream.record_event()
        cpo.wait_event(ev_free[bb])
        with torch.cuda.stream(cpo):
            hdx.copy_(DXs[0][r0:r0 + rows], non_blocking=True)
        ev_dx = cpo.record_event()
    stream.wait_stream(cp)
    stream.wait_stream(cpo)
    t1.record(stream)
    barrier()
    te = max_over_ranks(t0.elapsed_time(t1) / ne)
    return {"value": fl / world / (te * 1e-3) / 1e12, "unit": "TFLOP/s",
            "h2d_bytes_per_step": 2 * hx.numel() * 2, "d2h_bytes_per_step": 2 * hx.numel() * 2,
            "ms_per_step": te, "steps": ne,
            "note": "per GPU; pinned-host x, dy up and y, dx down every step (upload and download copy streams), "
                    "double-buffered like an input pipeline, timed with the same event structure as `value` "
                    "(one event pair around back-to-back steps); the extra join after the last forward (y must be "
                    "complete before its download) is the only schedule difference; at T > 1 each rank moves its "
                    "1/T row slice over PCIe and the inputs are all-gathered over NVLink (NCCL); bytes are per GPU"}


def recompute_pass(cfg, L, stack, timed, ms_step, nx):
    """the same stack with every layer recomputing its activations in
    the backward (MERAK_FLAG_RECOMPUTE), and the stage-aware plan (merak_tune_alpha1 / merak_stage_alpha) for a
    pipeline of s stages of these L layers on this GPU's memory, timed with stage 1's recompute count."""
    import torch

    from paper_2206_04959_b200.planner import recompute_plan
    all_rc = [True] * L
    stack.step(recompute=all_rc)
    ms_rc, _, _ = timed(stack, nx, recompute=all_rc)
    lay = stack.layer
    sb = lay.saved_bytes()
    wbytes = sum(t.numel() * t.element_size() for t in stack.ws[0].values())
    gbytes = sum(t.numel() * t.element_size() for t in stack.grads[0].values())
    cap = float(torch.cuda.get_device_properties(stack.dev).total_memory)
    # runtime memory of a stage of L layers: weights + fp32 grads + one microbatch's activations (the one being
    # computed) + the boundary activations / workspace (x, y, dy, dx per layer), M_a = one microbatch's
    # activations of the stage
    act_io = 4 * stack.X.numel() * stack.X.element_size()
    m_r = L * (wbytes + gbytes + act_io) + L * sb
    out = {"all_layers_recompute_ms_per_step": ms_rc, "no_recompute_ms_per_step": ms_step,
           "recompute_overhead_frac": ms_rc / ms_step - 1.0, "saved_bytes_per_layer": sb,
           "note": "recompute regenerates LN1, QKV, attention, proj + AR#1 + LN2, fc1 + GeLU (fc2 / AR#2 skipped); "
                   "bit-identical results (tests/test_gpu_recompute.py)", "plans": {}}
    for s in (4, 8):
        try:
            plan = recompute_plan(s, L, cap, m_r, sb)
        except Exception as e:  # noqa: BLE001  (runtime memory alone exceeds capacity)
            out["plans"][f"s{s}"] = {"error": str(e)}
            continue
        keep0 = plan["layers_kept"][0]
        rc = [k >= keep0 for k in range(L)]  # stage 1 keeps the activations of its first layers_kept[0] layers
        ms_plan = timed(stack, nx, recompute=rc)[0] if keep0 < L else ms_step
        plan.update({"stage1_recomputed_layers": L - keep0, "stage1_ms_per_step": ms_plan,
                     "capacity_bytes": cap, "m_r_bytes": m_r, "m_a_bytes": L * sb})
        out["plans"][f"s{s}"] = plan
    return out


def nvls_pass(args, cfg, L, T, rank, dev, group, n_sub, timed, ms_step):
    """the same stack with MERAK_COMM_NVLS (reduce-scatter phase in the NVSwitch with
    multimem.ld_reduce / multimem.st): per-GPU TFLOP/s, exposed all-reduce, and the all-reduce alone."""
    from paper_2206_04959_b200 import FLAG_NO_COMM, MERAK_COMM_NVLS, MerakError
    nx = max(3, args.steps // 2)
    try:
        st = Stack(cfg, L, T, rank, dev, group, n_sub, comm=MERAK_COMM_NVLS, comm_ctas=args.comm_ctas)
    except MerakError as e:
        return {"unavailable": str(e)}
    for _ in range(3):
        st.step()
    ms, _, _ = timed(st, nx)
    ms_nc, _, _ = timed(st, nx, flags=FLAG_NO_COMM)
    rows = cfg.tokens // n_sub
    t_f = st.layer.bench_allreduce(0, rows, 20)
    t_b = st.layer.bench_allreduce(1, rows, 20)
    st.close()
    fl = L * layer_flops(cfg)
    msg = rows * cfg.hidden * 2
    return {"tflops_per_gpu": fl / T / (ms * 1e-3) / 1e12, "ms_per_step": ms, "vs_peer_two_shot": ms_step / ms,
            "exposed_allreduce_ms_per_layer": (ms - ms_nc) / L, "exposed_allreduce_frac": (ms - ms_nc) / ms,
            "allreduce": {"rows": rows, "msg_bytes": msg, "fwd_ar_us": t_f * 1e3, "bwd_ar_us": t_b * 1e3,
                          "algbw_GBps": msg / (t_f * 1e-3) / 1e9,
                          "note": "algorithmic bandwidth = message bytes / time (the all-reduce of one [m, h] bf16 "
                                  "partial incl. handshakes); NVLS moves ~(1 + 1/T) x msg per GPU and direction"}}


def seqpar_pass(args, cfg, L, T, rank, dev, group, n_sub, timed, ms_step):
    """the same stack in the sequence-parallel layout (token-sharded x / y, reduce-scatter
    epilogues on the own rows, all-gathers of u, u2, dy, dx1): per-GPU TFLOP/s next to the replicated layout."""
    from paper_2206_04959_b200 import MerakError
    nx = max(3, args.steps // 2)
    try:
        st = Stack(cfg, L, T, rank, dev, group, n_sub, comm_ctas=args.comm_ctas, seq_parallel=True)
    except MerakError as e:
        return {"unavailable": str(e)}
    for _ in range(3):
        st.step()
    ms, _, _ = timed(st, nx)
    st.close()
    return {"tflops_per_gpu": L * layer_flops(cfg) / T / (ms * 1e-3) / 1e12, "ms_per_step": ms,
            "vs_replicated": ms_step / ms,
            "note": "x / y / dx / dy token-sharded by T; the LN / residual epilogues run on the own rows"}


def push_pass(args, cfg, L, T, rank, dev, group, n_sub, timed, ms_step):
    """SURVEY §8(f) NEXT-2, tile-granular fusion (MERAK_AR_PUSH=1): the row-parallel GEMMs (proj, fc2, fc1 / QKV
    dgrad) store each 32-row output box straight into the owner rank's slot over NVLink, so the reduce-scatter
    phase (two-shot phase 1, or the sequence-parallel reduce-scatter) reads only local HBM.  Per-GPU TFLOP/s of
    the replicated two-shot and the sequence-parallel layouts next to the main line."""
    from paper_2206_04959_b200 import FLAG_NO_COMM, MerakError
    nx = max(3, args.steps // 2)
    keep = {k: os.environ.get(k) for k in ("MERAK_AR_PUSH", "MERAK_AR_TWO_SHOT")}
    os.environ["MERAK_AR_TWO_SHOT"] = "1"
    out = {}
    try:
        # mode 1: reduce-scatter push; mode 2: + the reduced rows pushed into every rank's all-gather slot
        for name, sp, mode in (("two_shot", False, "1"), ("two_shot_ag", False, "2"), ("seq_parallel", True, "1")):
            os.environ["MERAK_AR_PUSH"] = mode
            try:
                st = Stack(cfg, L, T, rank, dev, group, n_sub, comm_ctas=args.comm_ctas, seq_parallel=sp)
            except MerakError as e:
                out[name] = {"unavailable": str(e)}
                continue
            for _ in range(3):
                st.step()
            ms, _, _ = timed(st, nx)
            r = {"tflops_per_gpu": L * layer_flops(cfg) / T / (ms * 1e-3) / 1e12, "ms_per_step": ms,
                 "vs_main": ms_step / ms, "push_active": st.layer.debug_host()["push"]}
            if not sp:
                ms_nc, _, _ = timed(st, nx, flags=FLAG_NO_COMM)
                r["exposed_allreduce_ms_per_layer"] = (ms - ms_nc) / L
                r["exposed_allreduce_frac"] = (ms - ms_nc) / ms
            st.close()
            out[name] = r
    finally:
        for k, v in keep.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    out["note"] = "row-parallel GEMM epilogues push 32-row boxes to the owner's slot (TMA store via peer tensor maps)"
    return out


def pipeline_pass(args, rank, world, dev, barrier, max_over_ranks, K=2, layer_cfg="gpt1.5b"):
    """a pipeline of P = N stages (one per GPU, T = 1 each), K layers of the
    gpt1.5b shape per stage, m = 2P microbatches, driven by each schedule of merak_pipeline_schedule over NCCL
    point-to-point.  Per policy: iteration time (max over ranks) and the measured bubble ratio against the
    stage's own busy time -- the same actions run back to back on each GPU with no inputs to wait for (max
    over ranks) -- next to the paper's ratio (P:460 (s-1)/m, P:461 3(s-1)/(4m), P:470 3(s-2)/(4m))."""
    import torch
    import torch.distributed as dist

    from paper_2206_04959_b200 import TmpLayer, shard_weights, zero_grads_like
    from paper_2206_04959_b200.pipeline import PipelineStage, run_distributed, schedule
    from synth import CONFIGS, make_activations_torch, make_params_torch
    cfg = CONFIGS[layer_cfg].with_(tmp_degree=1)
    s, m = world, 2 * world
    fwd_g, bwd_g = dist.new_group(list(range(world))), dist.new_group(list(range(world)))
    lay = TmpLayer(cfg.hidden, cfg.heads, cfg.seq_len, cfg.microbatch, n_sub=cfg.n_sub, device=dev.index)
    ws = [shard_weights(make_params_torch(cfg, dev, layer=rank * K + k), cfg.heads, 1, 0, dev) for k in range(K)]
    grads = [zero_grads_like(w) for w in ws]
    X, DY = make_activations_torch(cfg, dev)
    xs, dys = [X] * m, [DY] * m
    shape, dt = (cfg.tokens, cfg.hidden), torch.bfloat16
    paper = {"1f1b": (s - 1) / m, "early": 3 * (s - 1) / (4 * m), "scp": 3 * (s - 2) / (4 * m),
             "none": (s - 1) / m}
    out = {"stages": s, "microbatches": m, "layers_per_stage": K, "layer_config": layer_cfg, "tmp_degree": 1,
           "policies": {}}
    stream = torch.cuda.current_stream()

    def run(actions, solo):
        acts = actions
        # stages whose schedule recomputes nothing (SCP's last stage, "none") keep every layer's activations
        kept = 0 if any(k in ("R", "BR") for k, _ in acts) else K
        st = PipelineStage(lay, ws, grads, rank, s, kept=kept)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        if solo:  # the stage's own work back to back: no waiting for neighbours (pure busy time)
            for kind, mb in acts:
                if kind == "F":
                    st.forward(mb, X)
                elif kind == "R":
                    st.recompute(mb)
                else:
                    st.backward(mb, DY, fused_recompute=kind == "BR")
        else:
            run_distributed(st, acts, xs, dys, fwd_g, bwd_g, shape, dt, dev)
        e1.record(stream)
        barrier()
        return max_over_ranks(e0.elapsed_time(e1))

    for pol in ("1f1b", "early", "scp", "none"):
        acts = schedule(pol, s, m)[rank]
        for _ in range(2):
            run(acts, False)
        it = min(run(acts, False) for _ in range(3))
        busy = min(run(acts, True) for _ in range(2))
        out["policies"][pol] = {"iteration_ms": it, "stage_busy_ms": busy, "measured_bubble_ratio": it / busy - 1.0,
                                "paper_bubble_ratio": paper[pol]}
    lay.close()
    return out


def roofline_pass(cfg, L, T, rank, dev, group, n_sub, args, timed, value):
    """Roofline of the dominant kernel class (the tcgen05 GEMM): algorithmic FLOPs (2MNK per launch) over the
    CUDA-event durations of every GEMM launch, recorded on the stream that launches it.  The timed run overlaps
    kernels of different sub-batches (and the wgrad filler), so per-launch spans there include time shared with
    other kernels: this pass uses a second handle with all compute on one stream (MERAK_STREAMS=1): the same
    kernels, shapes and order as the ncu launch list."""
    st = Stack(cfg, L, T, rank, dev, group, n_sub, comm_ctas=args.comm_ctas, streams1=True)
    for _ in range(2):
        st.step()
    nprof = max(3, args.steps // 4)
    ms_serial, _, prof = timed(st, nprof, prof=True)
    st.close()
    peak_burst, peak_sust, peak_src = measured_peaks()
    g = prof["gemm"]
    gemm_tflops = g["flops"] / (g["ms"] * 1e-3) / 1e12 if g["ms"] > 0 else 0.0
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", f"gemm_traffic_{cfg.name}_T{T}.json")
    if os.path.exists(tr_path):
        traffic = json.load(open(tr_path)).get("dram_bytes_per_launch")
    share = {k: v["ms"] / nprof / L for k, v in prof.items()}
    attn = {k: prof[k]["flops"] / (prof[k]["ms"] * 1e-3) / 1e12 if prof[k]["ms"] > 0 else None
            for k in ("attn_fwd", "attn_bwd")}
    return ({"bound": "tensor", "achieved": gemm_tflops, "peak": peak_burst, "unit": "TFLOP/s",
             "frac": gemm_tflops / peak_burst, "traffic": traffic,
             "kernel": "tcgen05 bf16 GEMM (all 12 layer GEMMs; FLOPs 2MNK per launch / event-timed duration, "
                       "serialized profiling pass)",
             "peak_source": f"{peak_src} bf16_tflops (burst); sustained {peak_sust}",
             "gemm_launches_per_step": g["launches"] / nprof, "gemm_ms_per_layer": g["ms"] / nprof / L,
             "class_ms_per_layer": share,
             "class_share_of_kernel_time": {k: v / max(sum(share.values()), 1e-9) for k, v in share.items()},
             "attention_tflops": attn,
             "layer_frac_of_peak": value / peak_burst}, ms_serial)


def side_workloads(args, T, rank, dev, group, timed, main_stack):
    """Extra measured keys: the gpt1.5b stack at the same T = N, and (N = 1 only) the per-rank compute of the
    TMP = 8 shards of gpt8.3b and gpt20b (MERAK_COMM_LOCAL: one process runs rank 0 of an 8-way group; every
    all-reduce reads the local partial, so this is per-GPU compute only, not the layer's result)."""
    from paper_2206_04959_b200 import MERAK_COMM_LOCAL
    from synth import CONFIGS
    out = {}
    nx = max(3, args.steps // 2)
    jobs = []
    if args.config != "gpt1.5b":
        jobs.append(("gpt1.5b", CONFIGS["gpt1.5b"].with_(tmp_degree=T), T, 0))
    if T == 1:
        jobs.append(("gpt8.3b_T8_rank_shard", CONFIGS["gpt8.3b"], 8, MERAK_COMM_LOCAL))
        jobs.append(("gpt20b_T8_rank_shard", CONFIGS["gpt20b"], 8, MERAK_COMM_LOCAL))
    for name, c, tt, comm in jobs:
        st = Stack(c, args.layers, tt, 0 if comm else rank, dev, None if comm else group, c.n_sub, comm=comm)
        for _ in range(3):
            st.step()
        ms, _, _ = timed(st, nx)
        st.close()
        fl = args.layers * layer_flops(c) / tt
        out[name] = {"tflops_per_gpu": fl / (ms * 1e-3) / 1e12, "ms_per_step": ms, "ms_per_layer": ms / args.layers,
                     "tmp_degree": tt, "n_sub": c.n_sub, "layers": args.layers,
                     "mode": "per-rank compute only (MERAK_COMM_LOCAL)" if comm else f"full layer at T={tt}"}
        if comm:  # where the shard's time goes: per-class kernel ms per layer, all compute on one stream
            st = Stack(c, args.layers, tt, 0, dev, None, c.n_sub, comm=comm, streams1=True)
            st.step()
            np_ = 3
            ms1, _, prof = timed(st, np_, prof=True)
            st.close()
            out[name]["serialized_ms_per_layer"] = ms1 / args.layers
            out[name]["class_ms_per_layer"] = {k: v["ms"] / np_ / args.layers for k, v in prof.items()}
            g = prof.get("gemm")
            if g and g["ms"] > 0:
                out[name]["gemm_tflops_serialized"] = g["flops"] / (g["ms"] * 1e-3) / 1e12
    return out


if __name__ == "__main__":
    main()
