"""TMP = 8 projection (SURVEY §8(d) "TMP=8", gpurun caps at 4 GPUs).  Every number it writes is
labelled "projected (4-GPU limit)".

  phase "compute" (1 GPU):  per-rank compute of the T = 8 shapes, measured with MERAK_COMM_LOCAL (one
                            process emulates rank 0 of 8; every all-reduce reads only the local partial):
                            K chained layers fwd+bwd, ms per layer, for n_sub in {1, 2, 4}.
  phase "comm" (torchrun, 4 GPUs): for each config at T = 4: the layer with and without communication
                            (calibration of the overlap model) and the all-reduce alone at the T = 8
                            message sizes (m x h bf16 rows; m does not depend on T).
  phase "project" (CPU):    t_ar(T=8) = t_ar(T=4) x (2*7/8)/(2*3/4) (two-shot NVLink bytes per GPU);
                            layer(T=8) = compute(T=8) + exposed, with exposed from the two-stream model
                            (simulate() below) scaled by the measured/model ratio of
                            the T = 4 exposure.

Usage:  python tools/project_t8.py compute > gpurun_out/t8_compute.json
        torchrun --nproc-per-node 4 tools/project_t8.py comm > gpurun_out/t8_comm.json
        python tools/project_t8.py project gpurun_out/t8_compute.json gpurun_out/t8_comm.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CONFIGS_T8 = os.environ.get("T8_CONFIGS", "gpt8.3b,gpt20b,gpt2.5b,gpt1.5b").split(",")
K = 4


def layer_flops(cfg):
    B, s, h, f = cfg.microbatch, cfg.seq_len, cfg.hidden, cfg.ffn
    return 6.0 * B * s * (4 * h * h + 2 * f * h) + 6.0 * B * h * s * (s + 1)


_PARAMS = {}


def params_for(cfg, T, rank, dev):
    """Weights of K layers, generated once per (config, T, rank) and reused across n_sub."""
    from paper_2206_04959_b200 import shard_weights
    from synth import make_params
    key = (cfg.name, T, rank)
    if key not in _PARAMS:
        _PARAMS.clear()
        _PARAMS[key] = [shard_weights(make_params(cfg.with_(tmp_degree=T), layer=k), cfg.heads, T, rank, dev)
                        for k in range(K)]
    return _PARAMS[key]


def run_layers(cfg, T, rank, n_sub, comm, group, steps=6, warmup=3, flags=0):
    import torch
    import torch.distributed as dist

    from paper_2206_04959_b200 import FLAG_CHAIN, TmpLayer, zero_grads_like
    from synth import make_activations
    dev = torch.device("cuda", torch.cuda.current_device())
    c = cfg.with_(tmp_degree=T, n_sub=n_sub)
    x, dy = make_activations(c)
    ws = params_for(cfg, T, rank, dev)
    M, h = c.tokens, c.hidden
    X = torch.as_tensor(x.reshape(M, h)).to(dev, torch.bfloat16)
    DY = torch.as_tensor(dy.reshape(M, h)).to(dev, torch.bfloat16)
    Ys = [torch.empty_like(X) for _ in range(K)]
    DXs = [torch.empty_like(X) for _ in range(K)]
    grads = [zero_grads_like(w) for w in ws]
    layer = TmpLayer(c.hidden, c.heads, c.seq_len, c.microbatch, tmp_degree=T, tmp_rank=rank, n_sub=n_sub,
                     device=dev.index, group=group, comm=comm)
    saved = [layer.new_saved() for _ in range(K)]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step(fl):
        for k in range(K):
            layer.forward(ws[k], X if k == 0 else Ys[k - 1], Ys[k], saved[k], flags=fl | FLAG_CHAIN)
        for k in reversed(range(K)):
            layer.backward(ws[k], X if k == 0 else Ys[k - 1], saved[k], DY if k == K - 1 else DXs[k + 1], DXs[k],
                           grads[k], flags=fl | (FLAG_CHAIN if k > 0 else 0))

    def timed(fl):
        for _ in range(warmup):
            step(fl)
        ts = []
        for _ in range(steps):
            flush.zero_()
            torch.cuda.synchronize()
            if group is not None:
                dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            step(fl)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        t = torch.tensor([sum(ts) / len(ts)], dtype=torch.float64, device=dev)
        if group is not None:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item() / K

    out = {"ms_per_layer": timed(flags)}
    return layer, out, timed


def phase_compute():
    import torch

    from paper_2206_04959_b200 import MERAK_COMM_LOCAL
    from synth import CONFIGS
    torch.cuda.set_device(0)
    res = {}
    for name in CONFIGS_T8:
        cfg = CONFIGS[name]
        for n in (1, 2, 4):
            if cfg.microbatch % n:
                continue
            layer, o, _ = run_layers(cfg, 8, 0, n, MERAK_COMM_LOCAL, None)
            layer.close()
            res[f"{name}/n{n}"] = {"compute_ms_per_layer": o["ms_per_layer"],
                                   "tflops_per_gpu": layer_flops(cfg) / 8 / (o["ms_per_layer"] * 1e-3) / 1e12}
            print(name, n, res[f"{name}/n{n}"], file=sys.stderr, flush=True)
            torch.cuda.empty_cache()
    print(json.dumps({"phase": "compute", "T": 8, "rank": 0, "layers": K, "res": res}))


def phase_comm():
    import torch
    import torch.distributed as dist

    from paper_2206_04959_b200 import FLAG_NO_COMM, MERAK_COMM_PEER
    from synth import CONFIGS
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    group = dist.group.WORLD
    res = {}
    for name in CONFIGS_T8:
        cfg = CONFIGS[name]
        for n in (1, 2, 4):
            if cfg.microbatch % n:
                continue
            layer, o, timed = run_layers(cfg, world, rank, n, MERAK_COMM_PEER, group)
            o["no_comm_ms_per_layer"] = timed(FLAG_NO_COMM)
            rows = cfg.tokens // n
            o["ar_fwd_ms"] = layer.bench_allreduce(0, rows, 10)
            o["ar_bwd_ms"] = layer.bench_allreduce(1, rows, 10)
            o["rows"] = rows
            layer.close()
            res[f"{name}/n{n}"] = o
            if rank == 0:
                print(name, n, o, file=sys.stderr, flush=True)
            torch.cuda.empty_cache()
    if rank == 0:
        print(json.dumps({"phase": "comm", "T": world, "layers": K, "res": res}))
    dist.barrier()
    dist.destroy_process_group()


def simulate(K_, Tm, Ta, n=2, direction="fwd"):
    """Two-stream FIFO model of the sub-pipelined schedule (fig:pipedtp(b); reading R15:
    per block and sub-batch, compute Tm/(2n) forward or 2Tm/(2n) backward, all-reduce Ta/(2n)).
    Written here from the paper (tools/ do not import the oracle package)."""
    c_blk = (Tm if direction == "fwd" else 2 * Tm) / (2 * n)
    a_blk = Ta / (2 * n)
    t_comp = t_comm = 0.0
    ar_done = [0.0] * n
    for _ in range(K_):
        for _blk in range(2):
            ends = []
            for j in range(n):
                t_comp = max(t_comp, ar_done[j]) + c_blk
                ends.append(t_comp)
            for j in range(n):
                t_comm = max(t_comm, ends[j]) + a_blk
                ar_done[j] = t_comm
    return max(t_comp, t_comm)


def phase_project(f_compute, f_comm):
    from synth import CONFIGS

    def load(p):
        return [json.loads(line) for line in open(p) if line.startswith("{")][-1]
    comp, comm = load(f_compute), load(f_comm)
    T4 = comm["T"]
    ratio = (2 * 7 / 8) / (2 * (T4 - 1) / T4)  # two-shot NVLink bytes per GPU, T = 8 vs T = 4
    out = {}
    for key, c8 in comp["res"].items():
        if key not in comm["res"]:
            continue
        name, n = key.split("/")
        n = int(n[1:])
        cfg = CONFIGS[name]
        c4 = comm["res"][key]
        # overlap model calibrated on T = 4: Tm = fwd compute per layer (total = 3 Tm),
        # Ta = both forward all-reduces of one layer over the microbatch = 2 n t_ar
        def model(tc, t_ar_f, t_ar_b):
            Tm, Ta_f, Ta_b = tc / 3, 2 * n * t_ar_f, 2 * n * t_ar_b
            return (simulate(K, Tm, Ta_f, n=n, direction="fwd") + simulate(K, Tm, Ta_b, n=n, direction="bwd")) / K
        exp4_meas = c4["ms_per_layer"] - c4["no_comm_ms_per_layer"]
        exp4_model = model(c4["no_comm_ms_per_layer"], c4["ar_fwd_ms"], c4["ar_bwd_ms"]) - c4["no_comm_ms_per_layer"]
        calib = exp4_meas / exp4_model if exp4_model > 1e-6 else 1.0
        t8f, t8b = c4["ar_fwd_ms"] * ratio, c4["ar_bwd_ms"] * ratio
        tc8 = c8["compute_ms_per_layer"]
        exp8 = max(0.0, (model(tc8, t8f, t8b) - tc8) * calib)
        layer8 = tc8 + exp8
        out[key] = {"label": "projected (4-GPU limit)", "T": 8, "n_sub": n,
                    "compute_ms_per_layer_measured_1gpu": tc8, "ar_fwd_ms_projected": t8f,
                    "ar_bwd_ms_projected": t8b, "exposed_ms_per_layer_projected": exp8,
                    "layer_ms_projected": layer8,
                    "tflops_per_gpu_projected": layer_flops(cfg) / 8 / (layer8 * 1e-3) / 1e12,
                    "frac_of_1644_projected": layer_flops(cfg) / 8 / (layer8 * 1e-3) / 1644e12,
                    "exposed_frac_projected": exp8 / layer8,
                    "calibration_T4": {"measured_exposed_ms": exp4_meas, "model_exposed_ms": exp4_model,
                                       "factor": calib, "ar_traffic_ratio_T8_vs_T4": ratio}}
    print(json.dumps({"phase": "project", "res": out}, indent=1))


if __name__ == "__main__":
    ph = sys.argv[1]
    if ph == "compute":
        phase_compute()
    elif ph == "comm":
        phase_comm()
    else:
        phase_project(sys.argv[2], sys.argv[3])
