"""A K-layer TMP stage driven by a pipeline schedule: the stage executor.

The action lists come from the C planner (merak_pipeline_schedule, csrc/schedule.cu); this module only
marshals them and issues the layer calls through the C ABI (merak_tmp_layer_fwd / _bwd with MERAK_FLAG_CHAIN
and MERAK_FLAG_RECOMPUTE) plus the point-to-point transfers between stages (torch.distributed over NCCL:
one communicator per direction, so an activation send and a gradient send between the same two stages never
queue behind each other).

Per stage j of s, K layers with their own weights, m microbatches of B samples:
  F(mb)  forward through the K layers; every layer's input is kept (one [B*s, h] tensor per layer); the layers
         that keep their activations (stage-aware recomputation: the first `kept` layers) keep
         their `saved` buffer, the others write a per-microbatch scratch that is then free;
  R(mb)  layer_fwd with MERAK_FLAG_RECOMPUTE for every recomputed layer into a recompute buffer set
         (early recomputation);
  B(mb)  backward through the K layers (reverse order) on the kept / recomputed activations;
  BR(mb) backward with MERAK_FLAG_RECOMPUTE on the recomputed layers (recomputation fused into the
         backward, Fig. 5a).
Gradients accumulate over the microbatches (fp32, +=) in microbatch order, so the result is bit-identical
to running the microbatches one after another.
"""
from __future__ import annotations

import ctypes

import torch

from .binding import FLAG_CHAIN, FLAG_RECOMPUTE, MerakError, lib

POLICIES = {"1f1b": 0, "early": 1, "scp": 2, "none": 3}
KINDS = {0: "F", 1: "R", 2: "B", 3: "BR"}


def schedule(policy: str, stages: int, microbatches: int) -> list:
    """Per-stage ordered action lists [(kind, mb), ...] from merak_pipeline_schedule."""
    L = lib()
    if not getattr(L, "_pipe_types", False):
        L.merak_pipeline_schedule.argtypes = [ctypes.c_int32] * 3 + [ctypes.POINTER(ctypes.c_int32), ctypes.c_int32,
                                                                      ctypes.POINTER(ctypes.c_int32)]
        L._pipe_types = True
    cap = 3 * microbatches
    acts = (ctypes.c_int32 * (stages * cap))()
    cnt = (ctypes.c_int32 * stages)()
    st = L.merak_pipeline_schedule(POLICIES[policy], stages, microbatches, acts, cap, cnt)
    if st != 0:
        raise MerakError(st, f"merak_pipeline_schedule({policy}, s={stages}, m={microbatches})")
    return [[(KINDS[acts[j * cap + k] >> 24], acts[j * cap + k] & 0xFFFFFF) for k in range(cnt[j])]
            for j in range(stages)]


class PipelineStage:
    """Stage `stage` of `stages`: K layers (weights `ws`, fp32 grads `grads`) on one TmpLayer handle."""

    def __init__(self, layer, ws, grads, stage: int, stages: int, kept: int = None):
        self.layer, self.ws, self.grads = layer, ws, grads
        self.K = len(ws)
        self.j, self.s = stage, stages
        self.kept = self.K if kept is None else kept  # layers 0..kept-1 keep their activations
        self.xin = {}        # mb -> list of K layer inputs
        self.saved = {}      # mb -> list of K saved buffers (None where recomputed)
        self.rbuf = {}       # mb -> K recompute buffers (R done)
        self.out = {}        # mb -> stage output (last layer's y)
        self.dxin = {}       # mb -> gradient w.r.t. the stage input
        self._pool = []      # free saved buffers
        self._rpool = []     # free recompute buffer sets

    def _buf(self):
        return self._pool.pop() if self._pool else self.layer.new_saved()

    def forward(self, mb, x):
        lay, K = self.layer, self.K
        xs, sv = [], []
        scratch = None
        h = x
        for k in range(K):
            xs.append(h)
            if k < self.kept:
                b = self._buf()
                sv.append(b)
            else:
                if scratch is None:
                    scratch = self._buf()
                b = scratch
                sv.append(None)
            y = torch.empty_like(h)
            # chained inside the stage; the last layer joins the caller stream (its output leaves the stage)
            lay.forward(self.ws[k], h, y, b, flags=FLAG_CHAIN if k < K - 1 else 0)
            h = y
        if scratch is not None:
            self._pool.append(scratch)  # stream-ordered: the next user runs after this forward
        self.xin[mb], self.saved[mb], self.out[mb] = xs, sv, h
        return h

    def recompute(self, mb):
        bufs = self._rpool.pop() if self._rpool else [self.layer.new_saved() for _ in range(self.K - self.kept)]
        for k in range(self.kept, self.K):
            self.layer.forward(self.ws[k], self.xin[mb][k], None, bufs[k - self.kept], flags=FLAG_CHAIN | FLAG_RECOMPUTE)
        self.rbuf[mb] = bufs

    def backward(self, mb, dy, fused_recompute=False):
        lay, K = self.layer, self.K
        xs, sv = self.xin.pop(mb), self.saved.pop(mb)
        rb = self.rbuf.pop(mb, None)
        tmp = None
        g = dy
        for k in reversed(range(K)):
            flags = FLAG_CHAIN if k > 0 else 0
            if sv[k] is not None:
                buf = sv[k]
            elif rb is not None:
                buf = rb[k - self.kept]
            else:  # recomputation fused into the backward (BR), or a B on a stage that recomputes
                if tmp is None:
                    tmp = self._buf()
                buf = tmp
                flags |= FLAG_RECOMPUTE
            dx = torch.empty_like(g)
            lay.backward(self.ws[k], xs[k], buf, g, dx, self.grads[k], flags=flags)
            g = dx
        for b in sv:
            if b is not None:
                self._pool.append(b)
        if tmp is not None:
            self._pool.append(tmp)
        if rb is not None:
            self._rpool.append(rb)
        self.out.pop(mb, None)
        self.dxin[mb] = g
        return g


def run_in_process(stages, actions, xs, dys):
    """Single-process emulation of a pipeline (one GPU): `stages` = PipelineStage list, `actions` = the
    schedule, xs[mb] = stage-0 inputs, dys[mb] = last-stage output gradients.  Actions run in a
    dependency-respecting order (round robin over the stages, each stage taking its next action once its
    input exists).  Returns (outputs of the last stage per mb, input gradients of stage 0 per mb)."""
    s = len(stages)
    nxt = [0] * s
    left = sum(len(a) for a in actions)
    while left:
        moved = False
        for j in range(s):
            if nxt[j] == len(actions[j]):
                continue
            kind, mb = actions[j][nxt[j]]
            st = stages[j]
            if kind == "F":
                if j > 0 and mb not in stages[j - 1].out:
                    continue
                st.forward(mb, xs[mb] if j == 0 else stages[j - 1].out[mb])
            elif kind == "R":
                st.recompute(mb)
            else:
                if j < s - 1 and mb not in stages[j + 1].dxin:
                    continue
                st.backward(mb, dys[mb] if j == s - 1 else stages[j + 1].dxin.pop(mb), fused_recompute=kind == "BR")
            nxt[j] += 1
            left -= 1
            moved = True
        if not moved:
            raise RuntimeError("pipeline schedule deadlocked")
    outs = {mb: stages[-1].out.get(mb) for mb in range(len(xs))}
    return outs, dict(stages[0].dxin)


def run_distributed(stage, actions_j, xs, dys, fwd_group, bwd_group, shape, dtype, device):
    """This process's stage of a multi-GPU pipeline: stage j = rank j of the groups.  Activations travel
    j -> j+1 on fwd_group, gradients j+1 -> j on bwd_group (NCCL point-to-point).  xs / dys are used on the
    first / last stage only."""
    import torch.distributed as dist
    j, s = stage.j, stage.s
    pending = []
    for kind, mb in actions_j:
        if kind == "F":
            if j == 0:
                x = xs[mb]
            else:
                x = torch.empty(shape, dtype=dtype, device=device)
                dist.irecv(x, src=j - 1, group=fwd_group).wait()
            y = stage.forward(mb, x)
            if j < s - 1:
                pending.append(dist.isend(y, dst=j + 1, group=fwd_group))
        elif kind == "R":
            stage.recompute(mb)
        else:
            if j == s - 1:
                g = dys[mb]
            else:
                g = torch.empty(shape, dtype=dtype, device=device)
                dist.irecv(g, src=j + 1, group=bwd_group).wait()
            dx = stage.backward(mb, g, fused_recompute=kind == "BR")
            stage.dxin.pop(mb, None)
            if j > 0:
                pending.append(dist.isend(dx, dst=j - 1, group=bwd_group))
        if len(pending) > 8:
            pending.pop(0).wait()
    for p in pending:
        p.wait()
