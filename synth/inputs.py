"""Seeded synthetic inputs for the sub-pipelined TMP layer (shared by oracle and GPU tests).

This module holds NO arithmetic of the method: it only defines the workload
shapes (BASELINE.json "configs") and draws seeded random tensors with the value
distributions stated in DESIGN.md ("Input recipe"), quantised to bf16 so both
sides consume bit-identical values (reading R11).

Every tensor is a *global* (unsharded) float32 numpy array whose values are
exactly representable in bf16.  Per-rank slicing is NOT done here: the oracle
(oracle/) and the GPU binding (paper_2206_04959_b200/) each implement their own
partition, so the two sides share nothing but these numbers.

Shapes (nn.Linear convention, [out, in]); P:557 splits a layer into an attention
block and an FFN block, P:107 / P:557-558 give the Megatron row/column split:
  x, dy         [B, s, h]
  ln1_g, ln1_b  [h]          ln2_g, ln2_b [h]
  w_qkv         [3h, h]      rows: all q heads, then all k heads, then all v heads
  b_qkv         [3h]
  w_o           [h, h]       b_o [h]
  w_1           [f, h]       b_1 [f]      (f = 4h, reading R7)
  w_2           [h, f]       b_2 [h]
"""
from __future__ import annotations

import dataclasses

import numpy as np

SEED = 220604959  # arXiv id 2206.04959

PARAM_NAMES = (
    "ln1_g", "ln1_b", "w_qkv", "b_qkv", "w_o", "b_o",
    "ln2_g", "ln2_b", "w_1", "b_1", "w_2", "b_2",
)


@dataclasses.dataclass(frozen=True)
class LayerConfig:
    """One GPT-shaped layer workload (BASELINE.json `configs`)."""

    name: str
    hidden: int          # h
    heads: int           # H
    seq_len: int         # s
    microbatch: int      # B
    tmp_degree: int      # T (the configuration's TMP degree)
    n_sub: int           # n sub-microbatches ("evenly split ... into two")
    ffn_mult: int = 4    # f = 4h

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    @property
    def ffn(self) -> int:
        return self.ffn_mult * self.hidden

    @property
    def tokens(self) -> int:
        return self.microbatch * self.seq_len

    def with_(self, **kw) -> "LayerConfig":
        return dataclasses.replace(self, **kw)


CONFIGS = {
    # BASELINE.json configs[0..4]
    "tiny": LayerConfig("tiny", 64, 2, 16, 2, 2, 2),
    "gpt1.5b": LayerConfig("gpt1.5b", 1600, 25, 1024, 8, 2, 2),
    "gpt2.5b": LayerConfig("gpt2.5b", 2560, 32, 1024, 8, 4, 2),
    "gpt8.3b": LayerConfig("gpt8.3b", 3072, 32, 1024, 8, 8, 2),
    "gpt20b": LayerConfig("gpt20b", 6144, 64, 2048, 4, 8, 2),
}


def round_to_bf16(a: np.ndarray) -> np.ndarray:
    """Round to the nearest bf16 value (ties to even), returned as float32.

    Input quantisation only (reading R11): values go fp64/fp32 -> fp32 -> bf16.
    """
    f = np.ascontiguousarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).reshape(f.shape)


def _rng(index: int, seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=seed + index))


def _normal(index, shape, std, seed):
    a = _rng(index, seed).standard_normal(size=shape, dtype=np.float32)
    if std != 1.0:
        a *= np.float32(std)
    return round_to_bf16(a)


def _uniform(index, shape, lo, hi, seed):
    a = _rng(index, seed).uniform(lo, hi, size=shape).astype(np.float32)
    return round_to_bf16(a)


def make_params(cfg: LayerConfig, seed: int = SEED, layer: int = 0) -> dict:
    """Global layer parameters. W ~ N(0, 0.02^2) (GPT-2 init), biases N(0, 0.02^2)
    (non-zero so every bias path is exercised), gamma ~ U(0.5, 1.5), beta ~ N(0, 0.1^2)."""
    h, f = cfg.hidden, cfg.ffn
    base = 100 * (layer + 1)
    s = seed
    return {
        "ln1_g": _uniform(base + 0, (h,), 0.5, 1.5, s),
        "ln1_b": _normal(base + 1, (h,), 0.1, s),
        "w_qkv": _normal(base + 2, (3 * h, h), 0.02, s),
        "b_qkv": _normal(base + 3, (3 * h,), 0.02, s),
        "w_o": _normal(base + 4, (h, h), 0.02, s),
        "b_o": _normal(base + 5, (h,), 0.02, s),
        "ln2_g": _uniform(base + 6, (h,), 0.5, 1.5, s),
        "ln2_b": _normal(base + 7, (h,), 0.1, s),
        "w_1": _normal(base + 8, (f, h), 0.02, s),
        "b_1": _normal(base + 9, (f,), 0.02, s),
        "w_2": _normal(base + 10, (h, f), 0.02, s),
        "b_2": _normal(base + 11, (h,), 0.02, s),
    }


def make_activations(cfg: LayerConfig, seed: int = SEED, step: int = 0) -> tuple:
    """x ~ N(0,1) (post-embedding residual stream) and dy ~ N(0,1) (loss cotangent)."""
    shape = (cfg.microbatch, cfg.seq_len, cfg.hidden)
    x = _normal(10 + 2 * step, shape, 1.0, seed)
    dy = _normal(11 + 2 * step, shape, 1.0, seed)
    return x, dy


def make_all(cfg: LayerConfig, seed: int = SEED) -> tuple:
    """(params, x, dy) for one layer."""
    x, dy = make_activations(cfg, seed)
    return make_params(cfg, seed), x, dy


def make_params_torch(cfg: LayerConfig, device, seed: int = SEED, layer: int = 0) -> dict:
    """Same shapes and value distributions as make_params, drawn with torch's
    seeded device generator and RNE-rounded to bf16 on the device: used by bench.py, whose full-size
    weights (0.9 GB per gpt20b layer) numpy's Philox would take ~20 s per layer to draw.  The values are
    NOT those of make_params (different generator); parity tests use make_params."""
    import torch

    h, f = cfg.hidden, cfg.ffn
    base = 100 * (layer + 1)
    gen = torch.Generator(device=device)

    def normal(idx, shape, std):
        gen.manual_seed(seed + base + idx)
        return (torch.randn(shape, generator=gen, device=device) * std).to(torch.bfloat16)

    def uniform(idx, shape, lo, hi):
        gen.manual_seed(seed + base + idx)
        return (torch.rand(shape, generator=gen, device=device) * (hi - lo) + lo).to(torch.bfloat16)

    return {
        "ln1_g": uniform(0, (h,), 0.5, 1.5), "ln1_b": normal(1, (h,), 0.1),
        "w_qkv": normal(2, (3 * h, h), 0.02), "b_qkv": normal(3, (3 * h,), 0.02),
        "w_o": normal(4, (h, h), 0.02), "b_o": normal(5, (h,), 0.02),
        "ln2_g": uniform(6, (h,), 0.5, 1.5), "ln2_b": normal(7, (h,), 0.1),
        "w_1": normal(8, (f, h), 0.02), "b_1": normal(9, (f,), 0.02),
        "w_2": normal(10, (h, f), 0.02), "b_2": normal(11, (h,), 0.02),
    }


def make_activations_torch(cfg: LayerConfig, device, seed: int = SEED) -> tuple:
    """x, dy ~ N(0, 1) as [B*s, h] bf16 device tensors (bench.py; see make_params_torch)."""
    import torch

    gen = torch.Generator(device=device)
    out = []
    for idx in (10, 11):
        gen.manual_seed(seed + idx)
        out.append(torch.randn((cfg.tokens, cfg.hidden), generator=gen, device=device).to(torch.bfloat16))
    return tuple(out)
