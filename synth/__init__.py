"""Seeded synthetic workload generator (no method arithmetic; see inputs.py)."""
from .inputs import CONFIGS, PARAM_NAMES, SEED, LayerConfig, make_activations, make_all, make_params, round_to_bf16

__all__ = ["CONFIGS", "PARAM_NAMES", "SEED", "LayerConfig", "make_activations", "make_all", "make_params",
           "round_to_bf16"]
