"""Seeded synthetic workload generator (no method arithmetic; see inputs.py)."""
from .inputs import (CONFIGS, PARAM_NAMES, SEED, LayerConfig, make_activations, make_activations_torch, make_all,
                     make_params, make_params_torch, round_to_bf16)

__all__ = ["CONFIGS", "PARAM_NAMES", "SEED", "LayerConfig", "make_activations", "make_activations_torch", "make_all",
           "make_params", "make_params_torch", "round_to_bf16"]
