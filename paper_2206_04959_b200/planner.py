"""ctypes wrappers of the host planners in include/merak_sched.h (argument marshalling only; the
planning arithmetic lives in csrc/schedule.cu).

Stage-aware recomputation: alpha_i per pipeline stage, alpha_1 tuned
against a memory capacity, and the number of a stage's K layers that keep their activations (the others
run with MERAK_FLAG_RECOMPUTE)."""
from __future__ import annotations

import ctypes

from .binding import MerakError, lib

_D = ctypes.c_double


def _L():
    L = lib()
    if not getattr(L, "_planner_types", False):
        L.merak_stage_alpha.argtypes = [ctypes.c_int32, _D, ctypes.POINTER(_D)]
        L.merak_tune_alpha1.argtypes = [ctypes.c_int32, _D, _D, _D, _D, ctypes.POINTER(_D)]
        L.merak_layers_kept.argtypes = [_D, ctypes.c_int32]
        L.merak_layers_kept.restype = ctypes.c_int32
        L._planner_types = True
    return L


def stage_alphas(stages: int, alpha1: float) -> list:
    out = (_D * stages)()
    st = _L().merak_stage_alpha(stages, alpha1, out)
    if st != 0:
        raise MerakError(st, "merak_stage_alpha: invalid arguments")
    return list(out)


def tune_alpha1(stages: int, step: float, capacity: float, m_r: float, m_a: float) -> float:
    a = _D(0.0)
    st = _L().merak_tune_alpha1(stages, step, capacity, m_r, m_a, ctypes.byref(a))
    if st != 0:
        raise MerakError(st, "merak_tune_alpha1: " + ("runtime memory exceeds capacity" if st == -6 else "invalid"))
    return a.value


def layers_kept(alpha: float, layers: int) -> int:
    return int(_L().merak_layers_kept(alpha, layers))


def recompute_plan(stages: int, layers: int, capacity: float, m_r: float, m_a_layer: float) -> dict:
    """Stage-aware plan for pipeline stages of `layers` layers each: M_a = layers x m_a_layer (one
    microbatch's activations of a stage), alpha_1 tuned in steps of one layer (1 / layers), then per stage
    alpha_i and the number of layers that keep activations (the rest recompute)."""
    a1 = tune_alpha1(stages, 1.0 / layers, capacity, m_r, layers * m_a_layer)
    al = stage_alphas(stages, a1)
    return {"alpha1": a1, "alphas": al, "layers_kept": [layers_kept(a, layers) for a in al]}
