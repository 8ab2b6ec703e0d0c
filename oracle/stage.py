"""Stage-aware recomputation (Section 6.2) -- TEST INFRASTRUCTURE ONLY (see oracle/layer.py).

Plain restatement of the paper, 1-based stage index i of s pipeline stages, in the paper's order:
  P:520  "When alpha_i percent modules of the i-th stage are not using activation recomputation, they will
          require additional memory footprint of (s-i) alpha_i M_a.  And each stage should hold that the
          total memory M_r + (s-i) alpha_i M_a is not greater than device capacity."
  P:521  equal memory across stages: M_r + (s-i) alpha_i M_a = M_r + (s-j) alpha_j M_a.
  P:522  "we tune alpha_1 by increasing it at intervals until catching an out-of-memory error.  With the
          maximum alpha_1, we calculate alpha_i for i in [2, s] ... we take the smaller one between alpha_i
          and 1 as the final alpha_i."
  P:523-526 (displayed recursion, with the shifted critical path schedule):
          alpha_i = min(1, (s-1) alpha_1 / (s-i))  for i in [2, s-1);   alpha_{s-1} = alpha_{s-2};   alpha_s = 1.
The OOM of P:522 is replaced by the memory model of P:520 checked against a capacity (the model is what
the paper says the OOM tests).  s = 1: the only stage is the last one, alpha_1 = alpha_s = 1.
"""
from __future__ import annotations


def stage_alphas(s: int, alpha1: float) -> list:
    """alpha_1..alpha_s (list index i-1) per the P:523-526 recursion."""
    if s < 1 or not (0.0 <= alpha1 <= 1.0):
        raise ValueError("s >= 1 and 0 <= alpha_1 <= 1")
    alpha = {}
    for i in range(1, s + 1):
        if i == s:
            alpha[i] = 1.0
        elif i == 1:
            alpha[i] = alpha1
        elif 2 <= i < s - 1:
            alpha[i] = min(1.0, (s - 1) * alpha1 / (s - i))
        else:  # i == s - 1
            alpha[i] = alpha[s - 2]
    return [alpha[i] for i in range(1, s + 1)]


def stage_memory(s: int, alphas: list, m_r: float, m_a: float) -> list:
    """stage i needs M_r + (s - i) alpha_i M_a."""
    return [m_r + (s - i) * alphas[i - 1] * m_a for i in range(1, s + 1)]


def tune_alpha1(s: int, step: float, capacity: float, m_r: float, m_a: float) -> float:
    """P:522 by brute force: every candidate alpha_1 in {0, step, 2 step, ...} (and 1) is tried; the largest
    whose plan fits every stage is returned (None if even alpha_1 = 0 does not fit)."""
    cands, k = [], 0
    while k * step < 1.0:
        cands.append(k * step)
        k += 1
    cands.append(1.0)
    best = None
    for a in cands:
        if all(mem <= capacity for mem in stage_memory(s, stage_alphas(s, a), m_r, m_a)):
            best = a
    return best
