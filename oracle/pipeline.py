"""Pipeline schedules of PMP stages (Section 6.1) -- TEST INFRASTRUCTURE ONLY (see oracle/layer.py).

A plain discrete-event simulation of per-stage action lists under the paper's unit costs ("the forward time
of one microbatch is T_m, the recomputation time and backward time could be estimated as T_m and 2T_m",
P:459), and the paper's bubble formulas:
  1F1B (Fig. 5a, recomputation right before each backward, after the gradient arrived):
        bubble (s-1)(T_m + T_m + 2T_m) = 4(s-1)T_m, running time 4mT_m, ratio (s-1)/m
  1F1B + early recomputation (Fig. 5b, "the activation recomputation operation does not depend on the
        output of previous stages"): bubble (s-1)(T_m + 2T_m) = 3(s-1)T_m, ratio 3(s-1)/(4m)
  shifted critical path (Fig. 5c): bubble 3(s-2)T_m, ratio 3(s-2)/(4m)
Action kinds (as in include/merak_sched.h, but restated here): 'F' forward, 'R' recompute (no dependency on
other stages), 'B' backward on existing activations, 'BR' backward with its recomputation fused in front
(starts when the gradient arrives).  F on stage j > 0 needs stage j-1's F of the same microbatch; B / BR on
stage j < s-1 needs stage j+1's backward of the same microbatch.  Communication time is 0 (as in the paper).
"""
from __future__ import annotations

COST = {"F": 1.0, "R": 1.0, "B": 2.0, "BR": 3.0}


def paper_bubble(policy: str, s: int) -> float:
    """Bubble time in units of T_m; 'none' = 1F1B without recomputation (F + 2 B)."""
    return {"1f1b": 4 * (s - 1), "early": 3 * (s - 1), "scp": 3 * (s - 2), "none": 3 * (s - 1)}[policy]


def paper_run_time(policy: str, m: int) -> float:
    return (3 if policy == "none" else 4) * m


def simulate(sched, head: float = 0.0, cost=None):
    """sched: list over stages of [(kind, mb), ...] in stage order.  Every stage runs its list in order; an
    action starts when the stage is free and its cross-stage input exists.  head: extra cost of every forward
    on the last stage (task head layers).  Returns (makespan, per-stage finish times, per-stage busy
    time, per-action (start, end) dict keyed by (kind, stage, mb)).  Raises on a deadlock."""
    cost = cost or COST
    s = len(sched)
    t = [0.0] * s
    busy = [0.0] * s
    nxt = [0] * s
    done = {}
    bwd_done = {}
    left = sum(len(a) for a in sched)
    while left:
        moved = False
        for j in range(s):
            if nxt[j] == len(sched[j]):
                continue
            kind, mb = sched[j][nxt[j]]
            ready = 0.0
            if kind == "F" and j > 0:
                if ("F", j - 1, mb) not in done:
                    continue
                ready = done[("F", j - 1, mb)][1]
            if kind in ("B", "BR") and j < s - 1:
                if (j + 1, mb) not in bwd_done:
                    continue
                ready = bwd_done[(j + 1, mb)]
            c = cost[kind] + (head if (kind == "F" and j == s - 1) else 0.0)
            start = max(t[j], ready)
            t[j] = start + c
            busy[j] += c
            done[(kind, j, mb)] = (start, t[j])
            if kind in ("B", "BR"):
                bwd_done[(j, mb)] = t[j]
            nxt[j] += 1
            left -= 1
            moved = True
        if not moved:
            raise RuntimeError("schedule deadlocks")
    return max(t), t, busy, done


def check_schedule(sched, m: int) -> list:
    """Violations of the schedule invariants: each stage runs exactly one forward and one backward (B or BR)
    per microbatch; a stage's R(mb) lies between its F(mb) and its backward of mb, at most once; a plain B
    follows an R of the same microbatch unless the stage recomputes nothing (keeps every activation)."""
    bad = []
    for j, acts in enumerate(sched):
        recomputes = any(k in ("R", "BR") for k, _ in acts)
        for mb in range(m):
            pos = {k: [i for i, a in enumerate(acts) if a == (k, mb)] for k in ("F", "R", "B", "BR")}
            if len(pos["F"]) != 1:
                bad.append((j, mb, "forward count"))
                continue
            nb = len(pos["B"]) + len(pos["BR"])
            if nb != 1:
                bad.append((j, mb, "backward count"))
                continue
            b = (pos["B"] + pos["BR"])[0]
            if b < pos["F"][0]:
                bad.append((j, mb, "backward before forward"))
            if len(pos["R"]) > 1:
                bad.append((j, mb, "two recomputes"))
            if pos["R"] and not (pos["F"][0] < pos["R"][0] < b):
                bad.append((j, mb, "recompute outside [F, B]"))
            if pos["R"] and pos["BR"]:
                bad.append((j, mb, "recomputed twice"))
            if pos["B"] and not pos["R"] and recomputes:
                bad.append((j, mb, "B without its recompute on a recomputing stage"))
    return bad
