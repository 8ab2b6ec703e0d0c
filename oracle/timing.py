"""The paper's analytic cost model of sub-pipelined TMP and a two-stream
FIFO simulation of the inner pipeline (fig:pipedtp(b)).

TEST INFRASTRUCTURE ONLY (see oracle/layer.py header); bench.py also uses it to
report the model's prediction next to the measured layer time.

P:573: "Let T_m and T_a denote the computation and communication overheads of
one transformer layer during forward pass.  The overheads during backward can be
represented as 2T_m and T_a.  Hence in a TMP module with K transformer layers,
one microbatch will cost a total (3T_m+2T_a)K with the default TMP approach.
We assume the attention blocks and FFN blocks own a similar load."
P:574: sub-pipelined forward 1/4 T_m + (K-1/4) max{T_m, T_a} + 1/4 T_a,
backward 1/2 T_m + (K-1/4) max{2T_m, T_a} + 1/4 T_a, total
3/4 T_m + 1/2 T_a + (K-1/4) max{3T_m, 2T_m+T_a, 2T_a}.

Reading R15: T_a covers both all-reduces of one layer in one pass
(T_a/2 per block per microbatch), so each of the n sub-microbatches spends
T_m/(2n) (forward; 2T_m/(2n) backward) computing and T_a/(2n) all-reducing per block.
"""
from __future__ import annotations


def default_cost(K, Tm, Ta):
    """Default (non-overlapped) TMP: fwd K(Tm+Ta), bwd K(2Tm+Ta), total (3Tm+2Ta)K."""
    return {"fwd": K * (Tm + Ta), "bwd": K * (2 * Tm + Ta), "total": K * (3 * Tm + 2 * Ta)}


def subpipelined_cost(K, Tm, Ta):
    """Sub-pipelined TMP with two sub-microbatches."""
    fwd = 0.25 * Tm + (K - 0.25) * max(Tm, Ta) + 0.25 * Ta
    bwd = 0.5 * Tm + (K - 0.25) * max(2 * Tm, Ta) + 0.25 * Ta
    total = 0.75 * Tm + 0.5 * Ta + (K - 0.25) * max(3 * Tm, 2 * Tm + Ta, 2 * Ta)
    return {"fwd": fwd, "bwd": bwd, "total": total}


def simulate(K, Tm, Ta, n=2, direction="fwd", trace=None):
    """Two-stream FIFO simulation (compute stream, comm stream) of K layers x 2 blocks x n
    sub-microbatches.  Compute order: for each layer, block 0 for j = 0..n-1, then block 1
    for j = 0..n-1 (fig:pipedtp(b)); comm order identical.  Dependencies: AR(l,blk,j) after
    compute(l,blk,j); compute(l,blk,j) after AR of the previous block of sub-batch j
    (across layers too: "overlapped across transformer layers").
    Returns the makespan; appends (stream, l, blk, j, start, end) to `trace` if given."""
    c_blk = (Tm if direction == "fwd" else 2 * Tm) / (2 * n)
    a_blk = Ta / (2 * n)
    t_comp = 0.0
    t_comm = 0.0
    ar_done = [0.0] * n  # completion time of sub-batch j's latest all-reduce
    for layer in range(K):
        for blk in range(2):
            comp_end = []
            for j in range(n):
                start = max(t_comp, ar_done[j])
                t_comp = start + c_blk
                comp_end.append(t_comp)
                if trace is not None:
                    trace.append(("comp", layer, blk, j, start, t_comp))
            for j in range(n):
                start = max(t_comm, comp_end[j])
                t_comm = start + a_blk
                ar_done[j] = t_comm
                if trace is not None:
                    trace.append(("comm", layer, blk, j, start, t_comm))
    return max(t_comp, t_comm)
