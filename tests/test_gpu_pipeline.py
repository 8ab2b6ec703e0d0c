"""A K-layer TMP stage driven by the pipeline schedules on one GPU: the
stages of a pipeline run in-process through the C ABI in schedule order (1F1B with recomputation fused into
the backward, early recomputation, shifted critical path, no recomputation; with stage-aware recomputation
keeping some layers' activations).  Every policy gives bit-identical gradients and outputs to running the
microbatches one after another, and those match the fp64 oracle."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from synth import CONFIGS, make_activations, make_params  # noqa: E402

torch = pytest.importorskip("torch")

CFG = CONFIGS["tiny"].with_(hidden=128, heads=2, seq_len=64, microbatch=2, n_sub=2, tmp_degree=1)
S, K, M = 3, 2, 4  # stages, layers per stage, microbatches


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def build(kept):
    from paper_2206_04959_b200 import PARAM_NAMES, TmpLayer, shard_weights, zero_grads_like
    from paper_2206_04959_b200.pipeline import PipelineStage
    dev = torch.device("cuda", torch.cuda.current_device())
    stages = []
    for j in range(S):
        lay = TmpLayer(CFG.hidden, CFG.heads, CFG.seq_len, CFG.microbatch, n_sub=2, device=dev.index)
        ws = [shard_weights(make_params(CFG, layer=j * K + k), CFG.heads, 1, 0, dev) for k in range(K)]
        stages.append(PipelineStage(lay, ws, [zero_grads_like(w) for w in ws], j, S, kept=kept[j]))
    xs, dys = [], []
    for mb in range(M):
        x, dy = make_activations(CFG, step=mb)
        xs.append(torch.as_tensor(np.asarray(x).reshape(CFG.tokens, CFG.hidden)).to(dev, torch.bfloat16))
        dys.append(torch.as_tensor(np.asarray(dy).reshape(CFG.tokens, CFG.hidden)).to(dev, torch.bfloat16))
    return stages, xs, dys, PARAM_NAMES


def sequential():
    stages, xs, dys, names = build([K] * S)
    outs, dxs = {}, {}
    for mb in range(M):
        h = xs[mb]
        for st in stages:
            h = st.forward(mb, h)
        outs[mb] = h.clone()
        g = dys[mb]
        for st in reversed(stages):
            g = st.backward(mb, g)
        dxs[mb] = g
    torch.cuda.synchronize()
    res = {"y": outs, "dx": dxs, "g": [[{n: st.grads[k][n].clone() for n in names} for k in range(K)] for st in stages]}
    for st in stages:
        st.layer.close()
    return res


@pytest.fixture(scope="module")
def reference():
    return sequential()


@pytest.mark.parametrize("policy,kept", [("1f1b", [0, 0, 0]), ("early", [0, 0, 0]), ("scp", [0, 1, K]),
                                         ("none", [K, K, K]), ("scp", [1, 1, K]), ("1f1b", [1, 2, 0])])
def test_pipeline_policy_bit_identical(reference, policy, kept):
    from paper_2206_04959_b200.pipeline import run_in_process, schedule
    stages, xs, dys, names = build(kept)
    outs, dxs = {}, {}
    acts = schedule(policy, S, M)
    # keep the last stage's outputs: run_in_process drops them at the backward
    orig = stages[-1].forward

    def fwd_keep(mb, x):
        y = orig(mb, x)
        outs[mb] = y.clone()
        return y
    stages[-1].forward = fwd_keep
    _, dx0 = run_in_process(stages, acts, xs, dys)
    torch.cuda.synchronize()
    for mb in range(M):
        assert torch.equal(outs[mb], reference["y"][mb]), mb
        assert torch.equal(dx0[mb], reference["dx"][mb]), mb
    for j, st in enumerate(stages):
        for k in range(K):
            for n in names:
                assert torch.equal(st.grads[k][n], reference["g"][j][k][n]), (j, k, n)
        st.layer.close()


def test_pipeline_matches_oracle(reference):
    """The composed S*K-layer model over M microbatches (gradients summed over microbatches) vs fp64."""
    from gpu_layer_util import TOL_BF16, oracle_chain, rel_err
    params = [make_params(CFG, layer=i) for i in range(S * K)]
    gsum = None
    for mb in range(M):
        x, dy = make_activations(CFG, step=mb)
        y, dx, g = oracle_chain(params, x, dy, CFG.heads)
        assert rel_err(reference["y"][mb].float().cpu().numpy(), y.reshape(CFG.tokens, CFG.hidden)) <= TOL_BF16
        assert rel_err(reference["dx"][mb].float().cpu().numpy(), dx.reshape(CFG.tokens, CFG.hidden)) <= TOL_BF16
        gsum = g if gsum is None else [{n: a[n] + b[n] for n in a} for a, b in zip(gsum, g)]
    for i in range(S * K):
        for n, r in gsum[i].items():
            e = rel_err(reference["g"][i // K][i % K][n].cpu().numpy(), r)
            assert e <= TOL_BF16, (i, n, e)
