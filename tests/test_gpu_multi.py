"""Multi-GPU parity (GPU, >= 2 devices): torchrun the worker at T = 2 (and 4 when available)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _run(T, port, extra_env=None):
    env = dict(os.environ)
    env.update(extra_env or {})
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={T}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(HERE, "mp_worker.py")]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    print(p.stdout[-6000:])
    print(p.stderr[-4000:])
    return p.returncode


@pytest.mark.parametrize("T", [2, 4])
def test_tmp_layer_multi_gpu(T):
    if torch.cuda.device_count() < T:
        pytest.skip(f"needs {T} GPUs")
    full = "1" if T == 2 else "0"
    assert _run(T, 29600 + T, {"MERAK_TEST_FULL": full}) == 0
