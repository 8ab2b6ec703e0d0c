"""Host-side multi-process logic on CPU (gloo, world_size 2): the init-time all-gather callback the C
library calls to exchange CUDA IPC handles, exercised through its C function-pointer type."""
import ctypes
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2206_04959_b200.binding import ALLGATHER_FN, _make_allgather
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cb = ALLGATHER_FN(_make_allgather(dist.group.WORLD))
    nbytes = 64  # sizeof(cudaIpcMemHandle_t)
    send = (ctypes.c_uint8 * nbytes)(*[(rank * 37 + i) % 256 for i in range(nbytes)])
    recv = (ctypes.c_uint8 * (nbytes * world))()
    rc = cb(None, ctypes.addressof(send), ctypes.addressof(recv), nbytes)
    expect = [(r * 37 + i) % 256 for r in range(world) for i in range(nbytes)]
    q.put((rank, rc, list(recv) == expect))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_allgather_callback_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(rc == 0 and ok for _, rc, ok in res), res
