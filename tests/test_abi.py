"""CPU checks of the boundary: libmerak_tmp.so loads, exports every symbol include/*.h declares, and
config validation returns the documented status codes without touching a GPU."""
import ctypes
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2206_04959_b200", "libmerak_tmp.so")


def declared_functions():
    names = set()
    for hdr in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(hdr).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b((?:merak)_\w+)\s*\(", src))
    return sorted(n for n in names if not n.endswith("_fn"))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        import __graft_entry__
        __graft_entry__.build()
    from paper_2206_04959_b200.binding import lib as load
    return load()


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 18, names
    for n in names:
        assert hasattr(lib, n), n


def _cfg(**kw):
    from paper_2206_04959_b200.binding import Config
    base = dict(hidden=64, heads=2, seq_len=16, microbatch=2, tmp_degree=1, tmp_rank=0, n_sub=2, ffn_hidden=0,
                ln_eps=1e-5, precision=0, comm=0, comm_ctas=0, device=0)
    base.update(kw)
    return Config(**base)


@pytest.mark.parametrize("kw,status", [
    (dict(hidden=0), -1), (dict(tmp_rank=3, tmp_degree=2), -1), (dict(precision=7), -1),
    (dict(microbatch=3, n_sub=2), -2), (dict(hidden=66, heads=4), -2), (dict(heads=2, tmp_degree=4), -2),
    (dict(hidden=48, heads=1), -3), (dict(hidden=60, heads=2, seq_len=16), -3), (dict(tmp_degree=3, heads=3, hidden=96), -3),
    (dict(seq_len=6, microbatch=2, n_sub=2), -3),
])
def test_validation_status_codes(lib, kw, status):
    from paper_2206_04959_b200.binding import ALLGATHER_FN
    h = ctypes.c_void_p()
    c = _cfg(**kw)
    st = lib.merak_tmp_init(ctypes.byref(c), ALLGATHER_FN(0), None, ctypes.byref(h))
    assert st == status, (kw, st, lib.merak_tmp_last_error(None))
    assert lib.merak_tmp_last_error(None)
    assert not h.value


def test_null_handle_calls(lib):
    assert lib.merak_tmp_set_subbatches(None, 2) == -1
    assert lib.merak_tmp_saved_bytes(None) == 0
    assert lib.merak_tmp_destroy(None) == 0
    assert lib.merak_tmp_launch_count(None) == 0
    assert lib.merak_tmp_join(None, None) == -1


def test_null_handle_measurement_hooks(lib):
    """The measurement / diagnostics hooks reject a NULL handle without touching the device."""
    i32 = ctypes.c_int32
    out = (i32 * 21)()
    assert lib.merak_tmp_debug_state(None, out) == -1
    assert lib.merak_tmp_debug_host(None, out) == -1
    t = ctypes.c_float()
    assert lib.merak_tmp_bench_allreduce(None, 0, 16, 1, ctypes.byref(t)) == -1
    n = i32()
    assert lib.merak_tmp_get_timeline(None, 0, ctypes.byref(n), None, None, None, None) == -1
    assert lib.merak_tmp_set_profiling(None, 1) == -1
    assert lib.merak_tmp_get_profile(None, None, None, None) == -1


@pytest.mark.parametrize("kw,status", [
    (dict(hidden=0), -1), (dict(microbatch=3, n_sub=2), -2), (dict(heads=2, tmp_degree=4), -2),
    (dict(hidden=96, heads=2), -3), (dict(comm=1, tmp_degree=2), -3), (dict(comm=2, tmp_degree=2), -3),
])
def test_init_group_validation(lib, kw, status):
    """merak_tmp_init_group (in-process TMP group) validates like merak_tmp_init and leaves no handle."""
    T = kw.get("tmp_degree", 2)
    kw = dict(kw, tmp_degree=T)
    hs = (ctypes.c_void_p * T)()
    st = lib.merak_tmp_init_group(ctypes.byref(_cfg(**kw)), hs)
    assert st == status, (kw, st, lib.merak_tmp_last_error(None))
    assert all(not v for v in hs)


def test_init_rejects_inproc_comm(lib):
    """MERAK_COMM_INPROC handles come only from merak_tmp_init_group."""
    from paper_2206_04959_b200.binding import ALLGATHER_FN
    h = ctypes.c_void_p()
    st = lib.merak_tmp_init(ctypes.byref(_cfg(comm=3, tmp_degree=2)), ALLGATHER_FN(0), None, ctypes.byref(h))
    assert st == -1 and not h.value
