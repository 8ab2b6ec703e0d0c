"""Thin ctypes binding of libmerak_tmp.so (include/merak_tmp.h) -- argument marshalling only.

Every step of the layer runs in the CUDA library; this module only turns torch tensors into
device pointers / streams and implements the init-time all-gather callback with
torch.distributed.  There is no CPU or PyTorch fallback: if the library is missing the
import fails loudly.
"""
from __future__ import annotations

import ctypes
import os

import torch

# MERAK_LIB: an alternative in-tree build of the same library (A/B measurements only)
LIB_PATH = os.environ.get("MERAK_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmerak_tmp.so")

MERAK_OK, MERAK_EINVAL, MERAK_EINDIVISIBLE, MERAK_EUNSUPPORTED = 0, -1, -2, -3
MERAK_ECUDA, MERAK_EPEER, MERAK_ENOMEM, MERAK_ETIMEOUT, MERAK_ESTATE = -4, -5, -6, -7, -8
STATUS_NAMES = {0: "OK", -1: "EINVAL", -2: "EINDIVISIBLE", -3: "EUNSUPPORTED", -4: "ECUDA", -5: "EPEER",
                -6: "ENOMEM", -7: "ETIMEOUT", -8: "ESTATE"}
MERAK_BF16, MERAK_FP32_CHECK = 0, 1
MERAK_COMM_PEER, MERAK_COMM_NCCL, MERAK_COMM_LOCAL, MERAK_COMM_INPROC, MERAK_COMM_NVLS = 0, 1, 2, 3, 4
FLAG_CHAIN, FLAG_NO_COMM, FLAG_RECOMPUTE = 1, 2, 4
KERNEL_CLASSES = ("gemm", "attn_fwd", "attn_bwd", "layernorm", "allreduce", "reduce")
PARAM_NAMES = ("ln1_g", "ln1_b", "w_qkv", "b_qkv", "w_o", "b_o", "ln2_g", "ln2_b", "w_1", "b_1", "w_2", "b_2")


class MerakError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"merak_tmp {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Config(ctypes.Structure):
    _fields_ = [("hidden", ctypes.c_int32), ("heads", ctypes.c_int32), ("seq_len", ctypes.c_int32),
                ("microbatch", ctypes.c_int32), ("tmp_degree", ctypes.c_int32), ("tmp_rank", ctypes.c_int32),
                ("n_sub", ctypes.c_int32), ("ffn_hidden", ctypes.c_int32), ("ln_eps", ctypes.c_float),
                ("precision", ctypes.c_int32), ("comm", ctypes.c_int32), ("comm_ctas", ctypes.c_int32),
                ("device", ctypes.c_int32), ("seq_parallel", ctypes.c_int32)]


class Weights(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in PARAM_NAMES]


class Grads(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in PARAM_NAMES]


ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t)

_lib = None


def lib():
    """Load libmerak_tmp.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        P, I32, U32, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint32, ctypes.c_size_t
        L.merak_tmp_init.argtypes = [ctypes.POINTER(Config), ALLGATHER_FN, P, ctypes.POINTER(P)]
        L.merak_tmp_init_group.argtypes = [ctypes.POINTER(Config), ctypes.POINTER(P)]
        L.merak_tmp_init_group.restype = ctypes.c_int
        L.merak_tmp_set_subbatches.argtypes = [P, I32]
        L.merak_tmp_saved_bytes.argtypes = [P]
        L.merak_tmp_saved_bytes.restype = SZ
        L.merak_tmp_layer_fwd.argtypes = [P, ctypes.POINTER(Weights), P, P, P, U32, P]
        L.merak_tmp_layer_bwd.argtypes = [P, ctypes.POINTER(Weights), P, P, P, P, ctypes.POINTER(Grads), U32, P]
        L.merak_tmp_join.argtypes = [P, P]
        L.merak_tmp_destroy.argtypes = [P]
        L.merak_tmp_last_error.argtypes = [P]
        L.merak_tmp_last_error.restype = ctypes.c_char_p
        L.merak_tmp_set_profiling.argtypes = [P, I32]
        L.merak_tmp_get_profile.argtypes = [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64),
                                            ctypes.POINTER(ctypes.c_double)]
        L.merak_tmp_get_timeline.argtypes = [P, I32, ctypes.POINTER(I32), ctypes.POINTER(I32), ctypes.POINTER(I32),
                                             ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float)]
        L.merak_tmp_get_timeline.restype = ctypes.c_int
        L.merak_tmp_launch_count.argtypes = [P]
        L.merak_tmp_launch_count.restype = ctypes.c_int64
        L.merak_tmp_bench_allreduce.argtypes = [P, I32, I32, I32, ctypes.POINTER(ctypes.c_float)]
        L.merak_tmp_bench_allreduce.restype = ctypes.c_int
        L.merak_tmp_debug_state.argtypes = [P, ctypes.POINTER(I32)]
        L.merak_tmp_debug_state.restype = ctypes.c_int
        L.merak_tmp_debug_host.argtypes = [P, ctypes.POINTER(I32)]
        L.merak_tmp_debug_host.restype = ctypes.c_int
        for fn in ("merak_tmp_init", "merak_tmp_set_subbatches", "merak_tmp_layer_fwd", "merak_tmp_layer_bwd",
                   "merak_tmp_join", "merak_tmp_destroy", "merak_tmp_set_profiling", "merak_tmp_get_profile"):
            getattr(L, fn).restype = ctypes.c_int
        L.merak_test_gemm.argtypes = [P, P] + [ctypes.c_int] * 8 + [P, ctypes.c_int, P, ctypes.c_int, P, P,
                                                                      ctypes.c_int, P, ctypes.c_int, P, ctypes.c_int,
                                                                      P]
        L.merak_test_attn_fwd.argtypes = [P, P, P] + [ctypes.c_int] * 4 + [P]
        L.merak_test_attn_bwd.argtypes = [P, P, P, P, P, P] + [ctypes.c_int] * 4 + [P]
        L.merak_test_attn_bwd_ws_bytes.argtypes = [ctypes.c_int] * 4
        L.merak_test_attn_bwd_ws_bytes.restype = ctypes.c_size_t
        L.merak_test_ln_fwd.argtypes = [P, P, P, P, P, P, ctypes.c_int, ctypes.c_int, ctypes.c_float, P]
        L.merak_test_ar_fwd.argtypes = [ctypes.POINTER(P), ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P,
                                        ctypes.c_int, P, P, P, P, P, ctypes.c_float, ctypes.c_int, P]
        L.merak_test_ar_bwd.argtypes = [ctypes.POINTER(P), ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P,
                                        P, P, P, P, P, P, P, P, ctypes.c_int, P]
        L.merak_test_colsum.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P]
        _lib = L
    return _lib


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def head_partition(H: int, T: int):
    """Reading R8: rank r owns H // T + (r < H % T) whole heads, contiguous."""
    out, start = [], 0
    for r in range(T):
        n = H // T + (1 if r < H % T else 0)
        out.append((start, n))
        start += n
    return out


def shard_weights(params: dict, heads: int, T: int, r: int, device, dtype=torch.bfloat16) -> dict:
    """Slice global [out, in] weights into rank r's shard in the layout merak_tmp.h documents
    (w_qkv_r = [q rows; k rows; v rows] of the rank's heads; w_o, w_2 column slices; w_1, b_1 row
    slices; LN params, b_o, b_2 replicated).  Returns contiguous device tensors."""
    def t(a):
        return torch.as_tensor(a)
    h = t(params["w_o"]).shape[0]
    f = t(params["w_1"]).shape[0]
    d = h // heads
    e0, ne = head_partition(heads, T)[r]
    c0, c1 = e0 * d, (e0 + ne) * d
    fr = f // T
    wqkv, bqkv = t(params["w_qkv"]), t(params["b_qkv"])
    out = {
        "w_qkv": torch.cat([wqkv[b * h + c0:b * h + c1] for b in range(3)], 0),
        "b_qkv": torch.cat([bqkv[b * h + c0:b * h + c1] for b in range(3)], 0),
        "w_o": t(params["w_o"])[:, c0:c1],
        "w_1": t(params["w_1"])[r * fr:(r + 1) * fr],
        "b_1": t(params["b_1"])[r * fr:(r + 1) * fr],
        "w_2": t(params["w_2"])[:, r * fr:(r + 1) * fr],
    }
    for k in ("ln1_g", "ln1_b", "ln2_g", "ln2_b", "b_o", "b_2"):
        out[k] = t(params[k])
    return {k: v.to(device=device, dtype=dtype).contiguous() for k, v in out.items()}


def zero_grads_like(w: dict) -> dict:
    return {k: torch.zeros(v.shape, dtype=torch.float32, device=v.device) for k, v in w.items()}


def _make_allgather(group):
    import torch.distributed as dist

    def cb(ctx, send, recv, nbytes):
        try:
            world = dist.get_world_size(group)
            dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
            src = (ctypes.c_uint8 * nbytes).from_address(send)
            inp = torch.frombuffer(bytearray(bytes(src)), dtype=torch.uint8).to(dev)
            out = torch.empty(world * nbytes, dtype=torch.uint8, device=dev)
            dist.all_gather_into_tensor(out, inp, group=group)
            data = out.cpu().numpy().tobytes()
            ctypes.memmove(recv, data, len(data))
            return 0
        except Exception as e:  # never raise through C
            print(f"merak allgather failed: {e!r}", flush=True)
            return 1

    return cb


def sp_rows(tokens: int, n_sub: int, T: int, r: int):
    """Global token indices of rank r's shard in the sequence-parallel layout (merak_tmp.h): for every
    sub-batch j of m = tokens / n_sub tokens, tokens [j*m + r*m/T, j*m + (r+1)*m/T), in that order."""
    m = tokens // n_sub
    mr = m // T
    return torch.cat([torch.arange(j * m + r * mr, j * m + (r + 1) * mr) for j in range(n_sub)])


class TmpLayer:
    """One rank's handle of the sub-pipelined TMP transformer layer (merak_tmp_t).

    forward / backward are asynchronous on `stream` (default: torch's current stream)."""

    def __init__(self, hidden, heads, seq_len, microbatch, tmp_degree=1, tmp_rank=0, n_sub=2, ffn_hidden=0,
                 ln_eps=1e-5, comm=MERAK_COMM_PEER, comm_ctas=0, device=None, group=None,
                 precision=MERAK_BF16, seq_parallel=False):
        L = lib()
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self.cfg = Config(hidden, heads, seq_len, microbatch, tmp_degree, tmp_rank, n_sub, ffn_hidden, ln_eps,
                          precision, comm, comm_ctas, self.device.index or 0, int(bool(seq_parallel)))
        self._cb = ALLGATHER_FN(_make_allgather(group)) if tmp_degree > 1 and comm != MERAK_COMM_LOCAL else ALLGATHER_FN(0)
        h = ctypes.c_void_p()
        st = L.merak_tmp_init(ctypes.byref(self.cfg), self._cb, None, ctypes.byref(h))
        if st != MERAK_OK:
            raise MerakError(st, L.merak_tmp_last_error(None).decode())
        self.h = h

    @classmethod
    def group(cls, hidden, heads, seq_len, microbatch, tmp_degree, n_sub=2, ffn_hidden=0, ln_eps=1e-5, comm_ctas=0,
              device=None, precision=MERAK_BF16, seq_parallel=False):
        """All T ranks of a TMP group as handles of this process on ONE device (merak_tmp_init_group,
        MERAK_COMM_INPROC): rank r's all-reduces read the other ranks' partials straight from their slots.
        Returns [rank 0, ..., rank T-1].  Issue every layer call on every rank, from one thread, in any rank
        order: the library defers each rank's call until all T ranks made it, then issues them together
        (merak_tmp.h, MERAK_COMM_INPROC); the layer calls never block the host."""
        L = lib()
        if device is None:
            device = torch.cuda.current_device()
        dev = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        cfg = Config(hidden, heads, seq_len, microbatch, tmp_degree, 0, n_sub, ffn_hidden, ln_eps, precision,
                     MERAK_COMM_INPROC, comm_ctas, dev.index or 0, int(bool(seq_parallel)))
        hs = (ctypes.c_void_p * tmp_degree)()
        st = L.merak_tmp_init_group(ctypes.byref(cfg), hs)
        if st != MERAK_OK:
            raise MerakError(st, L.merak_tmp_last_error(None).decode())
        out = []
        for r in range(tmp_degree):
            o = cls.__new__(cls)
            o.device = dev
            o.cfg = Config(hidden, heads, seq_len, microbatch, tmp_degree, r, n_sub, ffn_hidden, ln_eps, precision,
                           MERAK_COMM_INPROC, comm_ctas, dev.index or 0, int(bool(seq_parallel)))
            o._cb = ALLGATHER_FN(0)
            o.h = ctypes.c_void_p(hs[r])
            out.append(o)
        return out

    # -- helpers
    def _check(self, st):
        if st != MERAK_OK:
            raise MerakError(st, lib().merak_tmp_last_error(self.h).decode())

    @staticmethod
    def _weights(w):
        return Weights(*[w[n].data_ptr() for n in PARAM_NAMES])

    @staticmethod
    def _grads(g):
        return Grads(*[g[n].data_ptr() for n in PARAM_NAMES])

    # -- API
    @property
    def n_sub(self):
        return self.cfg.n_sub

    def saved_bytes(self) -> int:
        return lib().merak_tmp_saved_bytes(self.h)

    def new_saved(self):
        return torch.empty(self.saved_bytes(), dtype=torch.uint8, device=self.device)

    def set_subbatches(self, n):
        self._check(lib().merak_tmp_set_subbatches(self.h, n))
        self.cfg.n_sub = n

    def forward(self, w, x, y, saved, flags=0, stream=None):
        self._w = self._weights(w)
        self._check(lib().merak_tmp_layer_fwd(self.h, ctypes.byref(self._w), _ptr(x), _ptr(y), _ptr(saved), flags,
                                              _stream(stream)))

    def backward(self, w, x, saved, dy, dx, grads, flags=0, stream=None):
        self._w = self._weights(w)
        self._g = self._grads(grads)
        self._check(lib().merak_tmp_layer_bwd(self.h, ctypes.byref(self._w), _ptr(x), _ptr(saved), _ptr(dy), _ptr(dx),
                                              ctypes.byref(self._g), flags, _stream(stream)))

    def join(self, stream=None):
        self._check(lib().merak_tmp_join(self.h, _stream(stream)))

    def set_profiling(self, on: bool):
        self._check(lib().merak_tmp_set_profiling(self.h, 1 if on else 0))

    def get_profile(self) -> dict:
        n = len(KERNEL_CLASSES)
        ms, la, fl = (ctypes.c_double * n)(), (ctypes.c_int64 * n)(), (ctypes.c_double * n)()
        self._check(lib().merak_tmp_get_profile(self.h, ms, la, fl))
        return {k: {"ms": ms[i], "launches": la[i], "flops": fl[i]} for i, k in enumerate(KERNEL_CLASSES)}

    def get_timeline(self, cap=100000) -> list:
        """[(class, stream, t0_ms, t1_ms)] of every launch since set_profiling(True); call before get_profile."""
        n = ctypes.c_int32()
        cls, st = (ctypes.c_int32 * cap)(), (ctypes.c_int32 * cap)()
        t0, t1 = (ctypes.c_float * cap)(), (ctypes.c_float * cap)()
        self._check(lib().merak_tmp_get_timeline(self.h, cap, ctypes.byref(n), cls, st, t0, t1))
        names = {0: "comp", 1: "comm", 2: "wgrad"}  # compute streams, communication stream, wgrad filler stream
        return [(KERNEL_CLASSES[cls[i]], names.get(st[i], "comp"), t0[i], t1[i]) for i in range(n.value)]

    def bench_allreduce(self, which: int, rows: int, iters: int = 20) -> float:
        """Mean device ms of one all-reduce of rows x h (collective: every rank must call it)."""
        t = ctypes.c_float()
        self._check(lib().merak_tmp_bench_allreduce(self.h, which, rows, iters, ctypes.byref(t)))
        return t.value

    def debug_state(self) -> dict:
        """Non-blocking: which internal streams still have work, and the watchdog error word."""
        o = (ctypes.c_int32 * 21)()
        lib().merak_tmp_debug_state(self.h, o)
        names = ("cs", "cs1", "cw", "cr", "ms")
        return {"busy": {k: o[i] for i, k in enumerate(names)}, "err": list(o[5:10]), "epoch": o[10],
                "first_unfinished": {k: (KERNEL_CLASSES[o[11 + i]] if 0 <= o[11 + i] < len(KERNEL_CLASSES) else None,
                                         o[16 + i]) for i, k in enumerate(names)}}

    def debug_host(self) -> dict:
        """Host-memory-only diagnostics (never blocks)."""
        o = (ctypes.c_int32 * 14)()
        lib().merak_tmp_debug_host(self.h, o)
        return {"err": list(o[0:5]), "epoch": o[5], "launches": o[6],
                "traced": dict(zip(("cs", "cs1", "cw", "cr", "ms"), list(o[7:12]))),
                "push": bool(o[12]), "two_shot": bool(o[13])}

    def launch_count(self) -> int:
        return lib().merak_tmp_launch_count(self.h)

    def close(self):
        if getattr(self, "h", None):
            h, self.h = self.h, None
            st = lib().merak_tmp_destroy(h)
            if st != MERAK_OK:
                raise MerakError(st, lib().merak_tmp_last_error(None).decode())

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
