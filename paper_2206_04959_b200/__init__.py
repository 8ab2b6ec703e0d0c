"""B200-native sub-pipelined tensor-model-parallel transformer layer (Merak, arXiv 2206.04959 §6.3).

The hot path lives in libmerak_tmp.so (csrc/, C ABI in include/merak_tmp.h); `binding` is the
thin ctypes layer over it.
"""
from .binding import (FLAG_CHAIN, FLAG_NO_COMM, FLAG_RECOMPUTE, KERNEL_CLASSES, sp_rows, MERAK_BF16, MERAK_COMM_INPROC, MERAK_COMM_LOCAL,
                      MERAK_COMM_NCCL, MERAK_COMM_NVLS, MERAK_COMM_PEER, MERAK_FP32_CHECK, PARAM_NAMES,
                      MerakError, TmpLayer, head_partition, lib, shard_weights, zero_grads_like)

__all__ = ["FLAG_CHAIN", "FLAG_NO_COMM", "FLAG_RECOMPUTE", "sp_rows", "KERNEL_CLASSES", "MERAK_BF16", "MERAK_COMM_INPROC", "MERAK_COMM_LOCAL", "MERAK_COMM_NCCL", "MERAK_COMM_NVLS",
           "MERAK_COMM_PEER", "MERAK_FP32_CHECK", "PARAM_NAMES",
           "MerakError", "TmpLayer", "head_partition", "lib", "shard_weights", "zero_grads_like"]
