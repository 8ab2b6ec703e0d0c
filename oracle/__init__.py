"""CPU fp64 oracle for the sub-pipelined TMP layer -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  It shares no code with paper_2206_04959_b200/ and
imports nothing from it.  See layer.py for what it computes and the passages it follows.
"""
from .layer import (LN_EPS, causal_attention, causal_attention_backward, gelu, gelu_grad, layer_backward,
                    layer_flops, layer_forward, layer_fwd_bwd, layer_norm, layer_norm_backward)
from .sharded import head_partition, shard_params, sharded_fwd_bwd, unshard_grads
from .timing import default_cost, simulate, subpipelined_cost
