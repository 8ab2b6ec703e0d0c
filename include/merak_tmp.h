/*
 * merak_tmp.h -- C ABI of the B200-native sub-pipelined tensor-model-parallel (TMP)
 * transformer layer (Merak, arXiv 2206.04959, Section 6.3 "Sub-pipelined TMP").
 *
 * Citations: "P:n" = PAPER.md line n.
 *   P:557  a layer = attention block + FFN block
 *   P:107  Megatron TMP: weights split along rows/columns, AllReduce after row-parallel GEMMs
 *   P:558  two AllReduces in the forward pass, two in the backward pass
 *   P:571  "evenly split each microbatch ... into two sub-microbatches, whose procedures are
 *          independent ... when one sub-microbatch is communicating, the other ... calculations"
 *   P:572  communication and computation "overlapped across transformer layers"
 *   P:576  "asynchronous communication operations and an alternate execution schedule for
 *          both forward and backward passes"
 *   P:555  problem statement: hidden size, sequence length, microbatch size
 *   P:763  TMP degree = number of GPUs
 *
 * What a call computes: one pre-LN GPT decoder layer (readings R1-R7),
 *   forward   y  = x1 + gelu(LN2(x1) W1^T + b1) W2^T + b2,  x1 = x + Attn(LN1(x)) Wo^T + bo
 *   backward  dx and += weight/bias/LN gradients for cotangent dy,
 * executed on this rank's weight shard with the four TMP all-reduces done in-kernel over
 * NVLink peer memory, the microbatch split into n_sub sub-microbatches pipelined across a
 * compute stream and a communication stream.
 *
 * Conventions
 *  - Every function returns merak_status (0 = OK); none aborts or throws across the ABI.
 *    The text of the last error is available from merak_tmp_last_error().
 *  - All device pointers are plain CUDA device pointers (16-byte aligned; 256 recommended).
 *    Host pointers appear only in merak_tmp_init (config, callback) and the query calls.
 *  - All work is enqueued asynchronously in the order of the caller's stream `st`
 *    (a cudaStream_t passed as void*; NULL = legacy default stream).  The library owns two
 *    internal streams (compute, communication); they wait on an event recorded on `st` at
 *    entry, and `st` waits on the library's final event before the call returns (unless
 *    MERAK_FLAG_CHAIN defers that join, see below).
 *  - A handle is bound to one (process, device, layer shape); it is not thread-safe.
 *
 * Tensor layouts (token-major, features contiguous; tokens = B*s, token t = b*s + i):
 *  x, y, dx, dy : [B*s, h] bf16, replicated on every rank of the TMP group.
 *  Rank r owns heads [e0_r, e0_r + H_r) with H_r = H/T + (r < H % T) (reading R8: whole
 *  heads, uneven split allowed), h_r = H_r * d, and FFN rows [r f_r, (r+1) f_r), f_r = f/T.
 *  merak_tmp_weights (bf16, this rank's shard, nn.Linear [out, in] layout):
 *    ln1_g, ln1_b, ln2_g, ln2_b, b_o, b_2 : [h] replicated
 *    w_qkv : [3 h_r, h]  rows = q rows of the rank's heads, then k rows, then v rows;
 *            head e of the rank occupies rows e*d .. e*d+d-1 inside each of the three blocks
 *    b_qkv : [3 h_r]
 *    w_o   : [h, h_r]     (row-parallel: columns of the global w_o for the rank's heads)
 *    w_1   : [f_r, h]     b_1 : [f_r]
 *    w_2   : [h, f_r]     (row-parallel)
 *  merak_tmp_grads: same shapes, fp32, ACCUMULATED (+=).  The caller zeroes them.
 *  Replicated grads (LN, b_o, b_2) come out identical on every rank.
 *  saved: caller-owned device buffer of merak_tmp_saved_bytes() bytes written by layer_fwd
 *  and read by layer_bwd; its layout does not depend on n_sub.
 *
 * Numerics (reading R10-R12): bf16 operands (RNE), fp32 accumulation and
 * statistics; each all-reduce sums bf16 partials in fp32 in fixed rank order 0..T-1, adds
 * bias and residual in fp32 and rounds once to bf16; every reduction over tokens (bias,
 * LN and weight gradients) runs in a fixed order that does not depend on n_sub, so the
 * sub-pipelined (n_sub > 1) and the non-sub-pipelined (n_sub = 1) runs are bit-identical.
 *
 * fp32 check mode (precision = MERAK_FP32_CHECK; SURVEY §8(a) "the fp32 check mode is fp32
 * everywhere", north_star tolerance 1e-5): x, y, dx, dy, every weight and the saved buffer are
 * fp32 (same shapes and layouts; merak_tmp_saved_bytes() returns the fp32 size); the all-reduces
 * sum fp32 partials in rank order without rounding.  Same sharding, sub-batch loop and token-order
 * reductions (n_sub-independent), simple FP32-pipe kernels, all on one internal stream: a
 * numerical reference for the method, not a fast path.
 */
#ifndef MERAK_TMP_H
#define MERAK_TMP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct merak_tmp merak_tmp_t; /* opaque handle */

typedef enum {
  MERAK_OK = 0,
  MERAK_EINVAL = -1,       /* NULL/misaligned pointer, non-positive size, bad enum value      */
  MERAK_EINDIVISIBLE = -2, /* B % n_sub, h % H or f % T non-zero, or H < T                    */
  MERAK_EUNSUPPORTED = -3, /* head dim not in {32,64,80,96,128}, T not in {1,2,4,8}, h > 8192, no P2P */
  MERAK_ECUDA = -4,        /* a CUDA runtime/driver call failed (message has the CUDA error)  */
  MERAK_EPEER = -5,        /* IPC handle exchange / peer mapping failed                       */
  MERAK_ENOMEM = -6,       /* device allocation failed                                        */
  MERAK_ETIMEOUT = -7,     /* the in-kernel peer handshake watchdog fired (peer hung/absent); */
                           /* reported by the next call, the handle is unusable afterwards    */
  MERAK_ESTATE = -8        /* call not allowed in the current state (e.g. open chain)         */
} merak_status;

enum { MERAK_BF16 = 0, MERAK_FP32_CHECK = 1 };      /* merak_tmp_config.precision */
/* merak_tmp_config.comm.  MERAK_COMM_LOCAL is a measurement mode: one process emulates rank
 * tmp_rank of a T-way group on its own (no peers, no callback needed); every all-reduce reads only
 * the local partial, as with MERAK_FLAG_NO_COMM.  Used to time per-rank compute of T = 8 shapes
 * on one GPU (SURVEY §8(d) "TMP=8" projection).  Results are NOT the layer's. */
/* MERAK_COMM_INPROC: the T ranks of the group are T handles of ONE process on ONE device, created
 * together by merak_tmp_init_group; every all-reduce reads the peers' partials straight from their
 * slots (same context, no CUDA IPC), with the same kernels and arithmetic as MERAK_COMM_PEER.  The
 * cross-rank handshake is an event exchange instead of the spinning handshake kernel: a rank's
 * merak_tmp_layer_fwd / _bwd call is DEFERRED (returns MERAK_OK at once, nothing issued) until every rank
 * of the group has made its matching call; the call that completes the set issues all T calls from the
 * calling thread, switching between the ranks at each handshake point, and returns the first failure of
 * the set.  Pointers passed to a deferred call must stay valid until the set completes.  A second layer
 * call on a rank before the set completes, or merak_tmp_join / set_subbatches / profiling calls on a rank
 * with a deferred call, fail with MERAK_ESTATE.  It exists so that T > 1 runs of the method (P:107
 * partial sums over T ranks, P:571 sub-batch overlap) can be checked against the oracle on a single GPU.
 * Not for throughput (the ranks share one GPU). */
/* MERAK_COMM_NVLS: as MERAK_COMM_PEER, but the all-reduce slots of the T ranks are bound to one CUDA
 * multicast object (NVLink SHARP) and the reduce-scatter phase runs in the NVSwitch:
 * rank r reads the rows it owns with multimem.ld_reduce (the switch sums the T bf16 partials with fp32
 * accumulation and returns them rounded once to bf16 -- reading R10n) and broadcasts the result
 * (plus bias and residual in the forward, rounded again) with multimem.st into every rank's slot; the fused
 * epilogue then reads every row locally.  Init exchanges the multicast handle as a POSIX descriptor
 * (pidfd_getfd: the ranks must run as the same user).  EUNSUPPORTED when a device lacks multicast support
 * or in the fp32 check mode.  Same call sequence and results (up to the switch's rounding) as PEER. */
enum { MERAK_COMM_PEER = 0, MERAK_COMM_NCCL = 1, MERAK_COMM_LOCAL = 2, MERAK_COMM_INPROC = 3, MERAK_COMM_NVLS = 4 };
/* All-reduce algorithm of MERAK_COMM_PEER / INPROC (P:558's 2+2 AllReduces per layer, in-kernel): one-shot at
 * T = 2 (every rank sums all T partials), two-shot at T >= 4 (owner rows reduced, then gathered; env
 * MERAK_AR_TWO_SHOT=0/1 at init overrides).  Fused GEMM -> reduce-scatter push (env
 * MERAK_AR_PUSH at init, default 2 at T >= 4, else 0): 1 = the row-parallel GEMMs (proj, fc2, fc1 dgrad, QKV
 * dgrad) store each 32-row output box into the slot of the rank owning those rows (TMA stores over NVLink
 * through peer tensor maps), so the reduce-scatter reads local memory only; 2 = in addition the two-shot's
 * reduced rows are pushed into every rank's all-gather slot and the fused epilogue reads locally.  Applies to
 * calls whose owner row blocks B*s/(n T) are whole 32-row boxes, with the two-shot all-reduce or the
 * sequence-parallel layout; other calls use the pull layout.  A GEMM pushes only when its compute covers its
 * NVLink transfer, K T / (T-1) >= 1400 (env MERAK_AR_PUSH_MINK; e.g. proj at T = 8 stays on pull).  Results are
 * bit-identical in every mode. */

/* flags for layer_fwd / layer_bwd */
enum {
  MERAK_FLAG_CHAIN = 1u,   /* do not join the caller stream at the end; the next merak call
                              on this handle (or merak_tmp_join) joins.  Lets layer k+1's first
                              sub-batch start while layer k's last all-reduce is in flight.
                              With MERAK_FUSE_LN1=1 in the environment at init (SURVEY §8(a)
                              F1/F8), a chained layer_fwd's AR#2s (handshakes and the epilogue
                              kernels, which write y) are issued by the next call on the handle --
                              fused with that layer's LN1 when it is a layer_fwd whose x is this y
                              -- or by merak_tmp_join / merak_tmp_destroy.  Until then y is not
                              written and the layer's weights and `saved` buffer must stay
                              unchanged; a device synchronize does not complete y, merak_tmp_join
                              does (profiling calls fail with ESTATE before it).                 */
  MERAK_FLAG_NO_COMM = 2u, /* measurement only: every all-reduce reads the local partial alone
                              (wrong result for T > 1); used to measure exposed communication.   */
  MERAK_FLAG_RECOMPUTE = 4u /* activation recomputation ("the recomputation ... could be
                              estimated as T_m").  layer_bwd: `saved` is a
                              SCRATCH buffer of merak_tmp_saved_bytes() bytes whose contents on entry
                              are ignored; the backward first regenerates every activation it reads
                              from x (the attention block incl. AR#1 / LN2, and fc1 + GeLU; fc2 and
                              AR#2 are not needed), then runs as usual.  layer_fwd: that
                              regeneration alone (a separately schedulable recompute pass, e.g. the
                              early recomputation of P:461); y is not written and may be NULL.
                              Results are bit-identical to a backward on the forward's own `saved`,
                              so a forward whose activations are recomputed may write its `saved`
                              into the same scratch buffer that every recomputed layer shares.
                              Collective (it contains AR#1).  EUNSUPPORTED in fp32 check mode.     */
};

typedef struct {
  int32_t hidden;      /* h */
  int32_t heads;       /* H                                                           */
  int32_t seq_len;     /* s */
  int32_t microbatch;  /* B */
  int32_t tmp_degree;  /* T: GPUs in the TMP group */
  int32_t tmp_rank;    /* r in [0, T)                                                 */
  int32_t n_sub;       /* sub-microbatches n (P:571 uses 2); 1 = Megatron baseline     */
  int32_t ffn_hidden;  /* f; 0 => 4h (reading R7)                                     */
  float ln_eps;        /* LayerNorm epsilon; 0 => 1e-5 (reading R3)                   */
  int32_t precision;   /* MERAK_BF16 | MERAK_FP32_CHECK (see "fp32 check mode" above)   */
  int32_t comm;        /* MERAK_COMM_PEER | MERAK_COMM_NCCL | MERAK_COMM_LOCAL        */
  int32_t comm_ctas;   /* CTAs used by each all-reduce kernel; 0 => auto              */
  int32_t device;      /* CUDA device ordinal this handle lives on                    */
  int32_t seq_parallel; /* 1 = sequence-parallel layout, see below   */
} merak_tmp_config;

/* Sequence-parallel layout (seq_parallel = 1, T > 1, comm PEER or INPROC, bf16): the row-parallel
 * all-reduces become reduce-scatters and the replicated LN / residual work is sharded by T.  x, y, dx, dy
 * are then the rank's TOKEN SHARD, [B*s/T, h]: for every sub-batch j (m = B*s/n tokens) rank r holds tokens
 * [j*m + r*m/T, j*m + (r+1)*m/T) as its local rows [j*m/T, (j+1)*m/T) -- the shard depends on n (the caller
 * reshards after merak_tmp_set_subbatches).  Forward per sub-batch: LN1 on the own rows; all-gather of u;
 * QKV, attention, proj (partial); reduce-scatter + b_o + residual + LN2 on the own rows; all-gather of u2; fc1,
 * fc2 (partial); reduce-scatter + b_2 + residual = the own rows of y.  Backward mirrors it with all-gathers of
 * dy and dx1 and reduce-scatters of the fc1 / QKV dgrad partials; the LN gradients are summed over the own
 * rows, then over the ranks in rank order.  Requires (B*s/n) % (8 T) == 0 (EINDIVISIBLE).  Numerics: every
 * row is computed by the same kernels as without sequence parallelism, so y, dx and the weight / bias
 * gradients are bit-identical to the replicated layout; the LN-parameter gradients differ in summation order. */

/* Collective used ONLY during init to exchange CUDA IPC handles (and the NCCL unique id):
 * gathers `bytes_per_rank` bytes from every rank of the TMP group into `recv` in rank order
 * (recv holds T * bytes_per_rank bytes).  Returns 0 on success.  The Python binding implements
 * it with torch.distributed.all_gather on the caller's process group. */
typedef int (*merak_allgather_fn)(void *ctx, const void *send, void *recv, size_t bytes_per_rank);

typedef struct {
  const void *ln1_g, *ln1_b, *w_qkv, *b_qkv, *w_o, *b_o, *ln2_g, *ln2_b, *w_1, *b_1, *w_2, *b_2;
} merak_tmp_weights;

typedef struct {
  float *ln1_g, *ln1_b, *w_qkv, *b_qkv, *w_o, *b_o, *ln2_g, *ln2_b, *w_1, *b_1, *w_2, *b_2;
} merak_tmp_grads;

/* Create a handle.  Validates the config (EINVAL / EINDIVISIBLE / EUNSUPPORTED), allocates the
 * peer-visible all-reduce slots, flags and the workspace on cfg->device (ENOMEM), creates the
 * two internal streams, and for T > 1 exchanges CUDA IPC handles through `ag` and maps every
 * peer's slots (EPEER); with comm == MERAK_COMM_NCCL it also creates an NCCL communicator.
 * Collective over the TMP group: every rank must call it with the same shape fields.
 * On success *out owns everything; release with merak_tmp_destroy. */
merak_status merak_tmp_init(const merak_tmp_config *cfg, merak_allgather_fn ag, void *ag_ctx,
                            merak_tmp_t **out);

/* Create all T = cfg->tmp_degree ranks of a TMP group as handles of this process on cfg->device
 * (MERAK_COMM_INPROC above; cfg->comm must be MERAK_COMM_PEER or MERAK_COMM_INPROC, cfg->tmp_rank is
 * ignored).  out[0..T-1] (host array of T handles) receives rank 0..T-1; same validation and errors as
 * merak_tmp_init; on failure no handle is left allocated.  The layer calls of the ranks never block the
 * host, so one host thread may issue rank 0's call, then rank 1's, ...; every rank must issue the same
 * sequence of collective calls.  merak_tmp_destroy of a member synchronises the device (all ranks' work),
 * so destroy members only after every rank has issued its last call; merak_tmp_bench_allreduce blocks the
 * calling thread and is therefore not usable from a single thread in this mode.  The ranks' internal
 * streams share one context: set CUDA_DEVICE_MAX_CONNECTIONS=32 before CUDA initialises, so that no
 * rank's compute stream shares a hardware queue with (and waits behind) another rank's spinning handshake;
 * at T = 8 each member runs all non-communication kernels on one stream to stay within 32 queues. */
merak_status merak_tmp_init_group(const merak_tmp_config *cfg, merak_tmp_t **out);

/* Change the number of sub-microbatches.  Requires B % n_sub == 0 (EINDIVISIBLE) and no
 * open chain (ESTATE).  Takes effect for the next layer_fwd/layer_bwd; all ranks must agree. */
merak_status merak_tmp_set_subbatches(merak_tmp_t *h, int32_t n_sub);

/* Bytes of the caller-owned `saved` buffer (activations kept from fwd for bwd). */
size_t merak_tmp_saved_bytes(const merak_tmp_t *h);

/* Forward: reads x (device, [B*s, h] bf16) and the weight shard, writes
 * y (device, [B*s, h] bf16) and `saved`.  Collective over the TMP group.  `st` = cudaStream_t. */
merak_status merak_tmp_layer_fwd(merak_tmp_t *h, const merak_tmp_weights *w, const void *x, void *y,
                                 void *saved, uint32_t flags, void *st);

/* Backward: reads x, `saved` (from the matching layer_fwd), dy; writes dx
 * ([B*s, h] bf16) and ACCUMULATES fp32 gradients into *g.  Collective over the TMP group.
 * With MERAK_FLAG_RECOMPUTE, `saved` is written (regenerated from x) before it is read. */
merak_status merak_tmp_layer_bwd(merak_tmp_t *h, const merak_tmp_weights *w, const void *x,
                                 const void *saved, const void *dy, void *dx, const merak_tmp_grads *g,
                                 uint32_t flags, void *st);

/* Join a MERAK_FLAG_CHAIN sequence: issue a chained forward's deferred AR#2s (MERAK_FUSE_LN1=1, see
 * MERAK_FLAG_CHAIN; collective then: every rank joins) and make `st` wait for every outstanding all-reduce. */
merak_status merak_tmp_join(merak_tmp_t *h, void *st);

/* Release all resources (synchronises the internal streams first).  NULL is a no-op. */
merak_status merak_tmp_destroy(merak_tmp_t *h);

/* Text of the last error on this handle (or of the last failed init when h == NULL). */
const char *merak_tmp_last_error(const merak_tmp_t *h);

/* ---- measurement hooks (used by bench.py; cheap, off by default) -------------------------- */

/* Kernel classes timed when profiling is on (cudaEvents around each launch on its stream). */
enum {
  MERAK_K_GEMM = 0, MERAK_K_ATTN_FWD = 1, MERAK_K_ATTN_BWD = 2, MERAK_K_LN = 3,
  MERAK_K_ALLREDUCE = 4, MERAK_K_REDUCE = 5, MERAK_K_NUM = 6
};

/* Turn per-kernel-class event timing on/off (resets the accumulators). */
merak_status merak_tmp_set_profiling(merak_tmp_t *h, int32_t on);

/* Sum of device milliseconds, launch counts and algorithmic FLOPs per class since
 * set_profiling(1) (synchronises the internal streams).  Arrays have MERAK_K_NUM entries. */
merak_status merak_tmp_get_profile(merak_tmp_t *h, double *ms, int64_t *launches, double *flops);

/* Per-launch timeline since set_profiling(1) (call before get_profile, which consumes it): for up to
 * `cap` launches, the kernel class, the stream (0 = compute (sub-batch or reduction streams), 1 = communication, 2 = wgrad filler) and start / end in ms
 * relative to the first recorded launch; *count receives the number written.  Synchronises. */
merak_status merak_tmp_get_timeline(merak_tmp_t *h, int32_t cap, int32_t *count, int32_t *cls, int32_t *stream,
                                    float *t0, float *t1);

/* Total kernels this handle launched since init (all classes, profiling on or off). */
int64_t merak_tmp_launch_count(const merak_tmp_t *h);

/* All-reduce microbenchmark (NVLink roofline evidence; collective over the TMP group, T > 1, bf16).
 * Runs `iters` back-to-back all-reduces of `rows` x h bf16 partials (rows <= B*s) through the same
 * path the layer uses (handshake kernel + one-shot, or two-shot at T >= 4, + fused epilogue), on the
 * communication stream with nothing else running, and writes the mean device time per all-reduce in
 * milliseconds to *ms.  which = 0: forward epilogue (AR#2: + bias + residual), 1: backward epilogue
 * (AR#3: LayerNorm backward + residual), 2: the cross-rank handshake kernel alone.  Partial
 * contents are zeros.  Synchronises the handle. */
merak_status merak_tmp_bench_allreduce(merak_tmp_t *h, int32_t which, int32_t rows, int32_t iters, float *ms);

/* Diagnostics, callable from another host thread while work is pending (never blocks): out[0..4] =
 * 1 if the internal stream (compute even, compute odd, wgrad filler, reductions, communication) still
 * has unfinished work, else 0; out[5..9] = the watchdog error word (flag, epoch, cta, peer*16+kind,
 * last flag value); out[10] = the handle's current handshake epoch; with MERAK_DEBUG_TRACE=1 set at init,
 * out[11..15] = the kernel class (MERAK_K_*) of the first unfinished launch on each of those streams
 * and out[16..20] its launch sequence number (-1 when none / tracing off).  out has 21 entries. */
merak_status merak_tmp_debug_state(const merak_tmp_t *h, int32_t *out);

/* Host-memory-only part of the diagnostics (no CUDA call, so it cannot block behind a launch):
 * out[0..4] = watchdog error word, out[5] = handshake epoch, out[6] = launches enqueued so far,
 * out[7..11] = traced launches enqueued per stream (cs, cs1, cw, cr, ms; MERAK_DEBUG_TRACE=1), out[12] = 1 when
 * the fused GEMM -> reduce-scatter push is set up (MERAK_AR_PUSH above; PEER / INPROC, T > 1, bf16), out[13] = 1
 * when the two-shot all-reduce is selected.  out has 14 entries. */
merak_status merak_tmp_debug_host(const merak_tmp_t *h, int32_t *out);

#ifdef __cplusplus
}
#endif
#endif /* MERAK_TMP_H */
