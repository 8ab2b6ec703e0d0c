/*
 * merak_sched.h -- C ABI of the host-side planners around the sub-pipelined TMP layer (libmerak_tmp.so):
 * stage-aware recomputation and the pipeline schedules that drive a K-layer TMP
 * stage with several microbatches (NEXT-4).  Plain host computation: no device memory, no CUDA calls.
 * All functions return merak_status values (0 = OK, negative = error; see merak_tmp.h), never abort.
 * Stage and microbatch indices are 0-based here; the paper's formulas are 1-based (stage i = index i-1).
 */
#ifndef MERAK_SCHED_H
#define MERAK_SCHED_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- stage-aware recomputation (§6.2) ------------------------------------------------
 * alpha_i = fraction of the modules (here: transformer layers) of pipeline stage i that keep their
 * activations instead of recomputing them.  P:523-526 (1-based i, s stages):
 *   alpha_i = min(1, (s-1) alpha_1 / (s-i))   for i in [2, s-1)
 *   alpha_{s-1} = alpha_{s-2}
 *   alpha_s = 1
 * out: host array of `stages` doubles (out[0] = alpha_1).  EINVAL: stages < 1, alpha1 outside [0, 1],
 * out NULL.  For s = 1 the single stage is both first and last: out[0] = 1 ("i = s"); for s = 2,
 * out = {alpha_1, 1}; for s = 3, alpha_2 = alpha_{s-1} = alpha_{s-2} = alpha_1. */
int merak_stage_alpha(int32_t stages, double alpha1, double *out);

/* Stage memory model of P:520-521: stage i (1-based) needs M_r + (s - i) alpha_i M_a bytes
 * (runtime memory M_r: model states, buffers, one microbatch's activations; M_a: activations of one
 * microbatch kept without recomputation).  tune: "we tune alpha_1 by increasing it at intervals until
 * catching an out-of-memory error", the OOM replaced by the capacity check: returns in
 * *alpha1 the largest alpha_1 in {0, step, 2 step, ..., <= 1} (1 itself always a candidate) whose
 * stage-aware plan keeps every stage within `capacity` bytes.  EINVAL: bad arguments (stages < 1,
 * step <= 0, negative sizes); ENOMEM: even alpha_1 = 0 does not fit (M_r > capacity). */
int merak_tune_alpha1(int32_t stages, double step, double capacity, double m_r, double m_a, double *alpha1);

/* Layers of a K-layer stage that keep activations under alpha (rounded down to whole layers). */
int32_t merak_layers_kept(double alpha, int32_t layers);

/* ---- pipeline schedules of a K-layer TMP stage (§6.1) ---------------
 * One action per int32: (kind << 24) | microbatch.  Kinds:
 *   MERAK_ACT_F   forward of microbatch mb through the stage (keeps each layer's input; the layers that keep
 *                 their activations keep them, the others write a scratch buffer);
 *   MERAK_ACT_R   recomputation of mb's activations (layer_fwd with MERAK_FLAG_RECOMPUTE for every recomputed
 *                 layer); "the activation recomputation operation does not depend on the output of previous
 *                 stages", so it runs as soon as the stage reaches it;
 *   MERAK_ACT_B   backward of mb on activations that exist (kept or recomputed by an earlier R);
 *   MERAK_ACT_BR  backward of mb with the recomputation fused in front of it (layer_bwd with
 *                 MERAK_FLAG_RECOMPUTE): it starts only once mb's gradient has arrived (Fig. 5a's 1F1B).
 * A forward on stage j > 0 receives mb's activation from stage j-1; a backward on stage j < s-1 receives mb's
 * gradient from stage j+1 (sends are implied by the producer's F / B / BR).
 * Policies:
 *   MERAK_PIPE_1F1B            Fig. 5a: stage j runs min(s-1-j, m) warm-up forwards, then one forward / one
 *                              backward alternately, then drains the backwards; every backward is BR.
 *                              Bubble (s-1)(T_m + T_m + 2T_m), ratio (s-1)/m.
 *   MERAK_PIPE_EARLY_RECOMPUTE Fig. 5b: the same order with each backward split into R then B, so the
 *                              recomputation no longer waits for the gradient.  Bubble (s-1)(T_m + 2T_m),
 *                              ratio 3(s-1)/(4m).
 *   MERAK_PIPE_SCP             Fig. 5c, shifted critical path: EARLY_RECOMPUTE with (a) no
 *                              recomputation on the last stage ("the last stage only stores one activation":
 *                              its backwards are B), (b) on stage s-2, one forward brought ahead into the
 *                              warm-up bubble (the first forward after its first R / B moves in front of
 *                              them), (c) its first backwards' recomputations following that order.  Bubble
 *                              3(s-2)T_m, ratio 3(s-2)/(4m) for m >= max(s, 3).  Needs s >= 2 (EINVAL).
 *   MERAK_PIPE_1F1B_NO_RECOMPUTE  1F1B with every activation kept (F and B only).
 * actions: host array of stages x capacity int32; row j receives stage j's ordered actions and count[j]
 * their number (3 m at most).  EINVAL: bad policy / sizes; ENOMEM: capacity < 3 m. */
enum {
  MERAK_PIPE_1F1B = 0,
  MERAK_PIPE_EARLY_RECOMPUTE = 1,
  MERAK_PIPE_SCP = 2,
  MERAK_PIPE_1F1B_NO_RECOMPUTE = 3
};
enum { MERAK_ACT_F = 0, MERAK_ACT_R = 1, MERAK_ACT_B = 2, MERAK_ACT_BR = 3 };
int merak_pipeline_schedule(int32_t policy, int32_t stages, int32_t microbatches, int32_t *actions,
                            int32_t capacity, int32_t *count);

#ifdef __cplusplus
}
#endif
#endif
