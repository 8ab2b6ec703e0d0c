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

#ifdef __cplusplus
}
#endif
#endif
