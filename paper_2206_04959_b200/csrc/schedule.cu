// schedule.cu -- host-side planners of the C ABI in include/merak_sched.h (no device code).
//
// Stage-aware recomputation.  Read each function against the passage
// it cites; the fp64 oracle (oracle/stage.py) restates the same passages independently for the tests.
#include <math.h>
#include <stddef.h>

#include "merak_sched.h"
#include "merak_tmp.h"

namespace {

// P:523-526, 1-based stage i of s: alpha_i = min(1, (s-1) alpha_1 / (s-i)) for i in [2, s-1);
// alpha_{s-1} = alpha_{s-2}; alpha_s = 1.
void stage_alpha(int s, double a1, double *out) {
  for (int i = 1; i <= s; ++i) {
    double a;
    if (i == s)
      a = 1.0;
    else if (i == 1)
      a = a1;
    else if (i < s - 1)
      a = fmin(1.0, (double)(s - 1) * a1 / (double)(s - i));
    else  // i == s - 1 (s >= 3 here): equal to stage s - 2 (already computed)
      a = out[i - 2];
    out[i - 1] = a;
  }
}

// stage i needs M_r + (s - i) alpha_i M_a
bool plan_fits(int s, double a1, double cap, double m_r, double m_a, double *buf) {
  stage_alpha(s, a1, buf);
  for (int i = 1; i <= s; ++i)
    if (m_r + (double)(s - i) * buf[i - 1] * m_a > cap) return false;
  return true;
}

}  // namespace

extern "C" int merak_stage_alpha(int32_t stages, double alpha1, double *out) {
  if (stages < 1 || !out || !(alpha1 >= 0.0 && alpha1 <= 1.0)) return MERAK_EINVAL;
  stage_alpha(stages, alpha1, out);
  return MERAK_OK;
}

extern "C" int merak_tune_alpha1(int32_t stages, double step, double capacity, double m_r, double m_a,
                                 double *alpha1) {
  if (stages < 1 || !alpha1 || !(step > 0.0) || m_r < 0.0 || m_a < 0.0 || capacity < 0.0) return MERAK_EINVAL;
  if (stages > 4096) return MERAK_EINVAL;
  double buf[4096];
  if (!plan_fits(stages, 0.0, capacity, m_r, m_a, buf)) return MERAK_ENOMEM;
  // increase alpha_1 at intervals of `step` until the plan no longer fits (alpha_1 = 1 included)
  double best = 0.0;
  for (long k = 1;; ++k) {
    double a = (double)k * step;
    const bool last = a >= 1.0;
    if (last) a = 1.0;
    if (!plan_fits(stages, a, capacity, m_r, m_a, buf)) break;
    best = a;
    if (last) break;
  }
  *alpha1 = best;
  return MERAK_OK;
}

extern "C" int32_t merak_layers_kept(double alpha, int32_t layers) {
  if (layers <= 0 || !(alpha > 0.0)) return 0;
  if (alpha >= 1.0) return layers;
  return (int32_t)floor(alpha * (double)layers + 1e-9);
}
