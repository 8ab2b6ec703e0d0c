// schedule.cu -- host-side planners of the C ABI in include/merak_sched.h (no device code).
//
// Stage-aware recomputation and the pipeline schedules of a K-layer TMP
// stage (NEXT-4).  Read each function against the passage it cites; the oracle (oracle/stage.py,
// oracle/pipeline.py) restates the passages independently and simulates the schedules for the tests.
#include <math.h>
#include <stddef.h>

#include <vector>

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

// ------------------------------------------------------------------------------------ pipeline schedules
namespace {

inline int32_t act(int kind, int mb) { return (kind << 24) | mb; }
inline int kind_of(int32_t a) { return a >> 24; }

// P:460 / Fig. 5a order on stage j of s with m microbatches: min(s-1-j, m) warm-up forwards, then one
// forward / one backward, then the remaining backwards.  `bwd` lists the action kinds of one backward.
std::vector<int32_t> one_f_one_b(int s, int m, int j, const std::vector<int> &bwd) {
  std::vector<int32_t> a;
  const int w = (s - 1 - j) < m ? (s - 1 - j) : m;
  int f = 0, b = 0;
  for (; f < w; ++f) a.push_back(act(MERAK_ACT_F, f));
  auto backward = [&]() {
    for (int k : bwd) a.push_back(act(k, b));
    ++b;
  };
  while (f < m) {
    a.push_back(act(MERAK_ACT_F, f++));
    backward();
  }
  while (b < m) backward();
  return a;
}

}  // namespace

extern "C" int merak_pipeline_schedule(int32_t policy, int32_t stages, int32_t microbatches, int32_t *actions,
                                       int32_t capacity, int32_t *count) {
  const int s = stages, m = microbatches;
  if (s < 1 || m < 1 || m >= (1 << 24) || !actions || !count) return MERAK_EINVAL;
  if (policy < MERAK_PIPE_1F1B || policy > MERAK_PIPE_1F1B_NO_RECOMPUTE) return MERAK_EINVAL;
  if (policy == MERAK_PIPE_SCP && s < 2) return MERAK_EINVAL;
  if (capacity < 3 * m) return MERAK_ENOMEM;
  for (int j = 0; j < s; ++j) {
    std::vector<int32_t> a;
    switch (policy) {
      case MERAK_PIPE_1F1B: a = one_f_one_b(s, m, j, {MERAK_ACT_BR}); break;
      case MERAK_PIPE_1F1B_NO_RECOMPUTE: a = one_f_one_b(s, m, j, {MERAK_ACT_B}); break;
      case MERAK_PIPE_EARLY_RECOMPUTE: a = one_f_one_b(s, m, j, {MERAK_ACT_R, MERAK_ACT_B}); break;
      case MERAK_PIPE_SCP:
        if (j == s - 1) {  // (a) "drop the recomputation of the last stage"
          a = one_f_one_b(s, m, j, {MERAK_ACT_B});
        } else {
          a = one_f_one_b(s, m, j, {MERAK_ACT_R, MERAK_ACT_B});
          if (j == s - 2) {  // (b) "bring one forward pass computation of the second to last stage ahead"
            size_t first_rb = 0;
            while (first_rb < a.size() && kind_of(a[first_rb]) == MERAK_ACT_F) ++first_rb;
            size_t nf = first_rb;
            while (nf < a.size() && kind_of(a[nf]) != MERAK_ACT_F) ++nf;
            if (nf < a.size()) {  // (c) the first backwards' recomputations then follow that forward
              const int32_t f = a[nf];
              a.erase(a.begin() + (long)nf);
              a.insert(a.begin() + (long)first_rb, f);
            }
          }
        }
        break;
    }
    count[j] = (int32_t)a.size();
    for (size_t k = 0; k < a.size(); ++k) actions[(size_t)j * capacity + k] = a[k];
  }
  return MERAK_OK;
}
