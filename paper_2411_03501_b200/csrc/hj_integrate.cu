// hj_integrate.cu -- the native integration loop (host C++): the scalar step
// logic of the reference integrator (integrator.py:76-109) replayed in IEEE
// doubles, every TVD-RK stage one fused kernel launch, no host<->device
// synchronisation inside the loop.  Used by the package whenever the term is
// a registered device Hamiltonian with range-free dissipation bounds.
#include <cmath>
#include <cstring>
#include "hj_kernels.cuh"

namespace hj {
cudaError_t launch_stage_generic(int scheme, const StageArgs& P, cudaStream_t s);
cudaError_t launch_stage_fast(int scheme, const StageArgs& P, cudaStream_t s, bool* handled);
}  // namespace hj

using namespace hj;

extern "C" int hj_stage(const hj_grid* g, int scheme, const hj_ham* ham, const double* alpha, double dt, int stage,
                        const double* y_in, const double* y0, double* y_out, const double* mask_prev, int mask,
                        hj_stats* stats, int32_t tag, void* stream);
extern "C" const char* hj_last_error(void);

namespace {
int stages_of(int order, int* kinds) {
  if (order == 1) { kinds[0] = HJ_STAGE_EULER; return 1; }
  if (order == 2) { kinds[0] = HJ_STAGE_EULER; kinds[1] = HJ_STAGE_RK2_AVG; return 2; }
  kinds[0] = HJ_STAGE_EULER; kinds[1] = HJ_STAGE_RK3_QUARTER; kinds[2] = HJ_STAGE_RK3_THIRD;
  return 3;
}
}  // namespace

extern "C" int hj_integrate(const hj_grid* g, int scheme, const hj_ham* ham, const double* alpha, int order,
                            double t0, double t1, double cfl, double max_step, int single_step, double bound,
                            const double* y_init, double* buf0, double* buf1, double* buf2,
                            const double* mask_prev, int mask, hj_stats* stats, double* info, double** y_final,
                            void* stream) {
  if (order < 1 || order > 3) return HJ_EINVAL;
  if (!info || !y_final || !y_init || !buf0 || !buf1 || !buf2) return HJ_EINVAL;
  int kinds[3];
  const int nst = stages_of(order, kinds);
  double* bufs[3] = {buf0, buf1, buf2};
  const double* cur = y_init;
  double t = t0;
  long long steps = 0;
  double min_dt = INFINITY, max_dt = 0.0;
  int rc = HJ_OK;
  info[4] = 0.0;   // 1 when the step-size test failed (reference: RuntimeError "no usable step size")
  while (t < t1) {
    double dt = cfl * bound;                         // integrator.py:82
    if (max_step > 0.0) dt = (max_step < dt) ? max_step : dt;   // min(dt, max_step)
    const double remaining = t1 - t;                 // integrator.py:85
    const bool last = dt >= remaining;
    if (last) dt = remaining;
    if (!(dt > 0.0 && std::isfinite(dt))) {         // integrator.py:89-90
      info[4] = 1.0;
      info[5] = dt;
      break;
    }
    const double t_next = last ? t1 : t + dt;        // integrator.py:106
    const bool final_step = last || single_step || !(t_next < t1);
    // the three buffers never alias the step input; rotate outputs among those != cur
    double* outs[2];
    int k = 0;
    for (int b = 0; b < 3 && k < 2; ++b)
      if (bufs[b] != cur) outs[k++] = bufs[b];
    const double* src = cur;
    double* dst = outs[0];
    for (int s = 0; s < nst; ++s) {
      if (s > 0) dst = (src == outs[0]) ? outs[1] : outs[0];
      const bool lastst = final_step && s == nst - 1;
      rc = hj_stage(g, scheme, ham, alpha, dt, kinds[s], src, kinds[s] == HJ_STAGE_EULER ? nullptr : cur, dst,
                    lastst ? mask_prev : nullptr, lastst ? mask : HJ_MASK_NONE, stats,
                    (int32_t)(steps * 4 + s), stream);
      if (rc) return rc;
      src = dst;
    }
    cur = src;
    t = t_next;
    ++steps;
    min_dt = (dt < min_dt) ? dt : min_dt;
    max_dt = (dt > max_dt) ? dt : max_dt;
    if (single_step) break;
  }
  if (steps == 0) min_dt = 0.0;
  info[0] = t;
  info[1] = (double)steps;
  info[2] = min_dt;
  info[3] = max_dt;
  *y_final = const_cast<double*>(cur);
  return rc;
}
