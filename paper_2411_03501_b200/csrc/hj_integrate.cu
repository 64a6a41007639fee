// hj_integrate.cu -- the native integration loop (host C++): the scalar step
// logic of the reference integrator (integrator.py:76-109) replayed in IEEE
// doubles, every TVD-RK stage one fused kernel launch, no host<->device
// synchronisation inside the loop.  Used by the package whenever the term is
// a registered device Hamiltonian with range-free dissipation bounds.
#include <cmath>
#include <string>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>
#include "hj_stage_generic.cuh"

namespace hj {
cudaError_t launch_stage_generic(int scheme, const StageArgs& P, cudaStream_t s);
cudaError_t launch_stage_fast(int scheme, const StageArgs& P, cudaStream_t s, bool* handled);
cudaError_t launch_persist(int scheme, const StageArgs& P, const PersistArgs& A, cudaStream_t s);
bool persist_applies(const StageArgs& P);
int set_error(int code, const char* msg);
void count_launches(uint64_t n);
int stage_args(const hj_grid* g, int scheme, const hj_ham* ham, const double* alpha, double dt, int stage,
               const double* y_in, const double* y0, double* y_out, const double* mask_prev, int mask,
               hj_stats* stats, int32_t tag, StageArgs* P);
}  // namespace hj

using namespace hj;

extern "C" int hj_stage(const hj_grid* g, int scheme, const hj_ham* ham, const double* alpha, double dt, int stage,
                        const double* y_in, const double* y0, double* y_out, const double* mask_prev, int mask,
                        hj_stats* stats, int32_t tag, void* stream);
extern "C" const char* hj_last_error(void);

namespace {
// One stage of the schedule: what hj_stage would be called with.
struct StageRec {
  const double* src;
  const double* y0;
  double* dst;
  int kind;
  bool masked;
  double dt;
  int32_t tag;
};

// The whole schedule as ONE persistent launch per PERSIST_MAX_STAGES stages
// (k_stage_persist).  Returns HJ_OK, an error code (< 0), or NOT_PERSISTENT
// when the configuration is not one the persistent kernel covers (the caller
// then launches stage by stage).
constexpr int NOT_PERSISTENT = 1;

// Barrier words of the persistent launches, one pair per (device, stream):
// launches on one stream are ordered, so they may share it; launches on two
// streams never do.  Allocated once per stream and kept (a cache; at most
// BARRIER_STREAMS streams, beyond that the per-stage path runs).
constexpr size_t BARRIER_STREAMS = 64;
unsigned* barrier_for(cudaStream_t s) {
  struct Entry {
    int dev;
    cudaStream_t stream;
    unsigned* p;
  };
  static std::mutex mu;
  static std::vector<Entry> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  for (const Entry& e : cache)
    if (e.dev == dev && e.stream == s) return e.p;
  if (cache.size() >= BARRIER_STREAMS) return nullptr;
  unsigned* p = nullptr;
  if (cudaMalloc((void**)&p, BAR_WORDS * sizeof(unsigned)) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  cache.push_back(Entry{dev, s, p});
  return p;
}
int run_persistent(const hj_grid* g, int scheme, const hj_ham* ham, const double* alpha,
                   const std::vector<StageRec>& recs, const double* y_init, double* const* bufs,
                   const double* mask_prev, int mask, hj_stats* stats, void* stream) {
#ifdef HJ_CHECK_BOUNDS
  return NOT_PERSISTENT;   // the bounds-checking build checks per-stage extents: per-stage launches only
#else
  if (recs.empty() || g->halo_lo || g->halo_hi) return NOT_PERSISTENT;
  // validate what the per-stage calls would validate: the first stage of
  // every kind and the masked stage (the others differ only in pointers the
  // rotation above produces)
  StageArgs P;
  bool seen[8] = {false};
  for (const StageRec& r : recs) {
    if (seen[r.kind] && !r.masked) continue;
    seen[r.kind] = true;
    const int rc = stage_args(g, scheme, ham, alpha, r.dt, r.kind, r.src, r.y0, r.dst, r.masked ? mask_prev : nullptr,
                              r.masked ? mask : HJ_MASK_NONE, stats, r.tag, &P);
    if (rc) return rc;
  }
  if (!persist_applies(P)) return NOT_PERSISTENT;
  const double* ids[4] = {y_init, bufs[0], bufs[1], bufs[2]};
  auto id_of = [&](const double* p) -> int {
    for (int i = 0; i < 4; ++i)
      if (ids[i] == p) return i;
    return -1;
  };
  cudaStream_t s = (cudaStream_t)stream;
  unsigned* bar = barrier_for(s);
  if (!bar) return NOT_PERSISTENT;
  std::unique_ptr<PersistArgs> X(new PersistArgs);   // 16 KB: becomes the launch's parameter block
  for (int i = 0; i < 4; ++i) X->buf[i] = ids[i];
  X->mask_prev = mask_prev;
  X->bar = bar;
  int rc = HJ_OK;
  for (size_t base = 0; base < recs.size() && rc == HJ_OK; base += PERSIST_MAX_STAGES) {
    const size_t n = recs.size() - base < (size_t)PERSIST_MAX_STAGES ? recs.size() - base : PERSIST_MAX_STAGES;
    X->nstages = (int)n;
    for (size_t k = 0; k < n; ++k) {
      const StageRec& r = recs[base + k];
      PersistStage& d = X->st[k];
      std::memset(&d, 0, sizeof d);
      d.dt = r.dt;
      d.tag = r.tag;
      d.src = (int8_t)id_of(r.src);
      d.y0 = (int8_t)(r.y0 ? id_of(r.y0) : -1);
      d.dst = (int8_t)id_of(r.dst);
      d.kind = (int8_t)r.kind;
      d.mask = (int8_t)(r.masked ? mask : HJ_MASK_NONE);
    }
    cudaError_t e = cudaMemsetAsync(bar, 0, BAR_WORDS * sizeof(unsigned), s);
    if (e == cudaSuccess) e = launch_persist(scheme, P, *X, s);
    if (e != cudaSuccess && base == 0 && e != cudaErrorIllegalAddress && e != cudaErrorLaunchFailure) {
      // the cooperative launch itself was refused (nothing ran): per-stage launches instead
      cudaGetLastError();
      return NOT_PERSISTENT;
    }
    if (e != cudaSuccess) {
      std::string msg = std::string("hj_integrate (persistent): ") + cudaGetErrorString(e);
      rc = set_error(HJ_ECUDA, msg.c_str());
    } else {
      count_launches(1);
    }
  }
  return rc;
#endif
}

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
  std::vector<StageRec> recs;   // the schedule: the stage calls of the reference loop, in order
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
      recs.push_back(StageRec{src, kinds[s] == HJ_STAGE_EULER ? nullptr : cur, dst, kinds[s], lastst, dt,
                              (int32_t)(steps * 4 + s)});
      src = dst;
    }
    cur = src;
    t = t_next;
    ++steps;
    min_dt = (dt < min_dt) ? dt : min_dt;
    max_dt = (dt > max_dt) ? dt : max_dt;
    if (single_step) break;
  }
  // run the schedule: one persistent launch where it applies, else one
  // fused-stage launch per stage
  rc = run_persistent(g, scheme, ham, alpha, recs, y_init, bufs, mask_prev, mask, stats, stream);
  if (rc < 0) return rc;
  if (rc == NOT_PERSISTENT) {
    for (const StageRec& r : recs) {
      rc = hj_stage(g, scheme, ham, alpha, r.dt, r.kind, r.src, r.y0, r.dst, r.masked ? mask_prev : nullptr,
                    r.masked ? mask : HJ_MASK_NONE, stats, r.tag, stream);
      if (rc) return rc;
    }
  }
  rc = HJ_OK;
  if (steps == 0) min_dt = 0.0;
  info[0] = t;
  info[1] = (double)steps;
  info[2] = min_dt;
  info[3] = max_dt;
  *y_final = const_cast<double*>(cur);
  return rc;
}
