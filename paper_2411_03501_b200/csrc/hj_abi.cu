// hj_abi.cu -- extern "C" entry points of libhjb200.so (declared in
// include/hjb200.h).  Validation mirrors the reference's ValueError checks;
// failures return HJ_E* and leave a thread-local message.
#include <algorithm>
#include <atomic>
#include <vector>
#include <mutex>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include "hj_kernels.cuh"

namespace hj {
cudaError_t launch_stage_generic(int scheme, const StageArgs& P, cudaStream_t s);
cudaError_t launch_stage_fast(int scheme, const StageArgs& P, cudaStream_t s, bool* handled);
cudaError_t launch_derivs(int scheme, const GridArgs& G, int axis, int eps_mode, const double* v,
                          double* left, double* right, cudaStream_t s);
cudaError_t launch_weno_ws(const GridArgs& G, int axis, int side, int eps_mode, const double* v,
                           double* ws, cudaStream_t s);
cudaError_t launch_extend(const GridArgs& G, int w, const double* v, double* ext, cudaStream_t s);
cudaError_t launch_shape(const GridArgs& G, int kind, const double* prm, int nprm, double* out, cudaStream_t s);
cudaError_t launch_csg(int op, long long n, const double* a, const double* b, double* out, cudaStream_t s);
cudaError_t launch_mask(long long n, const double* prev, double* v, int mask, cudaStream_t s);
cudaError_t launch_count_below(long long n, const double* v, double level, unsigned long long* c,
                               cudaStream_t s);
cudaError_t launch_stats_reset(hj_stats* st, cudaStream_t s);
cudaError_t launch_tube_check(long long n, const double* prev, const double* v, const double* target, int mask_min,
                              double level, unsigned long long* out, cudaStream_t s);
cudaError_t launch_costates(const GridArgs& G, const double* const* l, const double* const* r,
                            double* const* p, hj_stats* st, cudaStream_t s);
cudaError_t launch_glf_delta(const GridArgs& G, const double* ahalf, const double* const* l,
                             const double* const* r, const double* ham, double* diss, double* delta,
                             hj_stats* st, cudaStream_t s);
cudaError_t launch_rk_combine(long long n, int stage, double dt, const double* y, const double* y0,
                              const double* delta, double* out, hj_stats* st, int tag, cudaStream_t s);
cudaError_t launch_eval_ham(const GridArgs& G, const hj_ham& H, const double* const* p, double* out,
                            cudaStream_t s);
cudaError_t launch_check_division(long long n, unsigned long long seed, unsigned long long* mism, cudaStream_t s);
cudaError_t launch_fp64_probe(int iters, int blocks, double* out, cudaStream_t s);
cudaError_t launch_divdiff(const GridArgs& G, int axis, int w, int order, const double* v, double* d0,
                           double* d1, double* d2, double* d3, cudaStream_t s);
}  // namespace hj

using namespace hj;

static thread_local std::string g_err;
static std::atomic<uint64_t> g_launches{0};

static int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

namespace hj {
bool axes_applies(int scheme, const StageArgs& P, bool allow_halo);   // hj_fast.cu
cudaError_t launch_axes_weno5(const StageArgs& P, cudaStream_t s, bool* handled, int parts);   // hj_axes_weno.cu
// for the other translation units of the library (hj_dd.cu): set the
// thread-local message / count launches made outside this file
int set_error(int code, const char* msg) {
  g_err = msg ? msg : "";
  return code;
}
void count_launches(uint64_t n) { g_launches += n; }
}  // namespace hj

static int cuda_status(cudaError_t e, const char* what, uint64_t launches = 1) {
  if (e != cudaSuccess) return fail(HJ_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  g_launches += launches;
  g_err.clear();
  return HJ_OK;
}

// hj_grid -> GridArgs, with the reference's validation (grid.py:117-175, spatial.py:74-81).
static int make_grid(const hj_grid* g, int ghost_width, GridArgs* G, unsigned ghost_axes = 0xffu) {
  if (!g) return fail(HJ_EINVAL, "grid is NULL");
  if (g->dim < 1 || g->dim > 4) return fail(HJ_EINVAL, "grid dim %d unsupported (1..4)", g->dim);
  if (g->batch < 1) return fail(HJ_EINVAL, "batch must be >= 1, got %d", g->batch);
  std::memset(G, 0, sizeof *G);
  G->dim = g->dim;
  G->batch = g->batch;
  long long cells = 1;
  for (int a = 0; a < g->dim; ++a) {
    if (g->n[a] < 1 || g->n[a] > 0x7fffffffLL) return fail(HJ_EINVAL, "axis %d: bad node count %lld", a, (long long)g->n[a]);
    G->n[a] = (int)g->n[a];
    cells *= g->n[a];
  }
  G->cells = cells;
  long long st = 1;
  for (int a = g->dim - 1; a >= 0; --a) {
    G->stride[a] = st;
    st *= g->n[a];
  }
  G->batch_stride = g->batch_stride ? g->batch_stride : cells;
  for (int a = 0; a < g->dim; ++a) {
    AxisView& A = G->ax[a];
    A.stride = G->stride[a];
    A.n = G->n[a];
    A.bc = g->bc[a];
    A.bcv = g->bc_value[a];
    A.halo_lo = (a == 0) ? g->halo_lo : 0;
    A.halo_hi = (a == 0) ? g->halo_hi : 0;
    A.halo_n = (a == 0 && (g->halo_lo || g->halo_hi)) ? g->halo : 0;
    if (A.bc < HJ_BC_PERIODIC || A.bc > HJ_BC_DIRICHLET)
      return fail(HJ_EINVAL, "axis %d: unknown boundary kind %d", a, A.bc);
    // the brick kernels stage HJ_HALO_MIN exchanged planes per side whatever
    // the scheme's ghost width, so a thinner halo would be read out of bounds
    if (a == 0 && (A.halo_lo || A.halo_hi) && g->halo < HJ_HALO_MIN)
      return fail(HJ_EINVAL, "axis 0 halo %d thinner than the %d planes the stage kernels read", g->halo,
                  HJ_HALO_MIN);
    if (((ghost_axes >> a) & 1u) && (A.halo_lo || A.halo_hi) && g->halo < ghost_width)
      return fail(HJ_EINVAL, "axis 0 halo %d thinner than ghost width %d", g->halo, ghost_width);
    if (((ghost_axes >> a) & 1u) && ghost_width > 0 && A.bc == HJ_BC_PERIODIC && !(A.halo_lo && A.halo_hi) && ghost_width > A.n)
      return fail(HJ_EINVAL, "ghost width %d exceeds %d nodes on periodic axis %d", ghost_width, A.n, a);
    if (((ghost_axes >> a) & 1u) && ghost_width > 0 && A.bc == HJ_BC_EXTRAPOLATE && A.n < 2 && !(A.halo_lo && A.halo_hi))
      return fail(HJ_EINVAL, "axis %d: extrapolation needs at least 2 nodes", a);
    if (!(g->h[a] > 0.0)) return fail(HJ_EINVAL, "axis %d: spacing must be positive", a);
    G->sp[a].h = g->h[a];
    G->sp[a].h2 = 2.0 * g->h[a];
    G->sp[a].h3 = 3.0 * g->h[a];
    G->sp[a].rh = 1.0 / g->h[a];
    G->nodes[a] = g->nodes[a];
  }
  return HJ_OK;
}

static bool all_zero(const double* alpha, int dim) {
  for (int a = 0; a < dim; ++a)
    if (alpha[a] != 0.0) return false;
  return true;
}

static int ghost_width_of(int scheme) {
  switch (scheme) {
    case HJ_FIRST: return 1;
    case HJ_ENO2: return 2;
    case HJ_ENO3: return 3;
    case HJ_WENO5: return 3;
    case HJ_WENO5_FMA: return 3;
    default: return -1;
  }
}

static int check_ham(const hj_ham* ham, int dim) {
  if (!ham) return fail(HJ_EINVAL, "hamiltonian is NULL");
  switch (ham->kind) {
    case HJ_HAM_ADVECTION: return HJ_OK;
    case HJ_HAM_ROCKETS:
    case HJ_HAM_ROCKETS_EXTREMAL:
    case HJ_HAM_AIR3D:
      if (dim != 3) return fail(HJ_EINVAL, "hamiltonian kind %d needs a 3-D grid, got dim %d", ham->kind, dim);
      if (!ham->tab[0] || !ham->tab[1]) return fail(HJ_EINVAL, "hamiltonian kind %d needs trig tables", ham->kind);
      return HJ_OK;
    case HJ_HAM_DI4:
      if (dim != 4) return fail(HJ_EINVAL, "di4 hamiltonian needs a 4-D grid, got dim %d", dim);
      return HJ_OK;
    default: return fail(HJ_EINVAL, "unknown hamiltonian kind %d", ham->kind);
  }
}

// Device scratch for the 4-D pre-pass, cached per (device, stream) so that
// solvers on different streams never share it; grown on demand.  At most
// SCRATCH_ENTRIES buffers live at once: the least recently used one is freed
// (cudaFree synchronises the device, so a buffer is never released while a
// kernel still uses it).
constexpr size_t SCRATCH_ENTRIES = 16;   // (a batch solve runs one stream per problem)
static double* scratch_for(cudaStream_t s, size_t n_doubles) {
  struct Entry {
    int dev;
    cudaStream_t stream;
    double* p;
    size_t n;
    uint64_t used;
  };
  static std::mutex mu;
  static std::vector<Entry> cache;
  static uint64_t clock = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  Entry* e = nullptr;
  for (auto& c : cache)
    if (c.dev == dev && c.stream == s) e = &c;
  if (!e) {
    if (cache.size() >= SCRATCH_ENTRIES) {
      auto lru = std::min_element(cache.begin(), cache.end(),
                                  [](const Entry& a, const Entry& b) { return a.used < b.used; });
      int cur = 0;
      cudaGetDevice(&cur);
      cudaSetDevice(lru->dev);
      cudaFree(lru->p);
      cudaSetDevice(cur);
      cache.erase(lru);
    }
    cache.push_back(Entry{dev, s, nullptr, 0, 0});
    e = &cache.back();
  }
  e->used = ++clock;
  if (e->n < n_doubles) {
    if (e->p) cudaFree(e->p);
    e->p = nullptr;
    e->n = 0;
    if (cudaMalloc((void**)&e->p, n_doubles * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      e->p = nullptr;
      return nullptr;   // the caller falls back to the generic kernel
    }
    e->n = n_doubles;
  }
  return e->p;
}

// ---- bounds checking (libhjb200_check.so, -DHJ_CHECK_BOUNDS): the extents of
// the fields a stage touches and a per-device violation counter
#ifdef HJ_CHECK_BOUNDS
static unsigned long long* oob_counter() {
  static std::mutex mu;
  static unsigned long long* per_dev[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!per_dev[dev]) {
    if (cudaMalloc((void**)&per_dev[dev], sizeof(unsigned long long)) != cudaSuccess) return nullptr;
    cudaMemset(per_dev[dev], 0, sizeof(unsigned long long));
  }
  return per_dev[dev];
}
#endif

static void set_extents(StageArgs& P, const hj_grid* g) {
  const GridArgs& G = P.g;
  long long plane = 1;
  for (int a = 1; a < G.dim; ++a) plane *= G.n[a];
  const long long span = G.batch_stride * (G.batch - 1) + G.cells;
  const long long below = g->halo_lo ? (long long)g->halo * plane : 0;
  const long long above = g->halo_hi ? (long long)g->halo * plane : 0;
  P.bc.in = Extent{P.y_in - below, P.y_in + span + above};
  P.bc.y0 = Extent{P.y0, P.y0 ? P.y0 + span : nullptr};
  P.bc.out = Extent{P.y_out, P.y_out + span};
  P.bc.mask = Extent{P.mask_prev, P.mask_prev ? P.mask_prev + span : nullptr};
  P.bc.aux = Extent{P.aux0, P.aux0 ? P.aux0 + 2 * span : nullptr};
#ifdef HJ_CHECK_BOUNDS
  P.bc.oob = oob_counter();
#else
  P.bc.oob = nullptr;
#endif
}

// Derived constants computed once on the host side of the ABI.
static hj_ham prep_ham(const hj_ham* ham) {
  hj_ham h = *ham;
  if (ham->kind == HJ_HAM_ROCKETS_EXTREMAL) {
    // reachability.py:94-95: mid = 0.5*(u_max + u_min), half = 0.5*(u_max - u_min)
    h.p[4] = 0.5 * (ham->p[3] + ham->p[2]);
    h.p[5] = 0.5 * (ham->p[3] - ham->p[2]);
  }
  if (ham->kind == HJ_HAM_DI4) h.p[2] = ham->p[1] - ham->p[0];  // d_bar - u_bar
  return h;
}

extern "C" {

int hj_version(void) { return 1; }
const char* hj_last_error(void) { return g_err.c_str(); }
uint64_t hj_launch_count(void) { return g_launches.load(); }

int hj_extend_ghost(const hj_grid* g, int width, const double* v, double* ext, void* stream) {
  if (width < 1) return fail(HJ_EINVAL, "ghost width must be >= 1, got %d", width);
  GridArgs G;
  int rc = make_grid(g, width, &G);
  if (rc) return rc;
  if (G.batch != 1 || g->halo_lo || g->halo_hi) return fail(HJ_EINVAL, "extend_ghost takes one un-haloed field");
  if (!v || !ext) return fail(HJ_EINVAL, "NULL field pointer");
  return cuda_status(launch_extend(G, width, v, ext, (cudaStream_t)stream), "hj_extend_ghost");
}

int hj_derivs(const hj_grid* g, int scheme, int axis, int eps_mode, const double* v, double* left,
              double* right, void* stream) {
  const int w = ghost_width_of(scheme);
  if (w < 0) return fail(HJ_EINVAL, "unknown derivative scheme %d", scheme);
  GridArgs G;
  int rc = make_grid(g, w, &G, 1u << (axis & 7));
  if (rc) return rc;
  if (axis < 0 || axis >= G.dim) return fail(HJ_EINVAL, "axis %d out of range for dim %d", axis, G.dim);
  if (eps_mode != HJ_EPS_SQUARED && eps_mode != HJ_EPS_RAW) return fail(HJ_EINVAL, "eps_mode must be 'squared' or 'raw'");
  if (!v || !left || !right) return fail(HJ_EINVAL, "NULL field pointer");
  return cuda_status(launch_derivs(scheme, G, axis, eps_mode, v, left, right, (cudaStream_t)stream), "hj_derivs");
}

int hj_weno5_workspace(const hj_grid* g, int axis, int side, int eps_mode, const double* v, double* ws,
                       void* stream) {
  GridArgs G;
  int rc = make_grid(g, 3, &G, 1u << (axis & 7));
  if (rc) return rc;
  if (axis < 0 || axis >= G.dim) return fail(HJ_EINVAL, "axis %d out of range for dim %d", axis, G.dim);
  if (side != 0 && side != 1) return fail(HJ_EINVAL, "side must be 'left' or 'right'");
  if (eps_mode != HJ_EPS_SQUARED && eps_mode != HJ_EPS_RAW) return fail(HJ_EINVAL, "eps_mode must be 'squared' or 'raw'");
  if (G.batch != 1 || g->halo_lo || g->halo_hi) return fail(HJ_EINVAL, "workspace takes one un-haloed field");
  return cuda_status(launch_weno_ws(G, axis, side, eps_mode, v, ws, (cudaStream_t)stream), "hj_weno5_workspace");
}

// Axis-0 rows of a stage launch.  part 0: every row; 1 (core): the rows whose
// stencils read no exchanged halo plane (halo_lo / halo_hi), so they can run
// while the exchange is in flight; 2 (rim): the rest.  unit = planes per row
// (8 for the 3-D brick rows, 8 for the 4-D pre-pass segments, 1 for planes);
// a row r covers planes [r*unit, r*unit+unit) and reads `reach` planes
// further on each side.
constexpr int STAGE_PLANES = 3;   // internal: an explicit plane range (hj_stage_planes)
// internal: the two halves of a per-axis-pipeline slab stage (hj_dd_stage):
// the contiguous-axis kernel (reads no exchanged plane), then the column kernels
constexpr int STAGE_AXES_X = 4, STAGE_AXES_REST = 5;

static RowSet row_set(int n0, int unit, int reach, int halo_lo, int halo_hi, int part) {
  const int nrows = (n0 + unit - 1) / unit;
  RowSet R{0, nrows, nrows, nrows};
  if (part == HJ_PART_ALL) return R;
  int lo = 0, hi = nrows;                                   // core rows [lo, hi)
  if (halo_lo) lo = (reach + unit - 1) / unit;              // first row with r*unit >= reach
  if (halo_hi) hi = (n0 - reach - unit) >= 0 ? (n0 - reach - unit) / unit + 1 : 0;   // r*unit+unit+reach <= n0
  if (hi < lo) hi = lo;
  if (part == HJ_PART_CORE) return RowSet{lo, hi - lo, hi, hi - lo};
  return RowSet{0, lo, hi, lo + (nrows - hi)};              // HJ_PART_RIM
}

static void set_rows(StageArgs& P, int w, int part, int64_t plo = 0, int64_t phi = 0) {
  const GridArgs& G = P.g;
  if (part == STAGE_PLANES) {   // explicit plane range [plo, phi), validated by the caller
    const int r0 = (int)(plo / 8), r1 = (int)((phi + 7) / 8);
    P.zr = RowSet{r0, r1 - r0, r1, r1 - r0};
    P.zp = RowSet{(int)plo, (int)(phi - plo), (int)phi, (int)(phi - plo)};
    return;
  }
  const int hl = G.ax[0].halo_lo, hh = G.ax[0].halo_hi;
  // the brick rows (3-D) and pre-pass segments (4-D) are both 8 planes deep;
  // the per-node kernel and the 4-D brick slices work per plane
  P.zr = row_set(G.n[0], 8, w, hl, hh, part);
  const RowSet& r = P.zr;
  // planes covered by those rows (clipped to the slab)
  auto clip = [&](int row) { return row * 8 < G.n[0] ? row * 8 : G.n[0]; };
  const int a0 = clip(r.lo), a1 = clip(r.lo + r.split), b0 = clip(r.hs), b1 = clip(r.hs + (r.cnt - r.split));
  P.zp = RowSet{a0, a1 - a0, b0, (a1 - a0) + (b1 - b0)};
}

static int stage_impl(const hj_grid* g, int scheme, const hj_ham* ham, const double* alpha, double dt, int stage,
                      const double* y_in, const double* y0, double* y_out, const double* mask_prev, int mask,
                      hj_stats* stats, int32_t tag, int part, int64_t plo, int64_t phi, void* stream,
                      StageArgs* build_only = nullptr) {
  const int w = ghost_width_of(scheme);
  if (w < 0) return fail(HJ_EINVAL, "unknown derivative scheme %d", scheme);
  StageArgs P;
  std::memset(&P, 0, sizeof P);
  int rc = make_grid(g, w, &P.g);
  if (rc) return rc;
  if (part == STAGE_PLANES) {
    const int64_t n0 = P.g.n[0];
    if (plo < 0 || phi > n0 || plo > phi || plo % 8 != 0 || (phi % 8 != 0 && phi != n0))
      return fail(HJ_EINVAL, "plane range [%lld, %lld) must lie in [0, %lld) on multiples of 8 (or end at n[0])",
                  (long long)plo, (long long)phi, (long long)n0);
    if (plo == phi) return HJ_OK;
  }
  const bool axes_split = part == STAGE_AXES_X || part == STAGE_AXES_REST;
  set_rows(P, w, axes_split ? HJ_PART_ALL : part, plo, phi);
  rc = check_ham(ham, P.g.dim);
  if (rc) return rc;
  if (!alpha) return fail(HJ_EINVAL, "alpha is NULL");
  for (int a = 0; a < P.g.dim; ++a) {
    if (!(alpha[a] >= 0.0) || alpha[a] == INFINITY)
      return fail(HJ_EINVAL, "partials returned invalid bound %g for axis %d", alpha[a], a);
    P.alpha_half[a] = alpha[a] * 0.5;
  }
  if (stage < HJ_STAGE_DELTA || stage > HJ_STAGE_RK3_THIRD) return fail(HJ_EINVAL, "unknown stage kind %d", stage);
  if (!y_in || !y_out) return fail(HJ_EINVAL, "NULL field pointer");
  if (y_in == y_out) return fail(HJ_EINVAL, "y_out must not alias y_in");
  if (stage >= HJ_STAGE_RK2_AVG && !y0) return fail(HJ_EINVAL, "stage %d needs y0", stage);
  if (mask != HJ_MASK_NONE && !mask_prev) return fail(HJ_EINVAL, "mask needs the previous snapshot");
  if (mask < HJ_MASK_NONE || mask > HJ_MASK_MAX) return fail(HJ_EINVAL, "unknown mask %d", mask);
  P.ham = prep_ham(ham);
  P.dt = dt;
  P.stage = stage;
  P.mask = mask;
  P.eps_mode = HJ_EPS_SQUARED;  // derivative_pair passes no eps_mode (spatial.py:276)
  P.want_ranges = 0;
  P.want_hnz = stats && all_zero(alpha, P.g.dim);
  P.tag = tag;
  P.y_in = y_in;
  P.y0 = y0;
  P.y_out = y_out;
  P.mask_prev = mask_prev;
  P.stats = stats;
  if (build_only) {   // validated arguments for a caller that launches itself (hj_integrate)
    *build_only = P;
    return HJ_OK;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const size_t span = (size_t)(P.g.batch_stride * (P.g.batch - 1) + P.g.cells);
  if (axes_split) {
    // one half of a slab stage on the per-axis walk pipeline (same stream, so
    // the same scratch for both halves)
    if (!axes_applies(scheme, P, true)) return fail(HJ_EINVAL, "stage does not run the per-axis walk pipeline");
    P.aux0 = scratch_for(s, axes_scratch_doubles(P.g.dim, span));
    if (!P.aux0) return fail(HJ_ECUDA, "no scratch for the per-axis walk pipeline");
    set_extents(P, g);
    bool handled = false;
    cudaError_t e = launch_axes_weno5(P, s, &handled, part == STAGE_AXES_X ? 1 : 2);
    return cuda_status(e, "hj_stage (per-axis pipeline)", part == STAGE_AXES_X ? 1 : (uint64_t)(P.g.dim - 1));
  }
  const bool axes = axes_applies(scheme, P, false);
  if (axes) {
    // per-axis walk pipeline (hj_axes.cuh): 2 (dim - 1) field-sized scratch arrays
    P.aux0 = scratch_for(s, axes_scratch_doubles(P.g.dim, span));
  } else if (P.g.dim == 4) {
    // 4-D brick path: scratch for the axis-0 pre-pass (p_avg0, d0)
    double* scratch = scratch_for(s, 2 * span);
    if (scratch) {
      P.aux0 = scratch;   // span (p_avg0, d0) pairs
    }
  }
  set_extents(P, g);
  bool handled = false;
  cudaError_t e = launch_stage_fast(scheme, P, s, &handled);
  if (!handled) e = launch_stage_generic(scheme, P, s);
  // kernels launched: one per axis (per-axis walk pipeline), pre-pass + brick (4-D bricks), else one
  const uint64_t nl = (handled && axes && P.aux0) ? (uint64_t)P.g.dim : (handled && P.g.dim == 4 && P.aux0) ? 2 : 1;
  return cuda_status(e, "hj_stage", nl);
}

int hj_stage_part(const hj_grid* g, int scheme, const hj_ham* ham, const double* alpha, double dt, int stage,
                  const double* y_in, const double* y0, double* y_out, const double* mask_prev, int mask,
                  hj_stats* stats, int32_t tag, int part, void* stream) {
  if (part < HJ_PART_ALL || part > HJ_PART_RIM) return fail(HJ_EINVAL, "unknown stage part %d", part);
  return stage_impl(g, scheme, ham, alpha, dt, stage, y_in, y0, y_out, mask_prev, mask, stats, tag, part, 0, 0,
                    stream);
}

int hj_stage_planes(const hj_grid* g, int scheme, const hj_ham* ham, const double* alpha, double dt, int stage,
                    const double* y_in, const double* y0, double* y_out, const double* mask_prev, int mask,
                    hj_stats* stats, int32_t tag, int64_t plane_lo, int64_t plane_hi, void* stream) {
  return stage_impl(g, scheme, ham, alpha, dt, stage, y_in, y0, y_out, mask_prev, mask, stats, tag, STAGE_PLANES,
                    plane_lo, plane_hi, stream);
}

int hj_stage(const hj_grid* g, int scheme, const hj_ham* ham, const double* alpha, double dt, int stage,
             const double* y_in, const double* y0, double* y_out, const double* mask_prev, int mask,
             hj_stats* stats, int32_t tag, void* stream) {
  return stage_impl(g, scheme, ham, alpha, dt, stage, y_in, y0, y_out, mask_prev, mask, stats, tag, HJ_PART_ALL,
                    0, 0, stream);
}

int hj_term(const hj_grid* g, int scheme, const hj_ham* ham, const double* alpha, const double* v,
            double* delta, hj_stats* stats, void* stream) {
  const int w = ghost_width_of(scheme);
  if (w < 0) return fail(HJ_EINVAL, "unknown derivative scheme %d", scheme);
  StageArgs P;
  std::memset(&P, 0, sizeof P);
  int rc = make_grid(g, w, &P.g);
  if (rc) return rc;
  set_rows(P, w, HJ_PART_ALL);
  rc = check_ham(ham, P.g.dim);
  if (rc) return rc;
  if (!alpha) return fail(HJ_EINVAL, "alpha is NULL");
  for (int a = 0; a < P.g.dim; ++a) {
    if (!(alpha[a] >= 0.0) || alpha[a] == INFINITY)
      return fail(HJ_EINVAL, "partials returned invalid bound %g for axis %d", alpha[a], a);
    P.alpha_half[a] = alpha[a] * 0.5;
  }
  if (!v || !delta) return fail(HJ_EINVAL, "NULL field pointer");
  if (v == delta) return fail(HJ_EINVAL, "delta must not alias v");
  P.ham = prep_ham(ham);
  P.stage = HJ_STAGE_DELTA;
  P.eps_mode = HJ_EPS_SQUARED;
  P.want_ranges = stats ? 1 : 0;
  P.want_hnz = stats && all_zero(alpha, P.g.dim);
  P.tag = 0;
  P.y_in = v;
  P.y_out = delta;
  P.stats = stats;
  set_extents(P, g);
  return cuda_status(launch_stage_generic(scheme, P, (cudaStream_t)stream), "hj_term");
}

int hj_costates(const hj_grid* g, const double* const* left, const double* const* right, double* const* p_avg,
                hj_stats* stats, void* stream) {
  GridArgs G;
  int rc = make_grid(g, 0, &G);
  if (rc) return rc;
  if (!left || !right || !p_avg) return fail(HJ_EINVAL, "NULL pointer array");
  for (int a = 0; a < G.dim; ++a)
    if (!left[a] || !right[a] || !p_avg[a]) return fail(HJ_EINVAL, "NULL field pointer for axis %d", a);
  return cuda_status(launch_costates(G, left, right, p_avg, stats, (cudaStream_t)stream), "hj_costates");
}

int hj_glf_delta(const hj_grid* g, const double* alpha, const double* const* left, const double* const* right,
                 const double* ham, double* diss, double* delta, hj_stats* stats, void* stream) {
  GridArgs G;
  int rc = make_grid(g, 0, &G);
  if (rc) return rc;
  if (!alpha || !left || !right || !ham || !delta) return fail(HJ_EINVAL, "NULL pointer");
  double ahalf[HJ_MAX_DIM];
  for (int a = 0; a < G.dim; ++a) {
    if (!(alpha[a] >= 0.0) || alpha[a] == INFINITY)
      return fail(HJ_EINVAL, "partials returned invalid bound %g for axis %d", alpha[a], a);
    ahalf[a] = alpha[a] * 0.5;
    if (!left[a] || !right[a]) return fail(HJ_EINVAL, "NULL field pointer for axis %d", a);
  }
  return cuda_status(launch_glf_delta(G, ahalf, left, right, ham, diss, delta, stats, (cudaStream_t)stream),
                     "hj_glf_delta");
}

int hj_rk_combine(int64_t count, int stage, double dt, const double* y_in, const double* y0, const double* delta,
                  double* out, hj_stats* stats, int32_t tag, void* stream) {
  if (count < 0) return fail(HJ_EINVAL, "negative count");
  if (stage < HJ_STAGE_EULER || stage > HJ_STAGE_RK3_THIRD) return fail(HJ_EINVAL, "unknown stage kind %d", stage);
  if (!y_in || !delta || !out) return fail(HJ_EINVAL, "NULL field pointer");
  if (stage >= HJ_STAGE_RK2_AVG && !y0) return fail(HJ_EINVAL, "stage %d needs y0", stage);
  if (count == 0) return HJ_OK;
  return cuda_status(launch_rk_combine(count, stage, dt, y_in, y0, delta, out, stats, tag, (cudaStream_t)stream),
                     "hj_rk_combine");
}

int hj_init_shape(const hj_grid* g, int kind, const double* params, int nparams, double* out, void* stream) {
  GridArgs G;
  int rc = make_grid(g, 0, &G);
  if (rc) return rc;
  int need;
  switch (kind) {
    case HJ_SHAPE_SPHERE: need = G.dim + 1; break;
    case HJ_SHAPE_CYLINDER: need = G.dim + 2; break;
    case HJ_SHAPE_ELLIPSOID: need = G.dim + 1; break;
    case HJ_SHAPE_BOX: need = 2 * G.dim; break;
    default: return fail(HJ_EINVAL, "unknown shape kind %d", kind);
  }
  if (!params || nparams != need) return fail(HJ_EINVAL, "shape %d needs %d params, got %d", kind, need, nparams);
  for (int a = 0; a < G.dim; ++a)
    if (!G.nodes[a]) return fail(HJ_EINVAL, "axis %d: node table missing", a);
  if (!out) return fail(HJ_EINVAL, "NULL output");
  cudaError_t e = launch_shape(G, kind, params, nparams, out, (cudaStream_t)stream);
  return cuda_status(e, "hj_init_shape");
}

int hj_csg(int op, int64_t count, const double* a, const double* b, double* out, void* stream) {
  if (op < HJ_CSG_UNION || op > HJ_CSG_DIFFERENCE) return fail(HJ_EINVAL, "unknown csg op %d", op);
  if (!a || !out || (op != HJ_CSG_COMPLEMENT && !b)) return fail(HJ_EINVAL, "NULL field pointer");
  if (count <= 0) return HJ_OK;
  return cuda_status(launch_csg(op, count, a, b, out, (cudaStream_t)stream), "hj_csg");
}

int hj_mask(int64_t count, const double* prev, double* v, int mask, void* stream) {
  if (mask != HJ_MASK_MIN && mask != HJ_MASK_MAX) return fail(HJ_EINVAL, "unknown mask %d", mask);
  if (!prev || !v) return fail(HJ_EINVAL, "NULL field pointer");
  if (count <= 0) return HJ_OK;
  return cuda_status(launch_mask(count, prev, v, mask, (cudaStream_t)stream), "hj_mask");
}

int hj_count_below(int64_t count, const double* v, double level, unsigned long long* d_count, void* stream) {
  if (!v || !d_count) return fail(HJ_EINVAL, "NULL pointer");
  if (count <= 0) return HJ_OK;
  return cuda_status(launch_count_below(count, v, level, d_count, (cudaStream_t)stream), "hj_count_below");
}

int hj_tube_check(int64_t count, const double* prev, const double* v, const double* target, int mask, double level,
                  unsigned long long* d_out, void* stream) {
  if (mask != HJ_MASK_MIN && mask != HJ_MASK_MAX) return fail(HJ_EINVAL, "unknown mask %d", mask);
  if (!prev || !v || !target || !d_out) return fail(HJ_EINVAL, "NULL pointer");
  if (count <= 0) return HJ_OK;
  return cuda_status(launch_tube_check(count, prev, v, target, mask == HJ_MASK_MIN, level, d_out,
                                       (cudaStream_t)stream), "hj_tube_check");
}

int hj_check_division(int64_t n, uint64_t seed, unsigned long long* d_mismatch, void* stream) {
  if (!d_mismatch || n < 0) return fail(HJ_EINVAL, "bad arguments");
  return cuda_status(launch_check_division(n, seed, d_mismatch, (cudaStream_t)stream), "hj_check_division");
}

int hj_fp64_probe(int iters, int blocks, double* d_sink, void* stream) {
  if (iters < 1 || blocks < 1 || !d_sink) return fail(HJ_EINVAL, "bad arguments");
  return cuda_status(launch_fp64_probe(iters, blocks, d_sink, (cudaStream_t)stream), "hj_fp64_probe");
}

int64_t hj_bounds_violations(void) {
#ifdef HJ_CHECK_BOUNDS
  unsigned long long* c = oob_counter();
  if (!c) return fail(HJ_ECUDA, "bounds counter unavailable");
  unsigned long long n = 0;
  cudaDeviceSynchronize();
  cudaMemcpy(&n, c, sizeof n, cudaMemcpyDeviceToHost);
  cudaMemset(c, 0, sizeof n);
  return (int64_t)n;
#else
  return -1;
#endif
}

int hj_stats_reset(hj_stats* stats, void* stream) {
  if (!stats) return fail(HJ_EINVAL, "NULL stats");
  return cuda_status(launch_stats_reset(stats, (cudaStream_t)stream), "hj_stats_reset");
}

int hj_eval_hamiltonian(const hj_grid* g, const hj_ham* ham, const double* const* p, double* out, void* stream) {
  GridArgs G;
  int rc = make_grid(g, 0, &G);
  if (rc) return rc;
  rc = check_ham(ham, G.dim);
  if (rc) return rc;
  if (!p || !out) return fail(HJ_EINVAL, "NULL pointer");
  for (int a = 0; a < G.dim; ++a)
    if (!p[a]) return fail(HJ_EINVAL, "NULL costate field for axis %d", a);
  const hj_ham h = prep_ham(ham);
  return cuda_status(launch_eval_ham(G, h, p, out, (cudaStream_t)stream), "hj_eval_hamiltonian");
}

int hj_divided_differences(const hj_grid* g, int axis, int width, int order, const double* v, double* d0,
                           double* d1, double* d2, double* d3, void* stream) {
  if (order < 1 || order > 3) return fail(HJ_EINVAL, "order must be 1..3, got %d", order);
  if (width < 1) return fail(HJ_EINVAL, "ghost width must be >= 1, got %d", width);
  GridArgs G;
  int rc = make_grid(g, width, &G, 1u << (axis & 7));
  if (rc) return rc;
  if (axis < 0 || axis >= G.dim) return fail(HJ_EINVAL, "axis %d out of range for dim %d", axis, G.dim);
  if (G.batch != 1 || g->halo_lo || g->halo_hi) return fail(HJ_EINVAL, "divided_differences takes one un-haloed field");
  if (!v || !d0 || !d1 || (order >= 2 && !d2) || (order >= 3 && !d3)) return fail(HJ_EINVAL, "NULL table pointer");
  if (G.n[axis] + 2 * width - order < 1) return fail(HJ_EINVAL, "axis %d too short for order %d", axis, order);
  return cuda_status(launch_divdiff(G, axis, width, order, v, d0, d1, d2, d3, (cudaStream_t)stream),
                     "hj_divided_differences");
}

}  // extern "C"

namespace hj {
// a slab stage on the per-axis walk pipeline, around its halo exchange
// (hj_dd_stage): axes_slab_applies says whether it runs there, then
// stage_axes_part(.., 1) launches the contiguous-axis kernel and
// stage_axes_part(.., 2) the column kernels
bool axes_slab_applies(const hj_grid* g, int scheme, const hj_ham* ham, const double* alpha, int stage,
                       const double* y_in, const double* y0, double* y_out) {
  StageArgs P;
  if (stage_impl(g, scheme, ham, alpha, 0.0, stage, y_in, y0, y_out, nullptr, HJ_MASK_NONE, nullptr, 0,
                 HJ_PART_ALL, 0, 0, nullptr, &P))
    return false;
  return axes_applies(scheme, P, true);
}
int stage_axes_part(const hj_grid* g, int scheme, const hj_ham* ham, const double* alpha, double dt, int stage,
                    const double* y_in, const double* y0, double* y_out, const double* mask_prev, int mask,
                    hj_stats* stats, int32_t tag, int which, void* stream) {
  return stage_impl(g, scheme, ham, alpha, dt, stage, y_in, y0, y_out, mask_prev, mask, stats, tag,
                    which == 1 ? STAGE_AXES_X : STAGE_AXES_REST, 0, 0, stream);
}

// hj_stage's validation and argument build without the launch
int stage_args(const hj_grid* g, int scheme, const hj_ham* ham, const double* alpha, double dt, int stage,
               const double* y_in, const double* y0, double* y_out, const double* mask_prev, int mask,
               hj_stats* stats, int32_t tag, StageArgs* P) {
  return stage_impl(g, scheme, ham, alpha, dt, stage, y_in, y0, y_out, mask_prev, mask, stats, tag, HJ_PART_ALL,
                    0, 0, nullptr, P);
}
}  // namespace hj

