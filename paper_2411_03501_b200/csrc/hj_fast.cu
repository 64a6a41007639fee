// hj_fast.cu -- routing of fused stages to the brick-tiled kernels.
#include <cstdlib>
#include <string>
#include "hj_kernels.cuh"

namespace hj {
cudaError_t launch_brick_weno5(const StageArgs& P, cudaStream_t s, bool* handled, int variant);
cudaError_t launch_brick_eno(int scheme, const StageArgs& P, cudaStream_t s, bool* handled);
cudaError_t launch_brick_weno5_fma(const StageArgs& P, cudaStream_t s, bool* handled, int variant);
cudaError_t launch_tile(int scheme, const StageArgs& P, cudaStream_t s, bool* handled);
cudaError_t launch_axes_weno5(const StageArgs& P, cudaStream_t s, bool* handled, int parts);

// HJ_STAGE_KERNEL selects the stage kernel for A/B measurements:
//   unset / "brick" : brick-tiled kernels, 2 CTAs per SM (default)
//   "brick1"        : brick-tiled WENO5 kernel compiled for 1 CTA per SM
//   "generic"       : per-node generic kernel everywhere
// process-wide A/B switch (set by hj_set_stage_kernel / HJ_STAGE_KERNEL);
// atomic, read once per launch
static std::atomic<int> g_variant{-1};   // -1: take HJ_STAGE_KERNEL from the environment

static int stage_variant() {
  if (g_variant.load(std::memory_order_relaxed) < 0) {
    const char* e = std::getenv("HJ_STAGE_KERNEL");
    int v = 1;
    if (e && std::string(e) == "generic") v = 0;
    if (e && std::string(e) == "brick1") v = 2;
    if (e && std::string(e) == "brick_always") v = 3;   // brick kernels even on tiny grids
    if (e && std::string(e) == "brick_u2") v = 4;       // WENO5 walks unrolled by 2
    if (e && std::string(e) == "brick_noload") v = 5;   // A/B bound: tiles loaded once per CTA (wrong results)
    if (e && std::string(e) == "brick_nopf") v = 6;     // A/B: no L2 prefetch of the next brick
    if (e && std::string(e) == "brick_x") v = 7;        // A/B slot (hj_brick_weno.cu: the variant under test)
    if (e && std::string(e) == "tile_stages") v = 8;    // small 3-D grids: tile kernel per stage, no persistent launch
    if (e && std::string(e) == "axes") v = 9;           // brick-sized WENO5 grids: the per-axis walk pipeline
    if (e && std::string(e) == "axes_r1") v = 10;       // per-axis A/B: every walk rolled (the r02g pipeline)
    if (e && std::string(e) == "axes_u2x") v = 11;      //  ... the contiguous-axis walk unrolled as well
    if (e && std::string(e) == "axes_l32") v = 12;      //  ... the last-axis kernel on 32-node segments
    if (e && std::string(e) == "axes_s16") v = 13;      //  ... column kernels on 16-node segments
    int expect = -1;
    g_variant.compare_exchange_strong(expect, v);
  }
  return g_variant.load(std::memory_order_relaxed);
}

// walk unroll of the per-axis pipeline (launch_axes_t's WU bits)
int axes_unroll() {
  switch (stage_variant()) {
    case 10: return 0;
    case 11: return 5;
    case 12: return 20;
    case 13: return 64;
    default: return -1;
  }
}

int set_stage_variant(int v) {
  const int old = stage_variant();
  g_variant.store(v);
  return old;
}

// The brick kernels cover 3-D stages without range statistics whose grid
// fits the launch geometry; everything else runs the generic per-node kernel.
// The per-axis walk pipeline (hj_axes.cuh) covers whole-grid WENO5 launches
// of 3-D / 4-D grids (no exchanged halos, contiguous batches, no range
// statistics) -- by default those of brick size (measured faster than the
// brick kernels at 301^3, 121^4 and 8 x 101^3: DESIGN.md); "axes" forces it
// on every size (tests).  It needs 2 (dim - 1) field-sized scratch arrays.
// allow_halo: a multi-GPU slab stage split around its halo exchange
// (hj_dd_stage: the contiguous-axis kernel overlaps the exchange; only the
// axis-0 walk reads exchanged planes).
bool axes_applies(int scheme, const StageArgs& P, bool allow_halo) {
  const int v = stage_variant();
  if ((v != 1 && v != 9 && v < 10) || scheme != HJ_WENO5) return false;
  if ((P.g.dim != 3 && P.g.dim != 4) || P.want_ranges) return false;
  if (!allow_halo && (P.g.ax[0].halo_lo || P.g.ax[0].halo_hi)) return false;
  if (P.zp.lo != 0 || P.zp.cnt != P.g.n[0]) return false;
  if (P.g.batch > 1 && P.g.batch_stride != P.g.cells) return false;
  bool ham_ok = false;
  switch (P.ham.kind) {
    case HJ_HAM_ADVECTION: ham_ok = true; break;
    case HJ_HAM_AIR3D: case HJ_HAM_ROCKETS: case HJ_HAM_ROCKETS_EXTREMAL: ham_ok = P.g.dim == 3; break;
    case HJ_HAM_DI4: ham_ok = P.g.dim == 4; break;
    default: ham_ok = false;
  }
  if (!ham_ok) return false;
  if (v == 9) return true;
  const int ao = P.g.dim - 3;   // default: where the brick kernels would run
  const long long nbricks = (long long)((P.g.n[ao + 2] + 15) / 16) * ((P.g.n[ao + 1] + 15) / 16) *
                            ((P.g.n[ao] + 7) / 8) * (ao ? (long long)P.g.n[0] : 1) * P.g.batch;
  int dev = 0;
  cudaGetDevice(&dev);
  return nbricks >= 2LL * sm_count(dev);
}

cudaError_t launch_stage_fast(int scheme, const StageArgs& P, cudaStream_t s, bool* handled) {
  *handled = false;
  const int variant = stage_variant();
  if (P.aux0 && axes_applies(scheme, P, false)) return launch_axes_weno5(P, s, handled, 3);
  if (variant == 0 || (P.g.dim != 3 && P.g.dim != 4) || P.want_ranges) return cudaSuccess;
  // too few bricks to occupy the SMs (small grids such as C1's 51x51x36):
  // the per-node kernel exposes more parallelism
  const int ao = P.g.dim - 3;
  const long long nbricks = (long long)((P.g.n[ao + 2] + 15) / 16) * ((P.g.n[ao + 1] + 15) / 16) *
                            ((P.g.n[ao] + 7) / 8) * (ao ? (long long)P.g.n[0] : 1) * P.g.batch;
  int dev = 0;
  cudaGetDevice(&dev);
  const int nsm = sm_count(dev);
  if (variant != 3 && variant != 5 && nbricks < 2LL * nsm) {
    // small 3-D grids: the tile kernel (one node per thread, stencils from
    // shared memory); the per-node generic kernel for the rest
    if ((variant == 1 || variant == 8) && P.g.dim == 3) return launch_tile(scheme, P, s, handled);
    return cudaSuccess;
  }
  if (variant == 6) {
    StageArgs Q = P;
    Q.no_prefetch = 1;
    if (scheme == HJ_WENO5) return launch_brick_weno5(Q, s, handled, 1);
    if (scheme == HJ_WENO5_FMA) return launch_brick_weno5_fma(Q, s, handled, 1);
    return launch_brick_eno(scheme, Q, s, handled);
  }
  if (variant == 5) {
    // upper bound of any load-phase optimisation (TMA staging included):
    // every brick after a CTA's first skips its global -> shared loads
    StageArgs Q = P;
    Q.skip_loads = 1;
    if (scheme == HJ_WENO5) return launch_brick_weno5(Q, s, handled, 1);
    return cudaSuccess;
  }
  if (scheme == HJ_WENO5) return launch_brick_weno5(P, s, handled, variant);
  if (scheme == HJ_WENO5_FMA) return launch_brick_weno5_fma(P, s, handled, variant);
  return launch_brick_eno(scheme, P, s, handled);
}
}  // namespace hj

namespace hj {
// hj_integrate runs an interval's stage sequence as one persistent launch
// (hj_stage_generic.cuh k_stage_persist) where the per-stage kernel would be
// the generic one anyway: the default dispatch, grids below the brick
// kernels' size (fewer bricks than 2 per SM; any 1-D/2-D grid), no range
// statistics, at most 2^22 nodes.
bool persist_applies(const StageArgs& P) {
  if (stage_variant() != 1 || P.want_ranges) return false;
  const long long total = P.g.cells * P.g.batch;
  if (total > (1LL << 22)) return false;
  if (P.g.dim == 3 || P.g.dim == 4) {
    const int ao = P.g.dim - 3;
    const long long nbricks = (long long)((P.g.n[ao + 2] + 15) / 16) * ((P.g.n[ao + 1] + 15) / 16) *
                              ((P.g.n[ao] + 7) / 8) * (ao ? (long long)P.g.n[0] : 1) * P.g.batch;
    int dev = 0;
    cudaGetDevice(&dev);
    if (nbricks >= 2LL * sm_count(dev)) return false;
  }
  return true;
}
}  // namespace hj

extern "C" int hj_set_stage_kernel(int variant) {
  if (variant < -1 || variant > 13) return -1;
  return hj::set_stage_variant(variant);
}
