// hj_kernels.cuh -- kernel argument blocks shared by the .cu translation units.
#pragma once
#include <atomic>
#include <cstdio>
#include <cuda_runtime.h>
#include "hj_ham.cuh"

namespace hj {

// Device view of hj_grid: owned extents, element strides, per-axis ghost rules.
struct GridArgs {
  int dim;
  int batch;
  int n[HJ_MAX_DIM];
  long long stride[HJ_MAX_DIM];
  long long batch_stride;
  long long cells;        // owned nodes of one problem
  AxisView ax[HJ_MAX_DIM];
  Spacing sp[HJ_MAX_DIM];
  const double* nodes[HJ_MAX_DIM];
};

// A subset of axis-0 rows (bricks rows, pre-pass segments or single planes):
// rows lo .. lo+split-1, then hs .. hs+(cnt-split)-1 (hj_stage_part splits).
struct RowSet {
  int lo, split, hs, cnt;
  __host__ __device__ __forceinline__ int map(int k) const { return k < split ? lo + k : hs + (k - split); }
  __host__ __device__ __forceinline__ bool has(int r) const {
    return (r >= lo && r < lo + split) || (r >= hs && r < hs + (cnt - split));
  }
};

// Bounds checking (builds with -DHJ_CHECK_BOUNDS, libhjb200_check.so): the
// extent of every field a stage kernel touches; each global access is tested
// against it and violations are counted in device memory (hj_bounds_violations).
// compute-sanitizer is closed on this pool, this is its replacement.
struct Extent {
  const void* lo;
  const void* hi;
};
struct BoundsCheck {
  Extent in, y0, out, mask, aux;
  unsigned long long* oob;   // device counter; NULL in normal builds
};

struct StageArgs {
  GridArgs g;
  RowSet zr;        // axis-0 brick rows (3-D brick) / pre-pass segments (4-D) of this launch
  RowSet zp;        // axis-0 planes of this launch (per-node kernel, 4-D brick slices)
  hj_ham ham;
  double alpha_half[HJ_MAX_DIM];  // alphas[i] * 0.5 (term.py:86)
  double dt;
  int stage;
  int mask;
  int eps_mode;
  int want_ranges;
  int want_hnz;       // record HJ_FLAG_HAM_NONZERO (only needed when every alpha is 0)
  int tag;
  int skip_loads;     // A/B only (stage kernel "brick_noload"): bricks after a CTA's first reuse its shared tiles
  int no_prefetch;    // A/B only (stage kernel "brick_nopf"): no L2 prefetch of the next brick
  const double* y_in;
  const double* y0;
  double* y_out;
  const double* mask_prev;
  hj_stats* stats;
  double* aux0;     // 4-D brick path: (p_avg0, d0) pairs per node from the axis-0 pre-pass
                    // (interleaved: one 16-B load per node in the fused walk)
  BoundsCheck bc;
};

// Stage sequence of one persistent launch (hj_integrate -> k_stage_persist,
// hj_stage_generic.cuh)
struct PersistStage {
  double dt;
  int32_t tag;
  int8_t src, y0, dst;   // buffer ids: 0 = the initial state (read only), 1..3 = work buffers; y0 -1: none
  int8_t kind;           // HJ_STAGE_*
  int8_t mask;           // HJ_MASK_* applied to this stage's output
  int8_t pad[7];
};
constexpr int PERSIST_MAX_STAGES = 1024;
struct PersistArgs {
  const double* buf[4];
  const double* mask_prev;
  unsigned* bar;         // grid barrier words (BAR_WORDS, hj_stage_generic.cuh), zeroed by the launcher
  int nstages;
  PersistStage st[PERSIST_MAX_STAGES];
};

// doubles of device scratch the per-axis walk pipeline (hj_axes.cuh) needs
// for a field of `span` nodes: 16-byte records (PX, DX) and (P_a, D_a),
// a = 0 .. dim-3
__host__ __device__ constexpr size_t axes_scratch_doubles(int dim, size_t span) {
  return (size_t)2 * (size_t)(dim - 1) * span;
}

#ifdef HJ_CHECK_BOUNDS
__device__ __forceinline__ void chk_extent(const BoundsCheck& b, const Extent& e, const void* p, int bytes,
                                           const char* what, const char* file, int line) {
  if (b.oob && (p < e.lo || (const char*)p + bytes > (const char*)e.hi)) {
    if (atomicAdd(b.oob, 1ull) < 8)
      printf("hj bounds: %s at %s:%d ptr %p outside [%p, %p)\n", what, file, line, p, e.lo, e.hi);
  }
}
#define HJ_CHK(P, which, ptr, bytes) ::hj::chk_extent((P).bc, (P).bc.which, (const void*)(ptr), (bytes), #which, __FILE__, __LINE__)
#else
#define HJ_CHK(P, which, ptr, bytes) ((void)0)
#endif

// Split a linear owned-node index into (problem, per-axis indices) and the
// element offset of that node from the problem-0 base pointer.
__device__ __forceinline__ long long locate(const GridArgs& g, long long idx, int* ix) {
  if (idx < (1LL << 31)) {
    // 32-bit index arithmetic (a 64-bit division is ~100 instructions; small
    // grids are instruction-bound on exactly this)
    unsigned rem = (unsigned)idx;
    long long off = 0;
    for (int a = g.dim - 1; a >= 0; --a) {
      const unsigned q = rem / (unsigned)g.n[a];
      ix[a] = (int)(rem - q * (unsigned)g.n[a]);
      off += (long long)ix[a] * g.stride[a];
      rem = q;
    }
    return off + (long long)rem * g.batch_stride;
  }
  long long rem = idx;
  long long off = 0;
  for (int a = g.dim - 1; a >= 0; --a) {
    const long long q = rem / g.n[a];
    ix[a] = (int)(rem - q * g.n[a]);
    off += (long long)ix[a] * g.stride[a];
    rem = q;
  }
  return off + rem * g.batch_stride;
}

// Block-wide reduction of the non-finite flags and optional costate ranges
// into the device hj_stats (one atomic per block and quantity).
// Error class of a node's flags in the order the reference would raise them
// (input field, derivative fields, H, delta, output field); 7 = no error.
__device__ __forceinline__ int error_code(unsigned flags) {
  if (flags & HJ_NF_INPUT) return 1;
  if (flags & HJ_NF_DERIV) return 2;
  if (flags & HJ_NF_HAM) return 3;
  if (flags & HJ_NF_DELTA) return 4;
  if (flags & HJ_NF_OUTPUT) return 5;
  return 7;
}

// first_bad_tag keeps min(tag*8 + error_code) over every failing node, so the
// host recovers the first failing stage AND the error it would have raised.
template <int DIM>
__device__ __forceinline__ void reduce_stats(hj_stats* st, unsigned flags, int tag, bool want_ranges,
                                             long long* lo, long long* hi) {
  const unsigned any = __any_sync(0xffffffffu, flags != 0u);
  if (any) {
    unsigned f = flags;
    int key = (flags & 31u) ? tag * 8 + error_code(flags) : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      f |= __shfl_xor_sync(0xffffffffu, f, o);
      key = min(key, __shfl_xor_sync(0xffffffffu, key, o));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicOr(&st->nonfinite, f);
      if (key != 0x7fffffff) atomicMin(&st->first_bad_tag, key);
    }
  }
  if (!want_ranges) return;
  __shared__ long long s_lo[HJ_MAX_DIM][32];
  __shared__ long long s_hi[HJ_MAX_DIM][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    long long l = lo[a], h = hi[a];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      l = min(l, __shfl_xor_sync(0xffffffffu, l, o));
      h = max(h, __shfl_xor_sync(0xffffffffu, h, o));
    }
    if (lane == 0) { s_lo[a][warp] = l; s_hi[a][warp] = h; }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      long long l = s_lo[a][0], h = s_hi[a][0];
      for (int w = 1; w < nw; ++w) { l = min(l, s_lo[a][w]); h = max(h, s_hi[a][w]); }
      atomicMin((long long*)&st->lo_key[a], l);
      atomicMax((long long*)&st->hi_key[a], h);
    }
  }
}

// SM count of a device, cached per device (host side; atomic, so ranks or
// threads driving different GPUs from one process see their own device)
inline int sm_count(int dev) {
  static std::atomic<int> cache[64];
  if (dev < 0 || dev >= 64) dev = 0;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n <= 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 148;
    }
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

constexpr long long KEY_POS_INF = 0x7ff0000000000000LL;                 // order_key(+inf)
constexpr long long KEY_NEG_INF = (long long)0xfff0000000000000ULL ^ 0x7fffffffffffffffLL;  // order_key(-inf)

}  // namespace hj
