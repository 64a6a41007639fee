/*
 * hjb200.h -- C ABI of libhjb200.so, the sm_100a grid-update path of the
 * Hamilton-Jacobi level-set solver (arXiv 2411.03501, LevelSetPy-style).
 *
 * Every entry point replaces one array pass of the reference's NumPy path
 * (reference = /root/reference/pkg/src/hjls, cited as file:line).  The
 * reference is pure Python, so its "FFI" is the Python call itself; the
 * package paper_2411_03501_b200 binds these symbols through ctypes (see
 * INTEGRATION.md) behind the reference's own function names.
 *
 * ABI rules
 *   - plain C types, device pointers, sizes; no torch / CUDA types in the
 *     signatures (streams travel as void* = cudaStream_t);
 *   - stream-ordered and asynchronous: no call synchronises the device;
 *   - no exceptions cross the ABI: every call returns HJ_OK or a negative
 *     HJ_E* code and leaves a thread-local message in hj_last_error();
 *   - the caller owns every buffer; fields are fp64, row-major (last axis
 *     contiguous), optionally preceded by a batch axis (independent problems
 *     sharing grid and dynamics) and, on axis 0, by exchanged halo planes.
 *
 * Bit-exactness: the library is compiled with --fmad=false and reproduces
 * the reference's operation order, so results equal
 * the NumPy reference value for value (np.array_equal).
 */
#ifndef HJB200_H
#define HJB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HJ_MAX_DIM 5

/* status codes */
enum {
  HJ_OK = 0,
  HJ_EINVAL = -1,     /* argument validation (reference: ValueError)           */
  HJ_ECUDA = -2,      /* CUDA launch / runtime failure                         */
  HJ_ENCCL = -3,      /* NCCL missing or failed (multi-GPU hj_dd_* calls)      */
  HJ_ENONFINITE = -4  /* reserved: non-finite data (reported through hj_stats) */
};

/* boundary kinds -- grid.py:26-52 (BoundaryCondition / periodic / extrapolate / dirichlet) */
enum { HJ_BC_PERIODIC = 0, HJ_BC_EXTRAPOLATE = 1, HJ_BC_DIRICHLET = 2 };

/* derivative schemes -- spatial.py:260-266 (_SCHEMES).
 * HJ_WENO5_FMA is an addition: the same WENO5 scheme evaluated in tolerance
 * mode (FMA contraction, reciprocal multiplies, one division per side for the
 * weights) -- not bit-exact, but within the north-star contract (L-inf
 * relative <= 1e-9 of the reference over a solve, sign(V) preserved); every
 * other scheme is bit-exact. */
enum { HJ_FIRST = 0, HJ_ENO2 = 1, HJ_ENO3 = 2, HJ_WENO5 = 3, HJ_WENO5_FMA = 4 };

/* WENO epsilon modes -- spatial.py:205-211 */
enum { HJ_EPS_SQUARED = 0, HJ_EPS_RAW = 1 };

/* device Hamiltonians (registered TermConfig factories)
 *   ADVECTION        term.py:129-145            p[0..dim-1] = speeds c_i
 *   ROCKETS          reachability.py:61-81      p = {a, grav, u_min, u_max}
 *   ROCKETS_EXTREMAL reachability.py:84-116     p = {a, grav, u_min, u_max}
 *   AIR3D            builder fixture p = {v_a, v_b, a_in, b_in}, tab[0]=v_b*cos(psi), tab[1]=v_b*sin(psi)
 *   DI4              builder fixture p = {u_bar, d_bar}
 * ROCKETS uses tab[0]=cos(theta), tab[1]=sin(theta) computed on the host with np.cos/np.sin
 * (the GPU never recomputes trig, so the tables are the reference's bits). */
enum {
  HJ_HAM_ADVECTION = 0,
  HJ_HAM_ROCKETS = 1,
  HJ_HAM_ROCKETS_EXTREMAL = 2,
  HJ_HAM_AIR3D = 3,
  HJ_HAM_DI4 = 4
};

/* RK stage kinds -- integrator.py:92-103 (Shu-Osher TVD-RK, Appendix A.3) */
enum {
  HJ_STAGE_DELTA = 0,        /* out = delta                         (term only)      */
  HJ_STAGE_EULER = 1,        /* out = y + dt*delta                                     */
  HJ_STAGE_RK2_AVG = 2,      /* out = 0.5*(y0 + (y + dt*delta))                        */
  HJ_STAGE_RK3_QUARTER = 3,  /* out = 0.25*(3.0*y0 + (y + dt*delta))                   */
  HJ_STAGE_RK3_THIRD = 4     /* out = (y0 + 2.0*(y + dt*delta)) / 3.0                  */
};

/* parts of a stage launch along axis 0 (multi-GPU overlap):
 * CORE = the owned planes whose stencils read no exchanged halo plane (runs
 * while the halo exchange is in flight), RIM = the rest; CORE + RIM = ALL,
 * bit for bit.  The split follows the kernel's own axis-0 tiling. */
enum { HJ_PART_ALL = 0, HJ_PART_CORE = 1, HJ_PART_RIM = 2 };

/* tube masks -- reachability.py:234,249 */
enum { HJ_MASK_NONE = 0, HJ_MASK_MIN = 1, HJ_MASK_MAX = 2 };

/* implicit surfaces -- shapes.py:24-83 */
enum { HJ_SHAPE_SPHERE = 0, HJ_SHAPE_CYLINDER = 1, HJ_SHAPE_ELLIPSOID = 2, HJ_SHAPE_BOX = 3 };

/* CSG -- shapes.py:91-111 */
enum { HJ_CSG_UNION = 0, HJ_CSG_INTERSECT = 1, HJ_CSG_COMPLEMENT = 2, HJ_CSG_DIFFERENCE = 3 };

/* non-finite flag bits (hj_stats.nonfinite) mapped by the host to the reference's messages */
enum {
  HJ_NF_INPUT = 1,  /* stage input y   -- grid.py:75-76 via integrator.py:81 ScalarField(y) */
  HJ_NF_DERIV = 2,  /* a derivative    -- spatial.py:84-89 ScalarField(left/right)          */
  HJ_NF_HAM = 4,    /* H(x, p)         -- term.py:109-110                                    */
  HJ_NF_DELTA = 8,  /* dv/dt           -- integrator.py:64-65                                */
  HJ_NF_OUTPUT = 16, /* stage output                                                          */
  HJ_FLAG_HAM_NONZERO = 32 /* H != 0 somewhere (term.py:120 zero-dissipation warning)           */
};

/* Grid metadata (grid.py:89-175 Grid) as seen by one device.
 * Axis 0 may be a slab [slab_lo, slab_lo + n[0]) of a global axis of
 * n_global0 nodes (multi-GPU domain decomposition).  When
 * halo_lo/halo_hi is 1 the field buffer carries `halo` exchanged planes in
 * front of / behind the owned planes and the kernels read them instead of
 * synthesising boundary ghosts; field pointers always point at the first
 * OWNED plane. */
/* exchanged halo planes per side a slab buffer must carry (hj_grid.halo):
 * the fused stage kernels stage this many whatever the scheme's ghost width */
#define HJ_HALO_MIN 3

typedef struct hj_grid {
  int32_t dim;                        /* 1..4 (HJ_MAX_DIM reserved)                         */
  int32_t batch;                      /* >= 1 independent problems stacked in front         */
  int64_t n[HJ_MAX_DIM];              /* nodes per axis (owned slab count on axis 0)        */
  double h[HJ_MAX_DIM];               /* spacings (grid.py:159-166)                         */
  int32_t bc[HJ_MAX_DIM];             /* HJ_BC_*                                            */
  double bc_value[HJ_MAX_DIM];        /* dirichlet constants                                */
  const double* nodes[HJ_MAX_DIM];    /* device copies of g.axis_nodes (owned slab on 0)    */
  int32_t halo_lo, halo_hi;           /* 1 = neighbour planes present on that side of axis 0 */
  int32_t halo;                       /* planes stored per side when halo_lo/hi             */
  int32_t _pad;
  int64_t batch_stride;               /* elements between consecutive problems (0 = dense)  */
} hj_grid;

/* Registered device Hamiltonian (TermConfig.hamiltonian, term.py:29). */
typedef struct hj_ham {
  int32_t kind;                       /* HJ_HAM_*                                           */
  int32_t _pad;
  double p[16];                       /* scalar constants                                   */
  const double* tab[4];               /* device tables (host-computed trig etc.)            */
} hj_ham;

/* Device-resident per-call statistics (zeroed with hj_stats_reset).
 * lo_key/hi_key: order-preserving int64 images of the per-axis costate range
 * min(p-, p+) / max(p-, p+) (term.py:71-77), decoded on the host. */
typedef struct hj_stats {
  int64_t lo_key[HJ_MAX_DIM];
  int64_t hi_key[HJ_MAX_DIM];
  uint32_t nonfinite;                 /* OR of HJ_NF_* bits                                 */
  int32_t first_bad_tag;              /* min over failing nodes of tag*8 + error class
                                         (1 input, 2 derivative, 3 H, 4 delta, 5 output);
                                         0x7fffffff when nothing failed                    */
} hj_stats;

/* ---------------------------------------------------------------- meta */
int hj_version(void);
const char* hj_last_error(void);
/* number of device kernels this thread has launched through the ABI (bench evidence) */
uint64_t hj_launch_count(void);

/* ---------------------------------------------------------------- grid / ghosts */
/* extend_with_ghost_cells (grid.py:228-243; per-axis rule _extend_axis grid.py:203-225).
 * ext has shape (n0+2w, ..., n_{d-1}+2w); corners are the per-axis composition. */
int hj_extend_ghost(const hj_grid* g, int width, const double* v, double* ext, void* stream);

/* ---------------------------------------------------------------- spatial */
/* upwind_first_{first,eno2,eno3,weno5} / derivative_pair (spatial.py:119-276):
 * the left/right one-sided derivative fields of v along `axis`. */
int hj_derivs(const hj_grid* g, int scheme, int axis, int eps_mode,
              const double* v, double* left, double* right, void* stream);

/* divided_differences (spatial.py:99-106, tables _tables 92-96): ghost-extend
 * `axis` by `width` and write D0 (the extension), D1, D2, D3 oriented with the
 * working axis last (np.moveaxis(ext, axis, -1)); d2/d3 may be NULL when
 * order < 2 / < 3. */
int hj_divided_differences(const hj_grid* g, int axis, int width, int order, const double* v,
                           double* d0, double* d1, double* d2, double* d3, void* stream);

/* weno5_workspace (spatial.py:250-257): the 10 diagnostic fields of one side
 * (side 0 = left, 1 = right) in the order sigma1..3, alpha1..3, eps, w1..3;
 * ws points at 10 consecutive fields of the grid's size. */
int hj_weno5_workspace(const hj_grid* g, int axis, int side, int eps_mode,
                       const double* v, double* ws, void* stream);

/* ---------------------------------------------------------------- term + RK stage (fused) */
/* One fused pass = ghosts -> per-axis upwind derivatives -> p_avg -> H(x,p_avg)
 * -> GLF dissipation -> delta = diss - H (term.py:90-126) -> stage update
 * (integrator.py:92-103) -> optional tube mask (reachability.py:249).
 *   alpha: host array of dim dissipation coefficients (partials, range-independent);
 *   stage: HJ_STAGE_*; y_in = the stage input, y0 = the step's initial state
 *          (RK2_AVG / RK3_* only), y_out may not alias y_in;
 *   mask_prev/mask: applied to the output when mask != HJ_MASK_NONE;
 *   stats: device pointer or NULL; tag identifies the stage for first_bad_tag. */
int hj_stage(const hj_grid* g, int scheme, const hj_ham* ham, const double* alpha,
             double dt, int stage, const double* y_in, const double* y0, double* y_out,
             const double* mask_prev, int mask, hj_stats* stats, int32_t tag, void* stream);

/* hj_stage restricted to one axis-0 part (HJ_PART_*): on a slab with exchanged
 * halos, launch CORE, wait for the exchange, launch RIM. */
int hj_stage_part(const hj_grid* g, int scheme, const hj_ham* ham, const double* alpha,
                  double dt, int stage, const double* y_in, const double* y0, double* y_out,
                  const double* mask_prev, int mask, hj_stats* stats, int32_t tag, int part,
                  void* stream);

/* hj_stage over the owned axis-0 planes [plane_lo, plane_hi) only (a pipeline
 * stage consuming host->device chunks as they land / producing device->host
 * chunks as they finish): plane_lo a multiple of HJ_ROW_PLANES, plane_hi a
 * multiple of it or n[0].  Reads planes plane_lo-w .. plane_hi+w-1 of y_in
 * (w = the scheme's ghost width), writes only [plane_lo, plane_hi). */
#define HJ_ROW_PLANES 8
int hj_stage_planes(const hj_grid* g, int scheme, const hj_ham* ham, const double* alpha,
                    double dt, int stage, const double* y_in, const double* y0, double* y_out,
                    const double* mask_prev, int mask, hj_stats* stats, int32_t tag,
                    int64_t plane_lo, int64_t plane_hi, void* stream);

/* rockets_hamiltonian / rockets_hamiltonian_extremal / advection H as an API
 * call (reachability.py:61-116, term.py:136-140): out = H(x, p) with p an array
 * of dim device pointers to costate fields. */
int hj_eval_hamiltonian(const hj_grid* g, const hj_ham* ham, const double* const* p, double* out,
                        void* stream);

/* The integration loop of ode_cfl_1/2/3 (integrator.py:69-126) natively:
 * dt = cfl*bound, min(max_step) (max_step <= 0: none), clipped to the span,
 * t = t1 on the last step; each TVD-RK stage one hj_stage launch (tags
 * step*4 + stage), the mask applied in the final stage; no device sync.
 * Small grids (where hj_stage would pick the per-node / tile kernel) run the
 * whole stage schedule as one cooperative launch per 1024 stages with a grid
 * barrier between stages -- the same node updates, bit for bit.
 * y_init is not written; buf0..2 are the work buffers (one of them, or
 * y_init when no step is taken, is returned in *y_final).
 * info (host, 6 doubles): t_final, steps, min_dt, max_dt, bad_dt_flag, bad_dt. */
int hj_integrate(const hj_grid* g, int scheme, const hj_ham* ham, const double* alpha, int order, double t0,
                 double t1, double cfl, double max_step, int single_step, double bound, const double* y_init,
                 double* buf0, double* buf1, double* buf2, const double* mask_prev, int mask, hj_stats* stats,
                 double* info, double** y_final, void* stream);

/* term_lax_friedrichs with a registered Hamiltonian: delta only (HJ_STAGE_DELTA). */
int hj_term(const hj_grid* g, int scheme, const hj_ham* ham, const double* alpha,
            const double* v, double* delta, hj_stats* stats, void* stream);

/* Host-Hamiltonian bridge (user TermConfig lambdas, term.py:90-126 with
 * Python H/partials): p_avg[a] = 0.5*(L_a + R_a) for every axis, plus the
 * costate ranges into stats.  left/right/p_avg: arrays of dim device pointers. */
int hj_costates(const hj_grid* g, const double* const* left, const double* const* right,
                double* const* p_avg, hj_stats* stats, void* stream);
/* delta = (sum_a (alpha_a*0.5)*(R_a - L_a)) - H  (term.py:84-86,113); diss optional. */
int hj_glf_delta(const hj_grid* g, const double* alpha, const double* const* left,
                 const double* const* right, const double* ham, double* diss, double* delta,
                 hj_stats* stats, void* stream);
/* Stage combination for an arbitrary term callable (integrator.py:92-103). */
int hj_rk_combine(int64_t count, int stage, double dt, const double* y_in, const double* y0,
                  const double* delta, double* out, hj_stats* stats, int32_t tag, void* stream);

/* ---------------------------------------------------------------- init / tube helpers */
/* shapes.py:24-83.  params:
 *   SPHERE    {c_0..c_{d-1}, radius}
 *   CYLINDER  {c_0..c_{d-1}, radius, ignore_mask (bit a = axis a ignored)}
 *   ELLIPSOID {w_0..w_{d-1}, radius}
 *   BOX       {lo_0..lo_{d-1}, hi_0..hi_{d-1}} */
int hj_init_shape(const hj_grid* g, int kind, const double* params, int nparams,
                  double* out, void* stream);
/* shapes.py:91-111 (b ignored for COMPLEMENT) */
int hj_csg(int op, int64_t count, const double* a, const double* b, double* out, void* stream);
/* reachability.py:249: v = min(v, prev) (HJ_MASK_MIN) or max (HJ_MASK_MAX), in place */
int hj_mask(int64_t count, const double* prev, double* v, int mask, void* stream);
/* reachability.py:257-260: *d_count += #{v < level} */
int hj_count_below(int64_t count, const double* v, double level,
                   unsigned long long* d_count, void* stream);
/* Tube acceptance checks on the device (test_reachability.py:218-285 over the
 * mask of reachability.py:249), no field leaves the GPU.  Adds to d_out[4]:
 *   [0] nesting violations   #{v > prev} (HJ_MASK_MIN) / #{v < prev} (HJ_MASK_MAX)
 *   [1] containment violations #{v > target} / #{v < target}
 *   [2] #{v < level}           (sublevel_volume's count, reachability.py:257-260)
 *   [3] #{prev >= level and v < level}  (nodes captured during the interval) */
int hj_tube_check(int64_t count, const double* prev, const double* v, const double* target, int mask, double level,
                  unsigned long long* d_out, void* stream);
/* Self-check of the hoisted-reciprocal division used by the fast kernels:
 * n random/special operand pairs, *d_mismatch += #{div_by(a,b) != a/b} (bitwise). */
int hj_check_division(int64_t n, uint64_t seed, unsigned long long* d_mismatch, void* stream);
/* Stage-kernel family (A/B measurements and test coverage): 0 per-node generic
 * kernel, 1 default dispatch (grids of brick size: the per-axis walk pipeline
 * for WENO5, the brick kernels otherwise; small 3-D grids: the tile kernel,
 * an hj_integrate interval as one persistent launch), 2 brick WENO5 kernel at
 * 1 CTA/SM, 3 brick kernels for every 3-D/4-D grid, 4 WENO5 walks rolled,
 * 5 timing bound only (WENO5 bricks after a CTA's first skip their
 * global->shared loads: WRONG results), 6 brick kernels without the L2
 * prefetch of the next brick, 7 the brick A/B slot, 8 small 3-D grids: tile
 * kernel per stage (no persistent launch), 9 the per-axis walk pipeline for
 * every WENO5 grid size, 10-12 per-axis pipeline A/B variants (10 every walk
 * rolled, 11 the contiguous-axis walk unrolled as well, 12 the last-axis
 * kernel on 32-node segments); -1 reads HJ_STAGE_KERNEL from the environment.
 * Returns the previous setting. */
int hj_set_stage_kernel(int variant);
/* FP64-pipe probe for the roofline denominator: blocks x 256 threads each run
 * iters x 8 independent DFMA chains (time it with events on `stream`). */
int hj_fp64_probe(int iters, int blocks, double* d_sink, void* stream);
/* Bounds-checking build only (libhjb200_check.so, compiled with
 * -DHJ_CHECK_BOUNDS; compute-sanitizer is closed on this pool): global
 * accesses of the stage kernels outside the extents of their fields since
 * the last call (synchronises the device, resets the count); -1 in the
 * normal build. */
int64_t hj_bounds_violations(void);
/* zero a device hj_stats (keys set to +inf/-inf images) */
int hj_stats_reset(hj_stats* stats, void* stream);

/* ---------------------------------------------------------------- multi-GPU slabs
 * Axis 0 split into contiguous slabs, one rank (process, GPU) each; the
 * field buffer of a slab carries hj_grid.halo (>= HJ_HALO_MIN) exchanged
 * planes in front of / behind its owned planes, and field pointers point at
 * the first owned plane.  NCCL is resolved at run time (dlopen libnccl.so.2,
 * or $HJ_NCCL_LIB); every call is stream-ordered, none synchronises the host.
 * Reference: the per-interval loop of reachability.py:242-249 with the ghost
 * extension of grid.py:203-225 along axis 0 replaced by the neighbours' planes
 * (halo depth = GHOST_WIDTH, spatial.py:27). */
#define HJ_DD_UID_BYTES 128
typedef struct hj_dd hj_dd;   /* opaque: communicator, exchange stream, events */
/* NCCL version code of the loaded library (>0) or HJ_ENCCL */
int hj_dd_nccl_version(void);
/* ncclGetUniqueId on the root rank; the host broadcasts the HJ_DD_UID_BYTES */
int hj_dd_unique_id(void* uid);
/* ncclCommInitRank on the current CUDA device; lo_rank / hi_rank = the axis-0
 * neighbours (-1 at a global edge; a periodic axis 0 makes a ring, a
 * one-rank ring exchanges with itself) */
int hj_dd_init(const void* uid, int nranks, int rank, int lo_rank, int hi_rank, hj_dd** dd);
/* One fused stage of this rank's slab (arguments as hj_stage): grouped
 * ncclSend/ncclRecv of the halo planes of y_in with both neighbours on the
 * communicator's stream, the CORE part on `stream` meanwhile (overlap != 0),
 * `stream` waits on the exchange, then the RIM part.  Bit-identical to the
 * undecomposed stage. */
int hj_dd_stage(hj_dd* dd, const hj_grid* g, int scheme, const hj_ham* ham, const double* alpha, double dt,
                int stage, const double* y_in, const double* y0, double* y_out, const double* mask_prev,
                int mask, hj_stats* stats, int32_t tag, int overlap, void* stream);
/* halo exchange of buf alone, `stream` ordered after it */
int hj_dd_exchange(hj_dd* dd, const hj_grid* g, double* buf, void* stream);
/* all-reduce a device hj_stats across the ranks: lo_key min, hi_key max,
 * nonfinite OR, first_bad_tag min -- every rank then holds the single-GPU run's
 * stats (the first failing stage and error class, the global costate ranges) */
int hj_dd_reduce_stats(hj_dd* dd, hj_stats* stats, void* stream);
/* gather every rank's owned planes (count doubles) into `full` on rank root,
 * in rank order; counts (host, nranks entries) are needed on the root only */
int hj_dd_gather(hj_dd* dd, const double* owned, int64_t count, double* full, const int64_t* counts, int root,
                 void* stream);
/* exchanges posted and halo bytes sent by this rank so far */
int hj_dd_stats(const hj_dd* dd, uint64_t* exchanges, uint64_t* halo_bytes);
int hj_dd_free(hj_dd* dd);

#ifdef __cplusplus
}
#endif
#endif /* HJB200_H */
