/*
 * hjoracle.c -- TEST INFRASTRUCTURE ONLY.  CPU restatement of the reference
 * grid-update path (/root/reference/pkg/src/hjls, cited file:line) used as
 * the parity checker for the sm_100a kernels and as the bench's CPU
 * baseline ("kind": "port").  Never imported by the product package.
 *
 * Pinned: tests/test_oracle_golden.py checks every function here against
 * golden vectors produced by running the reference itself
 * (tests/golden/make_golden.py writes the tests/golden npz fixtures).
 *
 * Structure deliberately follows the reference's array formulation, not the
 * CUDA kernel's per-node one: each axis is processed line by line, a line is
 * ghost-extended (_extend_axis, grid.py:203-225), full divided-difference
 * tables are built over the extension (_tables, spatial.py:92-96) and the
 * scheme formulas index into them with the reference's slice offsets
 * (_sl(t.dk, k, n), spatial.py:109-111).  Compile with -ffp-contract=off so
 * every operation is separately rounded, as in NumPy.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- minimal pthreads parallel-for (the container has no libgomp) ---- */
static int g_threads = 1;
void or_set_threads(int n) { g_threads = n < 1 ? 1 : (n > 256 ? 256 : n); }
int or_get_threads(void) { return g_threads; }

typedef void (*body_fn)(void* ctx, int64_t lo, int64_t hi);
typedef struct { body_fn fn; void* ctx; int64_t lo, hi; } par_job;
static void* par_run(void* p) { par_job* j = (par_job*)p; j->fn(j->ctx, j->lo, j->hi); return 0; }

static void par_for(int64_t n, body_fn fn, void* ctx) {
  int t = g_threads;
  if (t > n) t = (int)(n > 0 ? n : 1);
  if (t <= 1) { fn(ctx, 0, n); return; }
  pthread_t th[256];
  par_job jobs[256];
  for (int k = 0; k < t; ++k) {
    jobs[k].fn = fn; jobs[k].ctx = ctx;
    jobs[k].lo = n * k / t; jobs[k].hi = n * (k + 1) / t;
    if (k > 0) pthread_create(&th[k], 0, par_run, &jobs[k]);
  }
  par_run(&jobs[0]);
  for (int k = 1; k < t; ++k) pthread_join(th[k], 0);
}

#define OR_MAX_DIM 5

typedef struct {
  int dim;
  int64_t n[OR_MAX_DIM];
  double h[OR_MAX_DIM];
  int bc[OR_MAX_DIM]; /* 0 periodic, 1 extrapolate, 2 dirichlet */
  double bcv[OR_MAX_DIM];
  const double* nodes[OR_MAX_DIM];
} or_grid;

enum { OR_FIRST = 0, OR_ENO2 = 1, OR_ENO3 = 2, OR_WENO5 = 3 };
enum { OR_ADV = 0, OR_ROCKETS = 1, OR_ROCKETS_EXT = 2, OR_AIR3D = 3, OR_DI4 = 4 };

static int64_t total_nodes(const or_grid* g) {
  int64_t t = 1;
  for (int a = 0; a < g->dim; ++a) t *= g->n[a];
  return t;
}

static int64_t axis_stride(const or_grid* g, int axis) {
  int64_t s = 1;
  for (int a = g->dim - 1; a > axis; --a) s *= g->n[a];
  return s;
}

/* grid.py:203-225 for one line: ext[0 .. n+2w) from line values with stride */
static void extend_line(const double* line, int64_t stride, int64_t n, int w, int bc, double bcv, double* ext) {
  for (int64_t j = 0; j < n; ++j) ext[w + j] = line[j * stride];
  if (bc == 0) {            /* periodic: idx = arange(-w, n+w) % n (grid.py:212) */
    for (int k = 1; k <= w; ++k) {
      int64_t jl = ((-k) % n + n) % n;
      int64_t jr = (n - 1 + k) % n;
      ext[w - k] = line[jl * stride];
      ext[w + n - 1 + k] = line[jr * stride];
    }
  } else if (bc == 2) {     /* dirichlet: np.pad constant (grid.py:214-217) */
    for (int k = 1; k <= w; ++k) { ext[w - k] = bcv; ext[w + n - 1 + k] = bcv; }
  } else {                  /* extrapolate (grid.py:219-224) */
    const double v0 = line[0], v1 = line[stride];
    const double vn = line[(n - 1) * stride], vm = line[(n - 2) * stride];
    const double ls = v0 - v1, rs = vn - vm;
    for (int k = 1; k <= w; ++k) {
      ext[w - k] = v0 + (double)k * ls;
      ext[w + n - 1 + k] = vn + (double)k * rs;
    }
  }
}

static double pick(double a, double b) { return fabs(a) <= fabs(b) ? a : b; } /* spatial.py:481-483 */

/* _weno_side (spatial.py:182-221) */
static double weno_side(double m1, double m2, double m3, double m4, double m5, int raw, double* diag) {
  double s0 = m1 / 3.0 - 7.0 * m2 / 6.0 + 11.0 * m3 / 6.0;
  double s1 = -m2 / 6.0 + 5.0 * m3 / 6.0 + m4 / 3.0;
  double s2 = m3 / 3.0 + 5.0 * m4 / 6.0 - m5 / 6.0;
  double c = 13.0 / 12.0;
  double a1 = m1 - 2.0 * m2 + m3, b1 = m1 - 4.0 * m2 + 3.0 * m3;
  double a2 = m2 - 2.0 * m3 + m4, b2 = m2 - m4;
  double a3 = m3 - 2.0 * m4 + m5, b3 = 3.0 * m3 - 4.0 * m4 + m5;
  double sg1 = c * (a1 * a1) + 0.25 * (b1 * b1);
  double sg2 = c * (a2 * a2) + 0.25 * (b2 * b2);
  double sg3 = c * (a3 * a3) + 0.25 * (b3 * b3);
  double q[5];
  if (raw) { q[0] = m1; q[1] = m2; q[2] = m3; q[3] = m4; q[4] = m5; }
  else { q[0] = m1 * m1; q[1] = m2 * m2; q[2] = m3 * m3; q[3] = m4 * m4; q[4] = m5 * m5; }
  double local = q[0];
  for (int k = 1; k < 5; ++k) if (q[k] > local) local = q[k];
  double eps = 1e-6 * local + 1e-99;
  double e1 = sg1 + eps, e2 = sg2 + eps, e3 = sg3 + eps;
  double al1 = 0.1 / (e1 * e1), al2 = 0.6 / (e2 * e2), al3 = 0.3 / (e3 * e3);
  double tot = al1 + al2 + al3;
  double w1 = al1 / tot, w2 = al2 / tot, w3 = al3 / tot;
  if (diag) {
    diag[0] = sg1; diag[1] = sg2; diag[2] = sg3; diag[3] = al1; diag[4] = al2;
    diag[5] = al3; diag[6] = eps; diag[7] = w1; diag[8] = w2; diag[9] = w3;
  }
  return w1 * s0 + w2 * s1 + w3 * s2;
}

static int width_of(int scheme) { return scheme == OR_FIRST ? 1 : (scheme == OR_ENO2 ? 2 : 3); }

/* One line: derivative pair with the reference's table indexing.
 * work must hold 4*(n+2w) doubles. */
static void line_pair(const double* line, int64_t stride, int64_t n, int scheme, int raw, double h, int bc,
                      double bcv, double* work, double* L, double* R, int64_t ostride) {
  const int w = width_of(scheme);
  const int64_t ne = n + 2 * w;
  double* d0 = work;
  double* d1 = d0 + ne;
  double* d2 = d1 + ne;
  double* d3 = d2 + ne;
  extend_line(line, stride, n, w, bc, bcv, d0);
  for (int64_t p = 0; p + 1 < ne; ++p) d1[p] = (d0[p + 1] - d0[p]) / h;           /* spatial.py:93 */
  if (scheme == OR_ENO2 || scheme == OR_ENO3) {
    const double h2 = 2.0 * h;
    for (int64_t p = 0; p + 2 < ne; ++p) d2[p] = (d1[p + 1] - d1[p]) / h2;        /* spatial.py:94 */
  }
  if (scheme == OR_ENO3) {
    const double h3 = 3.0 * h;
    for (int64_t p = 0; p + 3 < ne; ++p) d3[p] = (d2[p + 1] - d2[p]) / h3;        /* spatial.py:95 */
  }
  for (int64_t i = 0; i < n; ++i) {
    double l, r;
    if (scheme == OR_FIRST) {                                                      /* spatial.py:119-126 */
      l = d1[w - 1 + i];
      r = d1[w + i];
    } else if (scheme == OR_WENO5) {                                               /* spatial.py:224-247 */
      l = weno_side(d1[i + w - 3], d1[i + w - 2], d1[i + w - 1], d1[i + w], d1[i + w + 1], raw, 0);
      r = weno_side(d1[i + w + 2], d1[i + w + 1], d1[i + w], d1[i + w - 1], d1[i + w - 2], raw, 0);
    } else {
      const double la = d2[w - 2 + i], lb = d2[w - 1 + i];                         /* spatial.py:135-140 */
      const int lc = fabs(la) <= fabs(lb);
      l = d1[w - 1 + i] + (lc ? la : lb) * h;
      const double ra = d2[w - 1 + i], rb = d2[w + i];
      const int rc = fabs(ra) <= fabs(rb);
      r = d1[w + i] - (rc ? ra : rb) * h;
      if (scheme == OR_ENO3) {                                                     /* spatial.py:170-178 */
        double first = lc ? d3[w - 3 + i] : d3[w - 2 + i];
        double second = lc ? d3[w - 2 + i] : d3[w - 1 + i];
        double mult = lc ? 2.0 : -1.0;
        l = l + pick(first, second) * mult * h * h;
        first = rc ? d3[w - 2 + i] : d3[w - 1 + i];
        second = rc ? d3[w - 1 + i] : d3[w + i];
        mult = rc ? -1.0 : 2.0;
        r = r + pick(first, second) * mult * h * h;
      }
    }
    L[i * ostride] = l;
    R[i * ostride] = r;
  }
}

/* derivative_pair(g, v, axis, scheme) -- spatial.py:268-276 */
typedef struct {
  const or_grid* g; int scheme, axis, raw; const double* v; double* left; double* right; int64_t n, s;
} deriv_ctx;

static void deriv_body(void* p, int64_t lo, int64_t hi) {
  const deriv_ctx* c = (const deriv_ctx*)p;
  const int w = width_of(c->scheme);
  double* work = (double*)malloc(sizeof(double) * 4 * (c->n + 2 * w));
  for (int64_t Lq = lo; Lq < hi; ++Lq) {
    const int64_t outer = Lq / c->s, inner = Lq % c->s;
    const int64_t base = outer * c->n * c->s + inner;
    line_pair(c->v + base, c->s, c->n, c->scheme, c->raw, c->g->h[c->axis], c->g->bc[c->axis],
              c->g->bcv[c->axis], work, c->left + base, c->right + base, c->s);
  }
  free(work);
}

void or_derivs(const or_grid* g, int scheme, int axis, int raw, const double* v, double* left, double* right) {
  deriv_ctx c = {g, scheme, axis, raw, v, left, right, g->n[axis], axis_stride(g, axis)};
  par_for(total_nodes(g) / c.n, deriv_body, &c);
}

/* weno5_workspace (spatial.py:250-257): ws = 10 consecutive fields */
void or_weno_workspace(const or_grid* g, int axis, int side, int raw, const double* v, double* ws) {
  const int64_t n = g->n[axis], s = axis_stride(g, axis), tot = total_nodes(g);
  const int64_t lines = tot / n;
  const int w = 3;
  double* work = (double*)malloc(sizeof(double) * 2 * (n + 2 * w));
  for (int64_t Lq = 0; Lq < lines; ++Lq) {
    const int64_t outer = Lq / s, inner = Lq % s, base = outer * n * s + inner;
    double* d0 = work;
    double* d1 = work + n + 2 * w;
    extend_line(v + base, s, n, w, g->bc[axis], g->bcv[axis], d0);
    for (int64_t p = 0; p + 1 < n + 2 * w; ++p) d1[p] = (d0[p + 1] - d0[p]) / g->h[axis];
    for (int64_t i = 0; i < n; ++i) {
      double diag[10];
      if (side == 0) weno_side(d1[i], d1[i + 1], d1[i + 2], d1[i + 3], d1[i + 4], raw, diag);
      else weno_side(d1[i + 5], d1[i + 4], d1[i + 3], d1[i + 2], d1[i + 1], raw, diag);
      for (int k = 0; k < 10; ++k) ws[k * tot + base + i * s] = diag[k];
    }
  }
  free(work);
}

/* extend_with_ghost_cells (grid.py:228-243): axes extended in order */
void or_extend_ghost(const or_grid* g, int w, const double* v, double* out) {
  int64_t shape[OR_MAX_DIM];
  for (int a = 0; a < g->dim; ++a) shape[a] = g->n[a];
  int64_t cur_total = total_nodes(g);
  double* cur = (double*)malloc(sizeof(double) * cur_total);
  memcpy(cur, v, sizeof(double) * cur_total);
  for (int axis = 0; axis < g->dim; ++axis) {
    const int64_t n = shape[axis];
    int64_t s = 1;
    for (int a = g->dim - 1; a > axis; --a) s *= shape[a];
    const int64_t lines = cur_total / n;
    const int64_t ne = n + 2 * w;
    double* nxt = (double*)malloc(sizeof(double) * lines * ne);
    double* ext = (double*)malloc(sizeof(double) * ne);
    for (int64_t Lq = 0; Lq < lines; ++Lq) {
      const int64_t outer = Lq / s, inner = Lq % s;
      extend_line(cur + outer * n * s + inner, s, n, w, g->bc[axis], g->bcv[axis], ext);
      for (int64_t p = 0; p < ne; ++p) nxt[outer * ne * s + p * s + inner] = ext[p];
    }
    free(ext);
    free(cur);
    cur = nxt;
    shape[axis] = ne;
    cur_total = lines * ne;
  }
  memcpy(out, cur, sizeof(double) * cur_total);
  free(cur);
}

/* H(x, p) for the registered Hamiltonians, elementwise over the grid.
 * prm layout = include/hjb200.h hj_ham.p; tab[0], tab[1] as there. */
typedef struct {
  const or_grid* g; int kind; const double* prm; const double* const* tab; const double* const* p; double* out;
} ham_ctx;

static void ham_body(void* pc, int64_t lo, int64_t hi) {
  const ham_ctx* c = (const ham_ctx*)pc;
  const or_grid* g = c->g;
  const int d = g->dim, kind = c->kind;
  const double* prm = c->prm;
  const double* const* tab = c->tab;
  const double* const* p = c->p;
  for (int64_t q = lo; q < hi; ++q) {
    int64_t ix[OR_MAX_DIM], rem = q;
    for (int a = d - 1; a >= 0; --a) { ix[a] = rem % g->n[a]; rem /= g->n[a]; }
    double H;
    if (kind == OR_ADV) {                        /* term.py:136-140 */
      H = 0.0;
      for (int a = 0; a < d; ++a) H += prm[a] * p[a][q];
    } else if (kind == OR_ROCKETS) {             /* reachability.py:70-80 */
      const double a = prm[0], grav = prm[1], umin = prm[2], umax = prm[3];
      const double x = g->nodes[0][ix[0]], ct = tab[0][ix[2]], st = tab[1][ix[2]];
      const double p1 = p[0][q], p2 = p[1][q], p3 = p[2][q];
      H = -a * p1 * ct - p2 * (grav - a - a * st) - umax * fabs(p1 * x + p3) + umin * fabs(p2 * x + p3);
    } else if (kind == OR_ROCKETS_EXT) {         /* reachability.py:101-115 */
      const double a = prm[0], grav = prm[1], umin = prm[2], umax = prm[3];
      const double mid = 0.5 * (umax + umin), half = 0.5 * (umax - umin);
      const double x = g->nodes[0][ix[0]], ct = tab[0][ix[2]], st = tab[1][ix[2]];
      const double p1 = p[0][q], p2 = p[1][q], p3 = p[2][q];
      const double c1 = p1 * x - p3, c2 = p2 * x + p3;
      H = -a * p1 * ct + p2 * (grav - a - a * st) - mid * (c1 + c2) - half * fabs(c1) + half * fabs(c2);
    } else if (kind == OR_AIR3D) {               /* problems.air3d_hamiltonian */
      const double va = prm[0], ain = prm[2], bin = prm[3];
      const double x = g->nodes[0][ix[0]], y = g->nodes[1][ix[1]];
      const double vbc = tab[0][ix[2]], vbs = tab[1][ix[2]];
      const double p1 = p[0][q], p2 = p[1][q], p3 = p[2][q];
      H = -(-va * p1 + vbc * p1 + vbs * p2 + ain * fabs(y * p1 - x * p2 - p3) - bin * fabs(p3));
    } else {                                     /* problems.di4_hamiltonian */
      const double ubar = prm[0], dbar = prm[1];
      const double wx = g->nodes[2][ix[2]], wy = g->nodes[3][ix[3]];
      H = -(p[0][q] * wx + p[1][q] * wy + (dbar - ubar) * (fabs(p[2][q]) + fabs(p[3][q])));
    }
    c->out[q] = H;
  }
}

void or_hamiltonian(const or_grid* g, int kind, const double* prm, const double* const* tab,
                    const double* const* p, double* out) {
  ham_ctx c = {g, kind, prm, tab, p, out};
  par_for(total_nodes(g), ham_body, &c);
}

/* term_lax_friedrichs (term.py:90-126) with alphas given (range-free
 * partials); lo/hi receive the costate ranges (term.py:71-77).  Returns
 * nonzero if any H != 0 (term.py:120). */
typedef struct {
  int d; const double* alpha; double* L[OR_MAX_DIM]; double* R[OR_MAX_DIM]; double* P[OR_MAX_DIM];
  double* delta; double mn[256][OR_MAX_DIM]; double mx[256][OR_MAX_DIM]; int nz[256]; int64_t chunks;
} term_ctx;

static void pavg_body(void* p, int64_t lo, int64_t hi) {
  term_ctx* c = (term_ctx*)p;
  for (int64_t k = lo; k < hi; ++k) {
    const int64_t q0 = k * c->chunks, q1 = q0 + c->chunks;
    for (int a = 0; a < c->d; ++a) {
      double mn = INFINITY, mx = -INFINITY;
      for (int64_t q = q0; q < q1; ++q) {
        const double l = c->L[a][q], r = c->R[a][q];
        c->P[a][q] = 0.5 * (l + r);                                             /* term.py:101 */
        mn = fmin(mn, fmin(l, r));
        mx = fmax(mx, fmax(l, r));
      }
      c->mn[k][a] = mn;
      c->mx[k][a] = mx;
    }
  }
}

static void delta_body(void* p, int64_t lo, int64_t hi) {
  term_ctx* c = (term_ctx*)p;
  for (int64_t k = lo; k < hi; ++k) {
    int nz = 0;
    for (int64_t q = k * c->chunks; q < (k + 1) * c->chunks; ++q) {
      double diss = 0.0;                                                        /* term.py:84 */
      for (int a = 0; a < c->d; ++a) diss += c->alpha[a] * 0.5 * (c->R[a][q] - c->L[a][q]); /* term.py:85-86 */
      const double H = c->delta[q];
      nz |= (H != 0.0);
      c->delta[q] = diss - H;                                                   /* term.py:113 */
    }
    c->nz[k] = nz;
  }
}

/* term_lax_friedrichs (term.py:90-126) with alphas given (range-free
 * partials); lo/hi receive the costate ranges (term.py:71-77).  Returns
 * nonzero if any H != 0 (term.py:120).  Work is split into `parts` equal
 * chunks of nodes (parts divides the node count; 1 is always valid). */
int or_term(const or_grid* g, int scheme, int kind, const double* prm, const double* const* tab,
            const double* alpha, const double* v, double* delta, double* lo, double* hi) {
  const int64_t tot = total_nodes(g);
  term_ctx* c = (term_ctx*)calloc(1, sizeof(term_ctx));
  c->d = g->dim;
  c->alpha = alpha;
  c->delta = delta;
  int parts = g_threads;
  while (parts > 1 && tot % parts) --parts;
  c->chunks = tot / parts;
  for (int a = 0; a < c->d; ++a) {
    c->L[a] = (double*)malloc(sizeof(double) * tot);
    c->R[a] = (double*)malloc(sizeof(double) * tot);
    c->P[a] = (double*)malloc(sizeof(double) * tot);
    or_derivs(g, scheme, a, 0, v, c->L[a], c->R[a]);                         /* term.py:100 */
  }
  par_for(parts, pavg_body, c);
  for (int a = 0; a < c->d; ++a) {
    double mn = INFINITY, mx = -INFINITY;
    for (int k = 0; k < parts; ++k) { mn = fmin(mn, c->mn[k][a]); mx = fmax(mx, c->mx[k][a]); }
    if (lo) lo[a] = mn;
    if (hi) hi[a] = mx;
  }
  or_hamiltonian(g, kind, prm, tab, (const double* const*)c->P, delta);     /* delta holds H for now */
  par_for(parts, delta_body, c);
  int nonzero = 0;
  for (int k = 0; k < parts; ++k) nonzero |= c->nz[k];
  for (int a = 0; a < c->d; ++a) { free(c->L[a]); free(c->R[a]); free(c->P[a]); }
  free(c);
  return nonzero;
}

/* stage combinations (integrator.py:93-103); stage 1 Euler, 2 RK2 avg,
 * 3 RK3 quarter, 4 RK3 third */
typedef struct { int stage; double dt; const double* y; const double* y0; const double* delta; double* out; } stage_ctx;

static void stage_body(void* p, int64_t lo, int64_t hi) {
  const stage_ctx* c = (const stage_ctx*)p;
  for (int64_t q = lo; q < hi; ++q) {
    const double e = c->y[q] + c->dt * c->delta[q];
    double r;
    if (c->stage == 1) r = e;
    else if (c->stage == 2) r = 0.5 * (c->y0[q] + e);
    else if (c->stage == 3) r = 0.25 * (3.0 * c->y0[q] + e);
    else r = (c->y0[q] + 2.0 * e) / 3.0;
    c->out[q] = r;
  }
}

void or_stage(int64_t n, int stage, double dt, const double* y, const double* y0, const double* delta, double* out) {
  stage_ctx c = {stage, dt, y, y0, delta, out};
  par_for(n, stage_body, &c);
}

/* mask (reachability.py:249) */
void or_mask(int64_t n, const double* prev, double* v, int use_min) {
  for (int64_t q = 0; q < n; ++q) v[q] = use_min ? fmin(v[q], prev[q]) : fmax(v[q], prev[q]);
}

/* shapes.py:24-83 (kinds as hjb200.h HJ_SHAPE_*) */
void or_shape(const or_grid* g, int kind, const double* prm, double* out) {
  const int64_t tot = total_nodes(g);
  const int d = g->dim;
  for (int64_t q = 0; q < tot; ++q) {
    int64_t ix[OR_MAX_DIM], rem = q;
    for (int a = d - 1; a >= 0; --a) { ix[a] = rem % g->n[a]; rem /= g->n[a]; }
    double r;
    if (kind == 0 || kind == 1) {
      const unsigned ignore = kind == 1 ? (unsigned)prm[d + 1] : 0u;
      double d2 = 0.0;
      for (int a = 0; a < d; ++a) {
        if (ignore & (1u << a)) continue;
        const double t = g->nodes[a][ix[a]] - prm[a];
        d2 += t * t;
      }
      r = sqrt(d2) - prm[d];
    } else if (kind == 2) {
      double e = 0.0;
      for (int a = 0; a < d; ++a) { const double x = g->nodes[a][ix[a]]; e += prm[a] * (x * x); }
      r = e - prm[d];
    } else {
      double s = 0.0, qm = 0.0;
      for (int a = 0; a < d; ++a) {
        const double x = g->nodes[a][ix[a]];
        const double qa = fmax(prm[a] - x, x - prm[d + a]);
        const double qp = fmax(qa, 0.0);
        s += qp * qp;
        qm = (a == 0) ? qa : fmax(qm, qa);
      }
      r = sqrt(s) + fmin(qm, 0.0);
    }
    out[q] = r;
  }
}
