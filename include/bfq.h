/*
 * bfq.h -- C ABI of the B200-native Q(f,f) engine.
 *
 * This is the boundary the reference's operator API binds to.  The reference
 * (`boltzfact`, pure Python) has no native layer; each entry point below
 * replaces one Python call on the hot path:
 *
 *   bfq_plan_create       <- FactorizedOperator(...) / build_operator(...) result
 *                            handed to the device once
 *                            (pkg/src/boltzfact/contraction.py:76-108, :158-177)
 *   bfq_plan_create_bfct  <- cache.load_cache(path)  (pkg/src/boltzfact/cache.py:92-166)
 *                            + upload, without going through numpy
 *   bfq_eval              <- q_angular_first(op, c, c2) batched over cells, device
 *                            buffers (contraction.py:293-317; strategy signature
 *                            :236-238, registered in STRATEGIES :320-324)
 *   bfq_eval_host         <- evaluate(op, c) called on host arrays
 *                            (contraction.py:327-340): copies in, evaluates, copies out
 *   bfq_plan_work         <- ContractionStats accounting (contraction.py:51-73, :314-316)
 *   bfq_rk4_step          <- one step of harness.rk4_integrate (harness.py:79-120)
 *   bfq_moments           <- basis.moments per cell (basis.py:346-363)
 *   bfq_project_maxwellians <- basis.project(M_{u,T}, cfg, order) batched over
 *                            drifting Maxwellians (basis.py:262-299), closed
 *                            angular form (input generator of configs 2-5)
 *   bfq_projector_* / bfq_project_samples <- basis.project(f, cfg, order) for
 *                            any f sampled on the reference's quadrature grid
 *
 * Conventions: plain pointers and sizes, no torch types.  Every function returns
 * 0 on success and a negative BFQ_E* code otherwise; bfq_strerror() maps a code
 * to text, bfq_last_error() gives the detail of the last failure on the calling
 * thread.  A plan is immutable after creation, so concurrent bfq_eval calls on
 * different streams are safe.  One plan per device.
 *
 * Cell layout: values[cell][k][q], fp64, C-contiguous, q 0-based = l*l+l+m
 * (basis.py:69-73, :85-93), i.e. each cell is the reference CoefficientField
 * .values array of shape (n_k, n_q).
 */
#ifndef BFQ_H
#define BFQ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BFQ_OK 0
#define BFQ_EINVAL -1     /* bad argument, shape or operator content (-> ValueError)   */
#define BFQ_EUNSORTED -2  /* COO rows not grouped by (tau, q1) (contraction.py:299-301) */
#define BFQ_ECUDA -3      /* CUDA runtime failure (-> RuntimeError)                     */
#define BFQ_ENOMEM -4     /* device or host allocation failed                           */
#define BFQ_ESMEM -5      /* no kernel configuration fits in shared memory              */
#define BFQ_EIO -6        /* BFCT file unreadable / truncated                            */
#define BFQ_EFORMAT -7    /* BFCT magic/version wrong   (cache.py CacheFormatError)      */
#define BFQ_EINTEGRITY -8 /* BFCT checksum/size mismatch (cache.py CacheIntegrityError)  */
#define BFQ_EDIVERGED -9  /* RK4 state not finite (harness.py:103-107)                   */

typedef struct bfq_plan bfq_plan;

/* Operator description.  All pointers are HOST pointers, only read during
 * bfq_plan_create.  Index arrays are 0-based (the reference stores 1-based
 * COO columns, angular.py:260-269; FactorizedOperator makes the 0-based
 * views, contraction.py:98-104). */
typedef struct bfq_desc {
  int32_t k_max, l_max;
  double gamma;               /* informational (SpectralConfig.gamma)                 */
  int32_t n_t;                /* channels                                             */
  int64_t n_g;                /* COO rows                                             */
  int64_t n_s;                /* (tau, q1) slices                                     */
  const int32_t* triplets;    /* [n_t][3] = (l1, l2, l3), angular.py:119-135          */
  const int32_t* q1;          /* [n_g] 0-based output (test) angular index            */
  const int32_t* q2;          /* [n_g] 0-based angular index of slot-2 input          */
  const int32_t* q3;          /* [n_g] 0-based angular index of slot-3 input          */
  const int32_t* tau;         /* [n_g] 0-based channel                                */
  const double* g;            /* [n_g] real Gaunt weight                              */
  const int64_t* slice_starts;/* [n_s+1] row offsets of each (tau, q1) slice          */
  const int32_t* slice_tau;   /* [n_s] 0-based                                        */
  const int32_t* slice_q1;    /* [n_s] 0-based                                        */
  const double* r;            /* (n_k, n_k, n_k, n_t) C-order, kinematic.py:574-578   */
  int32_t conservation;       /* R rows of the invariants zeroed (kinematic.py:594-610) */
  int32_t detailed_balance;   /* equilibrium column zeroed (kinematic.py:613-620)     */
} bfq_desc;

/* Per-plan facts for reporting / tests. */
typedef struct bfq_plan_info {
  int32_t n_k, n_q, n_t;
  int64_t n_g, n_s;
  int32_t folded;             /* slot-symmetry folding active for Q(f,f)              */
  int32_t cells_per_cta;      /* symmetric kernel                                     */
  int32_t warps_per_cta;
  int32_t stages;
  int32_t smem_bytes;
  int32_t items_per_tile;     /* CTAs per cell tile                                   */
  double exec_macs_per_cell;  /* DMMA MACs actually issued per cell, incl. padding    */
  double operator_bytes;      /* device bytes of the uploaded operator                */
  double useful_macs_per_cell; /* MACs of the evaluated (folded) channels without tile
                                  or row padding: stage 1 rows x n_k^2 (n_k(n_k+1)/2 on
                                  self-symmetric channels) + stage 2 slices x n_k x K     */
} bfq_plan_info;

int bfq_plan_create(const bfq_desc* desc, int device, bfq_plan** out);
/* Native BFCT reader (cache.py:21-39 layout, CRC-32 checked) + upload. */
int bfq_plan_create_bfct(const char* path, int device, bfq_plan** out);
int bfq_plan_destroy(bfq_plan* plan);
int bfq_plan_get_info(const bfq_plan* plan, bfq_plan_info* info);

/* Algorithmic work per cell: flops = 2*(N_G*n_k^2 + N_S*n_k^3),
 * bytes = 16*n_dof (read f, write Q). */
int bfq_plan_work(const bfq_plan* plan, double* flops_per_cell, double* bytes_per_cell);

/* Q(f2, f3) for n_cells cells.  DEVICE pointers on the plan's device, layout
 * (n_cells, n_k, n_q) fp64 C-contiguous.  f3 == f2 (or f3 == NULL) selects
 * Q(f,f).  Stream-ordered on `stream` (a cudaStream_t, NULL = legacy default),
 * no host synchronisation, no allocation.  q must not overlap f2 or f3: CTAs
 * of one cell tile still read its cells while others already write Q (BFQ_EINVAL). */
int bfq_eval(const bfq_plan* plan, const double* f2, const double* f3, double* q,
             int64_t n_cells, void* stream);

/* Same contract on HOST buffers: H2D, evaluate, D2H in pipelined chunks.
 * Blocks until q is written.  Pinned host buffers are copied asynchronously;
 * pageable ones are staged chunk by chunk through pinned buffers owned by the
 * plan (the host memcpy overlaps the device work of the chunks in flight).
 * q must not overlap f2 or f3 (BFQ_EINVAL). */
int bfq_eval_host(const bfq_plan* plan, const double* f2, const double* f3, double* q,
                  int64_t n_cells);

/* One classical RK4 step of dc/dt = Q(c,c) on device state y (n_cells, n_k, n_q):
 * y <- y + dt/6 (k1 + 2k2 + 2k3 + k4).  `work` must hold 3*n_cells*n_dof doubles
 * (device).  `flag` is a device int32 set to 1 if any new state entry is not
 * finite (the harness.py:103-107 divergence check, read back by the caller). */
int bfq_rk4_step(const bfq_plan* plan, double* y, double* work, int64_t n_cells,
                 double dt, int32_t* flag, void* stream);

/* Moments per cell (basis.py:346-363): out[cell] = {mass, px, py, pz, energy}. */
int bfq_moments(const bfq_plan* plan, const double* c, double* out, int64_t n_cells,
                void* stream);

/* Projection of drifting Maxwellians M_{u,T}(v) = (2 pi T)^{-3/2} exp(-|v-u|^2/2T)
 * onto the basis (basis.project, basis.py:262-299), one cell per (u_i, T_i):
 *   c_klm = (2/sqrt(pi)) e^{-|u|^2/2T} Y_lm(u^) sum_j w_j i_l(v_j |u|/T) phi_kl(v_j),
 *   v_j = sqrt(2 T x_j),
 * the angular integral done in closed form by the addition theorem.  (x_j, w_j)
 * is a generalised Gauss-Laguerre rule (alpha = 1/2) of n_rule points (HOST
 * arrays).  u [n][3], temp [n], out [n][n_k][n_q] and the optional additive
 * noise [n][n_k][n_q] (may be NULL) are DEVICE pointers; stream-ordered. */
int bfq_project_maxwellians(int32_t k_max, int32_t l_max, const double* rule_x, const double* rule_w,
                            int32_t n_rule, const double* u, const double* temp, const double* noise,
                            double* out, int64_t n, void* stream);

/* General batched projection basis.project(f, cfg, order) (basis.py:262-299)
 * of distributions SAMPLED on the reference's product grid: n_v radial
 * (generalised Gauss-Laguerre) x n_t polar (Gauss-Legendre) x n_p azimuthal
 * (periodic trapezoid) nodes, point order (v, t, p) with p fastest
 * (basis.py:284-290).  The projector owns device copies of the HOST tables
 * that carry the rule weights:
 *   phi_tab    [2 l_max + 1][n_p]  w_p x {1 (row 0), sin(m phi) (row 2m-1), cos(m phi) (row 2m)}
 *   theta_tab  [(l_max+1)(l_max+2)/2][n_t]  w_t x (-1)^m sqrt2 (m > 0) x N_lm P_l^m(cos t), row l(l+1)/2 + m
 *   radial_tab [l_max + 1][k_max + 1][n_v]  phi_kl(v) x the radial weight
 * bfq_project_samples maps samples [n][n_v][n_t][n_p] (DEVICE) to
 * out [n][n_k][n_q] (DEVICE), stream-ordered, one CTA per cell. */
typedef struct bfq_projector bfq_projector;
int bfq_projector_create(int32_t k_max, int32_t l_max, int32_t n_v, int32_t n_t, int32_t n_p,
                         const double* phi_tab, const double* theta_tab, const double* radial_tab, int device,
                         bfq_projector** out);
int bfq_project_samples(const bfq_projector* proj, const double* samples, double* out, int64_t n, void* stream);
int bfq_projector_destroy(bfq_projector* proj);
/* Algorithmic work per cell: flops of the azimuthal, polar and radial sums;
 * bytes = the samples read + the coefficients written. */
int bfq_projector_work(const bfq_projector* proj, double* flops_per_cell, double* bytes_per_cell);
/* Which kernel bfq_project_samples launches for this projector: 1 = the
 * general kernel, 2 = register-tiled W (shapes within its tiles), 3 = 2 with
 * the azimuth folded over the mirror pairs p <-> n_p - p (needs an azimuth
 * table that is even / odd under the mirror, as the reference's trapezoid
 * nodes make it; checked at create).  Negative: invalid handle. */
int bfq_projector_kernel(const bfq_projector* proj);

/* Diagnostic: validate `desc` and build the host-side plan (folding check,
 * tiling, CTA schedule) WITHOUT touching a GPU; fills `info` as
 * bfq_plan_get_info would for a device with `smem_limit` bytes of opt-in
 * shared memory per block.  Used by the CPU test-suite. */
int bfq_host_plan_info(const bfq_desc* desc, int smem_limit, bfq_plan_info* info);

const char* bfq_strerror(int code);
const char* bfq_last_error(void);
/* Provenance: hash of the sources, headers and flags this library was built
 * from (paper_2605_28475_b200/_build.py); the loader compares it with the tree. */
const char* bfq_build_id(void);

#ifdef __cplusplus
}
#endif
#endif /* BFQ_H */
