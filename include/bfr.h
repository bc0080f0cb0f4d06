/*
 * bfr.h -- C ABI of the B200-native R-tensor assembler.
 *
 * Replaces the reference's one-time operator build on CPU:
 *
 *   bfr_assemble  <- kinematic.assemble_r_tensor(cfg, grid, kernel_scale=...)
 *                    (pkg/src/boltzfact/kinematic.py:521-570), i.e. every
 *                    _AssemblyContext.channel_half / _patch_half integral
 *                    (kinematic.py:390-510) plus the full-plane combination,
 *                    slot-(2,3) symmetrisation and channel scale (:552-570).
 *                    The null-space corrections (apply_conservation /
 *                    apply_detailed_balance, :580-620) are plain zeroing and
 *                    stay on the host side (paper_2605_28475_b200/rbuild.py).
 *
 * The host passes the small exact tables (quadrature rules, Wigner 3-j values,
 * Laguerre monomial coefficients, radial norms, channel list) -- the same
 * quantities the reference computes in quadrature.py / angular.py /
 * basis.py -- and the library evaluates all kinematic grids, harmonics,
 * radial functions and the channel integrals on the device.
 *
 * Conventions as bfq.h: plain pointers, 0 on success, negative BFQ_E* codes
 * (bfq_strerror / bfq_last_error apply).  All pointers are HOST pointers.
 */
#ifndef BFR_H
#define BFR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BFR_LMAX_SUPPORTED 24

typedef struct bfr_desc {
  int32_t k_max, l_max;
  double gamma;         /* VHS exponent, kernel u^gamma/(4 pi)          (kinematic.py:76-90) */
  double kernel_scale;  /* multiplies the kernel                         (kinematic.py:470) */
  /* channels in enumerate_channels order (angular.py:117-131) */
  int32_t n_t;
  const int32_t* triplets;  /* [n_t*3] (l1, l2, l3) */
  const int32_t* swap;      /* [n_t] 0-based index of (l1, l3, l2) */
  const double* w3j;        /* [n_t*(l_max+1)] wigner3j(l1,l2,l3, m,0,-m), m = 0..l_max */
  const double* chan_scale; /* [n_t] _channel_scale(l1,l2,l3) (kinematic.py:513-518) */
  /* quadrature rules (quadrature.py): energy = generalised Gauss-Laguerre with
     a = gamma/2; chi = Gauss-Legendre on [-1,1]; eps = periodic trapezoid;
     patch p (0,1) outer / Duffy rules = Gauss-Legendre on [0,1] */
  int32_t n_e;
  const double *e_x, *e_w;
  int32_t n_chi;
  const double *chi_x, *chi_w;
  int32_t n_eps;
  const double *eps_x, *eps_w;
  int32_t n_outer[2], n_inner[2];
  const double *outer_x[2], *outer_w[2], *inner_x[2], *inner_w[2];
  /* radial constants (basis.py:112-173) */
  const double* mono;   /* [(l_max+1)*n_k*n_k]: L_k^(l+1/2)(x) = sum_j mono[l][k][j] x^j */
  const double* norms;  /* [(l_max+1)*n_k]: radial_norm(k, l) */
} bfr_desc;

typedef struct bfr_stats {
  double ms_total;       /* device time of the whole assembly (CUDA events)      */
  double ms_contract;    /* device time inside the channel-contraction kernels   */
  double contract_macs;  /* executed DMMA multiply-adds of the contraction        */
  double alg_macs;       /* algorithmic multiply-adds (3 n_k^3 per grid point per
                            channel: gain, fast loss, slow loss)                   */
  double x_bytes;        /* bytes of integrand rows written + read by the contraction */
  int64_t n_points[2];   /* contraction points per patch (E x outer [x Duffy])     */
  int64_t launches;      /* kernels launched by this assembly                     */
} bfr_stats;

/* Assemble the raw R tensor (before the null-space corrections) into
   r_out[(n_k, n_k, n_k, n_t)] C-order fp64 (host memory).  If `halves` is not
   NULL it receives the half-plane integrals gain / loss_fast / loss_slow,
   3 x [n_t][n_k][n_k][n_k] (kinematic.py:390-406), for diagnostics. */
int bfr_assemble(const bfr_desc* desc, int device, double* r_out, double* halves,
                 bfr_stats* stats);

#ifdef __cplusplus
}
#endif

#endif /* BFR_H */
