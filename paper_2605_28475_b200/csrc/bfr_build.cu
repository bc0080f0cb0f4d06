// bfr_build.cu -- R-tensor assembly on sm_100a (include/bfr.h).
//
// What the reference computes (pkg/src/boltzfact/kinematic.py), per channel
// tau = (l1, l2, l3) and per Duffy patch, on the tensor grid
// (E, outer o, Duffy t, deflection chi, azimuth eps):
//
//   p_gain   = Y_l2(0) sum_m b_m(o,t) ReY_{l1 m}(v'(chi,eps,o,t))           :427-445
//   g_j(o,t) = kern(o,t) sum_{chi,eps} w w |v'|^l1 (|v'|^2/2)^j p_gain       :456-464
//   core     = pref[k,E] sum_j mono[k,j] eta_E^j g_j(o,t)                     :466-471
//   gain     = sum_{E,o,t} core phi_l2(v) phi_l3(w) env                        :480-507
//   loss_f/s = sum phi_l1 phi_l2 phi_l3 env * loss_kern (fast / slow branch)
//
// and combines R = scale * sym(gain + swap(gain) - loss_f - loss_s) (:552-570).
//
// B200 restructuring (same integrals, different association):
//  * the chi/eps integral of |v'|^(l1+2j) ReY_{l1 m} depends on l1 only, not on
//    (l2, l3): one table A[l1,m,j](o,t) per patch (k_atab) replaces a per-channel
//    azimuth/deflection contraction; g_j is then a short m-sum (k_gstack);
//  * every channel integral is a triple product over the flattened point axis
//    p = (E, o[, t]):  out[r,a,b] = sum_p X[r,p] U[a,p] W[b,p], with rows X =
//    gain / fast-loss / slow-loss integrands (k_xrows) and U, W radial tables.
//    That is a GEMM with M = rows, N = (a,b), K = p, run on the FP64 tensor
//    pipe (DMMA m8n8k4) with the (a,b) operand formed in registers from two
//    staged radial rows (k_tri), split over p with a deterministic reduction.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "bfq.h"
#include "bfr.h"
#include "bfq_internal.h"

using namespace bfq;

namespace {

constexpr int LMX = BFR_LMAX_SUPPORTED;
constexpr int NK_MAX = 17;     // k_tri register tiling covers n_k <= 17
constexpr int PC = 64;         // points per staged chunk in k_tri
constexpr int SROW = PC + 4;   // smem row stride (doubles), = 4 mod 16: conflict-free fragments
constexpr double PI = 3.14159265358979323846;

// fully normalised associated Legendre recurrence coefficients (Condon-Shortley)
//   Ybar_{m,m}   = d_m sqrt(1-x^2) Ybar_{m-1,m-1},   d_m = -sqrt((2m+1)/(2m))
//   Ybar_{m+1,m} = e_m x Ybar_{m,m},                 e_m = sqrt(2m+3)
//   Ybar_{l,m}   = a_lm (x Ybar_{l-1,m} - b_lm Ybar_{l-2,m})
__constant__ double c_ya[(LMX + 1) * (LMX + 1)];
__constant__ double c_yb[(LMX + 1) * (LMX + 1)];
__constant__ double c_yd[LMX + 1];
__constant__ double c_ye[LMX + 1];

__host__ __device__ inline int lm_index(int l, int m) { return l * (l + 1) / 2 + m; }

// N_lm P_l^m(x) for one (l, m), m <= l (basis.py:176-193 sph_harm_theta)
__device__ double ybar(int l, int m, double x) {
  const double sx = sqrt(fmax((1.0 - x) * (1.0 + x), 0.0));
  double pmm = 0.28209479177387814347;  // 1/sqrt(4 pi)
  for (int i = 1; i <= m; ++i) pmm = c_yd[i] * sx * pmm;
  if (l == m) return pmm;
  double p0 = pmm, p1 = c_ye[m] * x * pmm;
  for (int ll = m + 2; ll <= l; ++ll) {
    const double p2 = c_ya[ll * (LMX + 1) + m] * (x * p1 - c_yb[ll * (LMX + 1) + m] * p0);
    p0 = p1;
    p1 = p2;
  }
  return p1;
}

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// ------------------------------------------------------------------ geometry
// per (o,t) point of one patch (kinematic.py:322-362); fields of g[f*n_ot + i]
enum { G_RHO, G_COSB, G_V0, G_W0, G_U0, G_FGEO, G_KERN, G_CX, G_CZ, G_UHX, G_UHZ, G_E1X, G_E1Z,
       G_E2Y, G_NF };

__global__ void k_geom(int patch, const double* ox, const double* tx, int n_o, int n_t,
                       double gamma, double kscale, double fgeo_c, double* g) {
  const int n_ot = n_o * n_t;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_ot) return;
  const int o = i / n_t, t = i - o * n_t;
  const double x = ox[o], tt = tx[t];
  double rho, h, duffy;
  if (patch == 0) {  // rho > h, h = rho t: Jacobian rho, duffy = rho^2 t
    rho = x;
    h = x * tt;
    duffy = rho * rho * tt;
  } else {  // h > rho, rho = h t: duffy = h^2
    h = x;
    rho = x * tt;
    duffy = x * x;
  }
  const double cos_b = 1.0 - 2.0 * (h * h);
  const double sin_b = 2.0 * h * sqrt(fmax(1.0 - h * h, 0.0));
  const double v0 = 1.0 + rho, w0 = 1.0 - rho;
  const double u0 = 2.0 * sqrt(rho * rho + (1.0 - rho * rho) * (h * h));
  const double om = 1.0 - rho * rho;
  const double fgeo = fgeo_c * duffy * (om * om);
  const double cx = 0.5 * w0 * sin_b, cz = 0.5 * (v0 + w0 * cos_b);
  const double su = u0 > 0.0 ? u0 : 1.0;
  const double uhx = -w0 * sin_b / su, uhz = (v0 - w0 * cos_b) / su;
  const double n1 = fabs(uhx);
  const bool deg = n1 < 1e-14;
  const double sn = deg ? 1.0 : n1;
  const double e1x = deg ? 1.0 : -uhz * uhx / sn;
  const double e1z = deg ? 0.0 : uhx * uhx / sn;
  const double e2y = uhz * e1x - uhx * e1z;
  const double kern = kscale * pow(u0, gamma) / (4.0 * PI);
  const double v[G_NF] = {rho, cos_b, v0, w0, u0, fgeo, kern, cx, cz, uhx, uhz, e1x, e1z, e2y};
#pragma unroll
  for (int f = 0; f < G_NF; ++f) g[(size_t)f * n_ot + i] = v[f];
}

// Ybar_{l,m}(cos beta) for all (l,m) at every (o,t): yb[lm][ot]
__global__ void k_ybar_table(const double* g, int n_ot, int L, double* yb) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_ot) return;
  const double x = g[(size_t)G_COSB * n_ot + i];
  const double sx = sqrt(fmax((1.0 - x) * (1.0 + x), 0.0));
  double pmm = 0.28209479177387814347;
  for (int m = 0; m <= L; ++m) {
    if (m > 0) pmm = c_yd[m] * sx * pmm;
    yb[(size_t)lm_index(m, m) * n_ot + i] = pmm;
    if (m == L) break;
    double p0 = pmm, p1 = c_ye[m] * x * pmm;
    yb[(size_t)lm_index(m + 1, m) * n_ot + i] = p1;
    for (int l = m + 2; l <= L; ++l) {
      const double p2 = c_ya[l * (LMX + 1) + m] * (x * p1 - c_yb[l * (LMX + 1) + m] * p0);
      p0 = p1;
      p1 = p2;
      yb[(size_t)lm_index(l, m) * n_ot + i] = p1;
    }
  }
}

// ------------------------------------------------------------------ dd arithmetic
// The reference expands the radial polynomial in monomials (kinematic.py:458-471):
// core_k = pref sum_j mono[k,j] eta^j g_j is an alternating sum whose terms exceed
// the result by ~1e3 at n_k = 13, so any rounding in g_j is amplified that much.
// g_j and the j-sum are therefore carried in double-double (error-free products
// via FMA); the result then differs from the reference only by the reference's
// own fp64 rounding ("R-tensor build: accuracy").
struct dd {
  double hi, lo;
};
__device__ __forceinline__ dd two_prod(double a, double b) {
  const double p = a * b;
  return {p, fma(a, b, -p)};
}
__device__ __forceinline__ dd two_sum(double a, double b) {
  const double s = a + b, bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd fast_two_sum(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  const dd t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = fast_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return fast_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo = fma(a.hi, b.lo, fma(a.lo, b.hi, p.lo));
  return fast_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_mul_d(dd a, double b) {
  dd p = two_prod(a.hi, b);
  p.lo = fma(a.lo, b, p.lo);
  return fast_two_sum(p.hi, p.lo);
}

// ------------------------------------------------------------------ A tables
// A[l1,m,j](o,t) = sum_{chi,eps} w_chi w_eps |v'|^l1 (|v'|^2/2)^j Ybar_{l1 m}(cos th') cos(m phi')
// in double-double.  One CTA (256 threads) per (o,t); the (chi,eps) axis is
// staged ATAB_SC points at a time (kinematic.py:366-380, 448-464):
//  1a  one thread per point: post-collision speed/direction, the dd power row
//      (|v'|^2/2)^j and the dd weight w_chi w_eps;
//  1b  one thread per (point, m): Ybar_{l,m} for l = m..L by the upward
//      recurrence, times cos(m phi') (rounded as the reference rounds it) and
//      the dd weighted radial power w |v'|^l;
//  2   one thread per (row (l1,m), 4 j's): compensated (Dot2) accumulation of
//      the point sum, carried across chunks in shared memory.
constexpr int ATAB_SC = 32;
constexpr int ATAB_JT = 4;

struct AtabParams {
  const double* g;
  int n_ot, L, nk, n_chi, n_eps;
  const double *chi_x, *chi_w, *eps_c, *eps_s, *eps_w;
  double *A_hi, *A_lo;  // [lm][j][ot]
  int fast;             // experiments only (BFR_ATAB_F64): plain fp64 accumulation
};

__host__ __device__ inline size_t atab_smem(int nlm, int nk) {
  const int njt = (nk + ATAB_JT - 1) / ATAB_JT;
  return ((size_t)2 * nlm * (ATAB_SC + 1)                 // yh, yl
          + (size_t)2 * ATAB_SC * njt * ATAB_JT            // vh, vl
          + (size_t)2 * nlm * njt * ATAB_JT                // acc s, c
          + (size_t)6 * ATAB_SC) * 8;                      // per-point scalars
}

__global__ void __launch_bounds__(256) k_atab(AtabParams p) {
  extern __shared__ double sm[];
  const int tid = threadIdx.x, nth = blockDim.x, ot = blockIdx.x;
  const int L = p.L, nlm = lm_index(L, L) + 1, nk = p.nk;
  const int njt = (nk + ATAB_JT - 1) / ATAB_JT, nkp = njt * ATAB_JT;
  constexpr int SC = ATAB_SC, SS = ATAB_SC + 1;
  double* yh = sm;                         // [nlm][SS]
  double* yl = yh + (size_t)nlm * SS;
  double* vh = yl + (size_t)nlm * SS;      // [SC][nkp]
  double* vl = vh + (size_t)SC * nkp;
  double* as = vl + (size_t)SC * nkp;      // [nlm][nkp]
  double* ac = as + (size_t)nlm * nkp;
  double* pv = ac + (size_t)nlm * nkp;     // per point: vps, ctp, sx, c1, w_hi, w_lo
  const int n_ot = p.n_ot;
  const double cx = p.g[(size_t)G_CX * n_ot + ot], cz = p.g[(size_t)G_CZ * n_ot + ot];
  const double hu = 0.5 * p.g[(size_t)G_U0 * n_ot + ot];
  const double uhx = p.g[(size_t)G_UHX * n_ot + ot], uhz = p.g[(size_t)G_UHZ * n_ot + ot];
  const double e1x = p.g[(size_t)G_E1X * n_ot + ot], e1z = p.g[(size_t)G_E1Z * n_ot + ot];
  const double e2y = p.g[(size_t)G_E2Y * n_ot + ot];
  for (int o = tid; o < nlm * nkp; o += nth) as[o] = ac[o] = 0.0;
  const int ns = p.n_chi * p.n_eps;
  for (int s0 = 0; s0 < ns; s0 += SC) {
    // 1a: per point
    if (tid < SC) {
      const int s = s0 + tid;
      double vps = 0.0, ctp = 1.0, c1 = 1.0;
      dd w = {0.0, 0.0};
      if (s < ns) {
        const int ic = s / p.n_eps, ie = s - ic * p.n_eps;
        const double cc = p.chi_x[ic];
        const double sch = sqrt(fmax(1.0 - cc * cc, 0.0));
        const double ce = p.eps_c[ie], se = p.eps_s[ie];
        const double vx = cx + hu * (cc * uhx + sch * ce * e1x);
        const double vy = hu * sch * se * e2y;
        const double vz = cz + hu * (cc * uhz + sch * ce * e1z);
        vps = sqrt(vx * vx + vy * vy + vz * vz);
        ctp = fmin(fmax(vps > 0.0 ? vz / vps : 1.0, -1.0), 1.0);
        c1 = cos(atan2(vy, vx));
        w = two_prod(p.chi_w[ic], p.eps_w[ie]);
      }
      dd step = two_prod(vps, vps);
      step.hi *= 0.5;
      step.lo *= 0.5;
      dd pw = {s < ns ? 1.0 : 0.0, 0.0};
      for (int j = 0; j < nkp; ++j) {
        vh[tid * nkp + j] = j < nk ? pw.hi : 0.0;
        vl[tid * nkp + j] = j < nk ? pw.lo : 0.0;
        pw = dd_mul(pw, step);
      }
      double* q = pv + tid * 6;
      q[0] = vps;
      q[1] = ctp;
      q[2] = sqrt(fmax((1.0 - ctp) * (1.0 + ctp), 0.0));
      q[3] = c1;
      q[4] = w.hi;
      q[5] = w.lo;
    }
    __syncthreads();
    // 1b: per (point, m)
    for (int it = tid; it < SC * (L + 1); it += nth) {
      const int m = it / SC, sl = it - m * SC;
      const double* q = pv + sl * 6;
      const double vps = q[0], ctp = q[1], sx = q[2], c1 = q[3];
      double cm = 1.0, cm1 = 1.0, cm2 = 0.0, pmm = 0.28209479177387814347;
      dd wl = {q[4], q[5]};
      for (int i = 1; i <= m; ++i) {
        cm = i == 1 ? c1 : 2.0 * c1 * cm1 - cm2;
        cm2 = cm1;
        cm1 = cm;
        pmm = c_yd[i] * sx * pmm;
        wl = dd_mul_d(wl, vps);
      }
      dd t = dd_mul_d(wl, pmm * cm);
      yh[(size_t)lm_index(m, m) * SS + sl] = t.hi;
      yl[(size_t)lm_index(m, m) * SS + sl] = t.lo;
      if (m < L) {
        double p0 = pmm, p1 = c_ye[m] * ctp * pmm;
        wl = dd_mul_d(wl, vps);
        t = dd_mul_d(wl, p1 * cm);
        yh[(size_t)lm_index(m + 1, m) * SS + sl] = t.hi;
        yl[(size_t)lm_index(m + 1, m) * SS + sl] = t.lo;
        for (int l = m + 2; l <= L; ++l) {
          const double p2 = c_ya[l * (LMX + 1) + m] * (ctp * p1 - c_yb[l * (LMX + 1) + m] * p0);
          p0 = p1;
          p1 = p2;
          wl = dd_mul_d(wl, vps);
          t = dd_mul_d(wl, p1 * cm);
          yh[(size_t)lm_index(l, m) * SS + sl] = t.hi;
          yl[(size_t)lm_index(l, m) * SS + sl] = t.lo;
        }
      }
    }
    __syncthreads();
    // 2: Dot2 accumulation, 4 j's per thread item
    for (int it = tid; it < nlm * njt; it += nth) {
      const int r = it / njt, j0 = (it - r * njt) * ATAB_JT;
      double sa[ATAB_JT], ca[ATAB_JT];
#pragma unroll
      for (int u = 0; u < ATAB_JT; ++u) {
        sa[u] = as[r * nkp + j0 + u];
        ca[u] = ac[r * nkp + j0 + u];
      }
      const double* yrh = yh + (size_t)r * SS;
      const double* yrl = yl + (size_t)r * SS;
      if (p.fast) {
        for (int q = 0; q < SC; ++q)
#pragma unroll
          for (int u = 0; u < ATAB_JT; ++u) sa[u] = fma(yrh[q], vh[q * nkp + j0 + u], sa[u]);
      } else {
#pragma unroll 4
        for (int q = 0; q < SC; ++q) {
          const double a_h = yrh[q], a_l = yrl[q];
#pragma unroll
          for (int u = 0; u < ATAB_JT; ++u) {
            const double b_h = vh[q * nkp + j0 + u], b_l = vl[q * nkp + j0 + u];
            const dd pr = two_prod(a_h, b_h);
            const dd sm2 = two_sum(sa[u], pr.hi);
            sa[u] = sm2.hi;
            ca[u] = fma(a_h, b_l, fma(a_l, b_h, ca[u] + (pr.lo + sm2.lo)));
          }
        }
      }
#pragma unroll
      for (int u = 0; u < ATAB_JT; ++u) {
        as[r * nkp + j0 + u] = sa[u];
        ac[r * nkp + j0 + u] = ca[u];
      }
    }
    __syncthreads();
  }
  for (int o = tid; o < nlm * nk; o += nth) {
    const int r = o / nk, j = o - r * nk;
    const dd v = fast_two_sum(as[r * nkp + j], ac[r * nkp + j]);
    p.A_hi[(size_t)o * n_ot + ot] = v.hi;
    p.A_lo[(size_t)o * n_ot + ot] = v.lo;
  }
}

// --------------------------------------------------------------- radial/env
// phi[(l*2 + which)*nk + k][p] at speed sqrt(eta_E) * (1 +- rho)  (basis.py:123-141,
// kinematic.py:304-319); env[p] = w_E eta^2 exp(-eta rho^2) w_o [w_t f_geo]
struct RadParams {
  const double* g;
  const double *eta, *w_e, *ow, *tw, *norms;
  int patch, n_e, n_o, n_t, nq, L, nk;
  long long P, PS;
  double *phi, *env;
};

__global__ void k_radial(RadParams p) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.P) return;
  const int E = (int)(i / p.nq), q = (int)(i - (long long)E * p.nq);
  const int n_ot = p.n_o * p.n_t;
  const int ot = p.patch == 0 ? q * p.n_t : q;  // patch 0: radial speeds use t = 0 (rho = outer node)
  const int o = p.patch == 0 ? q : q / p.n_t;
  const double eta = p.eta[E];
  const double rho = p.g[(size_t)G_RHO * n_ot + ot];
  const double se = sqrt(eta);
  double env = p.w_e[E] * (eta * eta) * exp(-eta * (rho * rho));
  if (p.patch == 0) env *= p.ow[o];
  else env *= (p.ow[o] * p.tw[q - o * p.n_t]) * p.g[(size_t)G_FGEO * n_ot + ot];
  p.env[i] = env;
  for (int which = 0; which < 2; ++which) {
    const double v = se * (which == 0 ? p.g[(size_t)G_V0 * n_ot + ot] : p.g[(size_t)G_W0 * n_ot + ot]);
    const double x = 0.5 * v * v;
    for (int l = 0; l <= p.L; ++l) {
      const double a = l + 0.5;
      const double sc = pow(v, (double)l);
      double* out = p.phi + (size_t)((l * 2 + which) * p.nk) * p.PS + i;
      double lm1 = 1.0, lk = 1.0 + a - x;
      out[0] = p.norms[l * p.nk] * sc * 1.0;
      if (p.nk > 1) out[(size_t)p.PS] = p.norms[l * p.nk + 1] * sc * lk;
      for (int k = 1; k < p.nk - 1; ++k) {
        const double ln = ((2 * k + a + 1 - x) * lk - (k + a) * lm1) / (k + 1);
        lm1 = lk;
        lk = ln;
        out[(size_t)(k + 1) * p.PS] = p.norms[l * p.nk + k + 1] * sc * lk;
      }
    }
  }
}

// --------------------------------------------------------------- per channel
// gq[c][j][q] = kern Y_l2(0) sum_m b_m A[l1,m,j]  (patch 1: (o,t); patch 0: the
// Duffy integral sum_t (.) f_geo w_t folded in, q = o), and the loss kernel
// lq[c][q] = 2 pi sum(w_chi) kern p_loss (patch 0: Duffy-integrated likewise)
struct GsParams {
  const double *g, *A_hi, *A_lo, *yb, *tw, *w3j;
  const int32_t* trip;
  const int32_t* chan;  // batch slot -> channel
  int nb;               // slots in the batch (gq holds hi then lo halves)
  int patch, n_o, n_t, nq, L, nk;
  double swc;  // 2 pi sum(w_chi)
  double *gq, *lq;
};

__global__ void k_gstack(GsParams p) {
  // one thread per (q, j): patch 0 loops over the Duffy axis, so (q) alone is too little parallelism
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (i >= p.nq * p.nk) return;
  const int jj = i / p.nq, q = i - jj * p.nq;
  const int tau = p.chan[c];
  const int l1 = p.trip[3 * tau], l2 = p.trip[3 * tau + 1], l3 = p.trip[3 * tau + 2];
  const int mm = min(l1, l3);
  const int n_ot = p.n_o * p.n_t;
  const double* w3 = p.w3j + (size_t)tau * (p.L + 1);
  const double zon1 = sqrt((2 * l1 + 1) / (4.0 * PI)), zon2 = sqrt((2 * l2 + 1) / (4.0 * PI));
  const int t_n = p.patch == 0 ? p.n_t : 1;
  {
    const int j = jj;
    dd acc = {0.0, 0.0};
    for (int tt = 0; tt < t_n; ++tt) {
      const int ot = p.patch == 0 ? q * p.n_t + tt : q;
      dd s = {0.0, 0.0};
      for (int m = 0; m <= mm; ++m) {
        const double w = w3[m];
        if (w == 0.0) continue;
        const double fac = (m == 0 ? 1.0 : 2.0) * ((m & 1) ? -1.0 : 1.0);
        const double b = fac * w * p.yb[(size_t)lm_index(l3, m) * n_ot + ot];
        const size_t ai = ((size_t)lm_index(l1, m) * p.nk + j) * n_ot + ot;
        s = dd_add(s, dd_mul_d({p.A_hi[ai], p.A_lo[ai]}, b));
      }
      dd gv = dd_mul_d(dd_mul_d(s, zon2), p.g[(size_t)G_KERN * n_ot + ot]);
      if (p.patch == 0) acc = dd_add(acc, dd_mul_d(dd_mul_d(gv, p.g[(size_t)G_FGEO * n_ot + ot]), p.tw[tt]));
      else acc = gv;
    }
    const dd g = fast_two_sum(acc.hi, acc.lo);
    p.gq[((size_t)c * p.nk + j) * p.nq + q] = g.hi;  // kept double-double into the monomial sum
    p.gq[((size_t)(p.nb + c) * p.nk + j) * p.nq + q] = g.lo;
  }
  if (jj != 0) return;
  double la = 0.0;
  for (int tt = 0; tt < t_n; ++tt) {
    const int ot = p.patch == 0 ? q * p.n_t + tt : q;
    const double pl = zon1 * zon2 * w3[0] * p.yb[(size_t)lm_index(l3, 0) * n_ot + ot];
    const double lk = p.swc * p.g[(size_t)G_KERN * n_ot + ot] * pl;
    if (p.patch == 0) la += p.g[(size_t)G_FGEO * n_ot + ot] * lk * p.tw[tt];
    else la = lk;
  }
  p.lq[(size_t)c * p.nq + q] = la;
}

// X[c][r][p]: r < nk gain integrand core*env, nk <= r < 2nk fast loss phi_l1(v) lenv,
// 2nk <= r < 3nk slow loss phi_l1(w) lenv
struct XrParams {
  const double *gq, *lq, *me, *pf, *phi, *env;
  const int32_t* trip;
  const int32_t* chan;  // batch slot -> channel
  int nb;               // slots in the batch (gq holds hi then lo halves)
  int n_e, nq, nk, L;
  long long P, PS;
  double* X;
};

template <int NK>
__global__ void k_xrows(XrParams p) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (i >= p.P) return;
  const int nk = NK > 0 ? NK : p.nk;
  const int tau = p.chan[c];
  const int l1 = p.trip[3 * tau];
  const int E = (int)(i / p.nq), q = (int)(i - (long long)E * p.nq);
  constexpr int NA = NK > 0 ? NK : NK_MAX;
  double gj[NA], gl[NA];
#pragma unroll
  for (int j = 0; j < NA; ++j) {
    gj[j] = j < nk ? p.gq[((size_t)c * nk + j) * p.nq + q] : 0.0;
    gl[j] = j < nk ? p.gq[((size_t)(p.nb + c) * nk + j) * p.nq + q] : 0.0;
  }
  const double env = p.env[i];
  const double lenv = env * p.lq[(size_t)c * p.nq + q];
  const double* me = p.me + ((size_t)l1 * p.n_e + E) * nk * nk;
  double* X = p.X + (size_t)c * 3 * nk * p.PS + i;
  const double* pv = p.phi + (size_t)((l1 * 2 + 0) * nk) * p.PS + i;
  const double* pw = p.phi + (size_t)((l1 * 2 + 1) * nk) * p.PS + i;
  const double* pf = p.pf + ((size_t)l1 * p.n_e + E) * nk;
  for (int k = 0; k < nk; ++k) {
    // compensated dot product (Ogita-Rump-Oishi Dot2) of the alternating monomial sum
    double s = 0.0, comp = 0.0;
#pragma unroll
    for (int j = 0; j < NA; ++j)
      if (j < nk) {
        // the reference rounds mono * eta^j before its j-sum (einsum path jE,kj->jkE); so do we
        const double ch = me[k * nk + j];
        const dd pr = two_prod(ch, gj[j]);
        const dd sm = two_sum(s, pr.hi);
        s = sm.hi;
        comp = fma(ch, gl[j], comp + (pr.lo + sm.lo));
      }
    X[(size_t)k * p.PS] = ((s + comp) * pf[k]) * env;
    X[(size_t)(nk + k) * p.PS] = pv[(size_t)k * p.PS] * lenv;
    X[(size_t)(2 * nk + k) * p.PS] = pw[(size_t)k * p.PS] * lenv;
  }
}

// ------------------------------------------------------------ contraction
// Jobs are ordered (l2, l3) = (x, y) pairs: every channel (l1, x, y) contributes
// its gain and fast-loss rows (U = phi_x(v), W = phi_y(w)), every channel
// (l1, y, x) its slow-loss rows -- those share the same U (x) W product with
// (a, b) swapped.  A job's rows are cut into blocks of <= MT 8-row tiles;
//   part[block][split][row][a*nk+b] = sum_{p in split} X[rowtab[row], p] U[a,p] W[b,p].
struct TriBlock {
  int x, y, row0, nrows;  // rows [row0, row0+nrows) of the batch row table
};

struct TriParams {
  const double *X, *phi;
  const TriBlock* blocks;
  const int32_t* rowtab;  // batch row -> X row (slot*3nk + offset)
  int nk, S, PR, rows_max;
  long long P, PS;
  double* part;  // [block][split][rows_max][nk*nk]
};

// NW warps per CTA: the (a,b) column tiles are dealt tile = warp + NW i, so NW x NPW
// should just cover ceil(n_k^2 / 8) tiles -- 22 at n_k = 13: 11 warps x 2 (8 warps x 3
// left warps 6 and 7 with two tiles where the others have three, idle a third of
// every chunk behind the per-chunk barrier)
template <int MT, int NPW, int NW = 8>
__global__ void __launch_bounds__(NW * 32, 2) k_tri(TriParams p) {
  extern __shared__ double sm[];
  const TriBlock blk = p.blocks[blockIdx.y];
  const int split = blockIdx.x;
  const int nk = p.nk, nn = nk * nk;
  const int rows = blk.nrows, mtn = (rows + 7) / 8;
  const int rs = rows + 2 * nk;  // staged rows per chunk
  const int* rt = p.rowtab + blk.row0;
  const double* U = p.phi + (size_t)((blk.x * 2 + 0) * nk) * p.PS;
  const double* W = p.phi + (size_t)((blk.y * 2 + 1) * nk) * p.PS;
  const long long pb = (long long)split * p.PR;
  const long long pe = min((long long)p.P, pb + p.PR);
  const int nchunk = (int)((pe - pb + PC - 1) / PC);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r0 = lane >> 2, kq = lane & 3;
  const int ntiles = (nn + 7) / 8;

  int xoff[MT];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) xoff[mt] = min(mt * 8 + r0, rows - 1) * SROW;
  int uoff[NPW], woff[NPW];
#pragma unroll
  for (int i = 0; i < NPW; ++i) {
    const int n = min((warp + NW * i) * 8 + r0, nn - 1);
    const int a = n / nk, b = n - a * nk;
    uoff[i] = (rows + a) * SROW;
    woff[i] = (rows + nk + b) * SROW;
  }
  double acc[MT][NPW][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int i = 0; i < NPW; ++i) acc[mt][i][0] = acc[mt][i][1] = 0.0;

  const int stage_d = (p.rows_max + 2 * nk) * SROW;
  auto load_chunk = [&](int ch, int st) {
    const long long p0 = pb + (long long)ch * PC;
    double* dst = sm + st * stage_d;
    const int nv = rs * (PC / 2);
    for (int v = threadIdx.x; v < nv; v += blockDim.x) {
      const int r = v / (PC / 2), cc = (v - r * (PC / 2)) * 2;
      const double* src = r < rows ? p.X + (size_t)rt[r] * p.PS
                                   : (r < rows + nk ? U + (size_t)(r - rows) * p.PS
                                                    : W + (size_t)(r - rows - nk) * p.PS);
      const long long pp = p0 + cc;
      const int bytes = pp + 2 <= pe ? 16 : (pp < pe ? 8 : 0);
      cp_async16(dst + r * SROW + cc, src + (bytes ? pp : 0), bytes);
    }
    cp_async_commit();
  };

  // three-stage ring, one barrier per chunk: the load of chunk ch+2 is issued after
  // the barrier that ends chunk ch-1's reads of the same stage
  if (nchunk > 0) load_chunk(0, 0);
  if (nchunk > 1) load_chunk(1, 1);
  for (int ch = 0; ch < nchunk; ++ch) {
    if (ch + 1 < nchunk) cp_async_wait1();
    else cp_async_wait0();
    __syncthreads();
    if (ch + 2 < nchunk) load_chunk(ch + 2, (ch + 2) % 3);
    const double* s = sm + (ch % 3) * stage_d;
#pragma unroll 2
    for (int kk = 0; kk < PC / 4; ++kk) {
      const int col = kk * 4 + kq;
      double a[MT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) a[mt] = s[xoff[mt] + col];
#pragma unroll
      for (int i = 0; i < NPW; ++i) {
        if (warp + NW * i < ntiles) {
          const double b = s[uoff[i] + col] * s[woff[i] + col];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt)
            if (mt < mtn) dmma884(acc[mt][i][0], acc[mt][i][1], a[mt], b);
        }
      }
    }
  }
  double* out = p.part + ((size_t)blockIdx.y * p.S + split) * (size_t)p.rows_max * nn;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int row = mt * 8 + r0;
    if (row >= rows) continue;
#pragma unroll
    for (int i = 0; i < NPW; ++i) {
      const int tile = warp + NW * i;
      if (tile >= ntiles) continue;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = tile * 8 + 2 * kq + e;
        if (n < nn) out[(size_t)row * nn + n] = acc[mt][i][e];
      }
    }
  }
}

// halves[h][tau][k][ab] += sum over splits (fixed order); rowmap[i] = (tau*3 + h)*nk + k,
// negative (-1 - code) when the job computed the transposed (b, a) block
__global__ void k_reduce(const double* part, const TriBlock* blocks, int nblk, const int32_t* rowmap, int nk,
                         int S, int rows_max, int n_t, double* halves) {
  const int nn = nk * nk;
  const long long tot = (long long)nblk * rows_max * nn;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= tot) return;
  const int ab = (int)(i % nn);
  const int row = (int)((i / nn) % rows_max);
  const int b = (int)(i / ((long long)nn * rows_max));
  const TriBlock blk = blocks[b];
  if (row >= blk.nrows) return;
  int code = rowmap[blk.row0 + row];
  const bool trans = code < 0;
  if (trans) code = -1 - code;
  const double* src = part + ((size_t)b * S) * (size_t)rows_max * nn + (size_t)row * nn + ab;
  double s = 0.0;
  for (int sp = 0; sp < S; ++sp) s += src[(size_t)sp * rows_max * nn];
  const int k = code % nk, th = code / nk, h = th % 3, tau = th / 3;
  const int a = ab / nk, bb = ab - a * nk;
  const int dst = trans ? bb * nk + a : ab;
  halves[(((size_t)h * n_t + tau) * nk + k) * nn + dst] += s;
}

// full[tau] = gain[tau] + gain[swap]^T(2,3) - (loss_f + loss_s)[tau]  (kinematic.py:552-558)
__global__ void k_full(const double* halves, const int32_t* swap, int n_t, int nk, double* full) {
  const int nn = nk * nk, n3 = nn * nk;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)n_t * n3) return;
  const int tau = (int)(i / n3), r = (int)(i - (long long)tau * n3);
  const int k = r / nn, a = (r / nk) % nk, b = r % nk;
  const size_t hs = (size_t)n_t * n3;
  const double g = halves[i];
  const double gs = halves[(size_t)swap[tau] * n3 + (size_t)k * nn + b * nk + a];
  const double lf = halves[hs + i], ls = halves[2 * hs + i];
  full[i] = g + gs - (lf + ls);
}

// R[k][a][b][tau] = scale * 0.5 (full[tau] + full[swap]^T)  (kinematic.py:559-569)
__global__ void k_final(const double* full, const int32_t* swap, const double* scale, int n_t, int nk,
                        double* r) {
  const int nn = nk * nk, n3 = nn * nk;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)n_t * n3) return;
  const int tau = (int)(i / n3), rr = (int)(i - (long long)tau * n3);
  const int k = rr / nn, a = (rr / nk) % nk, b = rr % nk;
  const double f = full[i];
  const double fs = full[(size_t)swap[tau] * n3 + (size_t)k * nn + b * nk + a];
  r[(size_t)rr * n_t + tau] = scale[tau] * (0.5 * (f + fs));
}

// ---------------------------------------------------------------- host side
typedef void (*TriKernel)(TriParams);

template <int MT>
TriKernel pick_tri_npw(int npw) {
  switch (npw) {
    case 1: return k_tri<MT, 1>;
    case 2: return k_tri<MT, 2>;
    case 3: return k_tri<MT, 3>;
    case 4: return k_tri<MT, 4>;
    case 5: return k_tri<MT, 5>;
  }
  return nullptr;
}

TriKernel pick_tri(int mt, int npw) {
  switch (mt) {
    case 1: return pick_tri_npw<1>(npw);
    case 2: return pick_tri_npw<2>(npw);
    case 3: return pick_tri_npw<3>(npw);
    case 4: return pick_tri_npw<4>(npw);
    case 5: return pick_tri_npw<5>(npw);
  }
  return nullptr;
}

typedef void (*XrKernel)(XrParams);
XrKernel pick_xrows(int nk) {
  switch (nk) {
    case 3: return k_xrows<3>;
    case 5: return k_xrows<5>;
    case 7: return k_xrows<7>;
    case 9: return k_xrows<9>;
    case 11: return k_xrows<11>;
    case 13: return k_xrows<13>;
    case 15: return k_xrows<15>;
    case 17: return k_xrows<17>;
  }
  return k_xrows<0>;
}

struct DevBuf {
  std::vector<void*> ptrs;
  ~DevBuf() {
    for (void* q : ptrs) cudaFree(q);
  }
  template <class T>
  T* alloc(size_t n) {
    void* q = nullptr;
    if (cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(T)) != cudaSuccess) return nullptr;
    ptrs.push_back(q);
    return (T*)q;
  }
  void release(void* q) {
    for (auto& x : ptrs)
      if (x == q) {
        cudaFree(x);
        x = nullptr;
      }
  }
};

template <class T>
int upload(DevBuf& db, const T* host, size_t n, T** out) {
  *out = db.alloc<T>(n);
  if (!*out) {
    set_error("device allocation failed");
    return BFQ_ENOMEM;
  }
  if (n && cudaMemcpy(*out, host, n * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess) {
    set_error("host-to-device copy failed");
    return BFQ_ECUDA;
  }
  return BFQ_OK;
}

int set_ybar_constants() {
  static bool done = false;  // device-independent values, but constant memory is per device
  (void)done;
  std::vector<double> ya((LMX + 1) * (LMX + 1), 0.0), yb((LMX + 1) * (LMX + 1), 0.0), yd(LMX + 1, 0.0),
      ye(LMX + 1, 0.0);
  for (int m = 0; m <= LMX; ++m) {
    yd[m] = m > 0 ? -std::sqrt((2.0 * m + 1.0) / (2.0 * m)) : 1.0;
    ye[m] = std::sqrt(2.0 * m + 3.0);
    for (int l = m + 2; l <= LMX; ++l) {
      const double l2 = (double)l * l, m2 = (double)m * m, lp = (double)(l - 1) * (l - 1);
      ya[l * (LMX + 1) + m] = std::sqrt((4.0 * l2 - 1.0) / (l2 - m2));
      yb[l * (LMX + 1) + m] = std::sqrt((lp - m2) / (4.0 * lp - 1.0));
    }
  }
  if (cudaMemcpyToSymbol(c_ya, ya.data(), ya.size() * 8) != cudaSuccess ||
      cudaMemcpyToSymbol(c_yb, yb.data(), yb.size() * 8) != cudaSuccess ||
      cudaMemcpyToSymbol(c_yd, yd.data(), yd.size() * 8) != cudaSuccess ||
      cudaMemcpyToSymbol(c_ye, ye.data(), ye.size() * 8) != cudaSuccess) {
    set_error("constant upload failed");
    return BFQ_ECUDA;
  }
  return BFQ_OK;
}

#define BFR_TRY(expr)                                                               \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      set_error(std::string(#expr) + ": " + cudaGetErrorString(e_));               \
      return BFQ_ECUDA;                                                             \
    }                                                                               \
  } while (0)

#define BFR_LAUNCH_CHECK(name)                                                      \
  do {                                                                              \
    ++n_launch;                                                                     \
    cudaError_t e_ = cudaGetLastError();                                            \
    if (e_ != cudaSuccess) {                                                        \
      set_error(std::string("kernel launch " name ": ") + cudaGetErrorString(e_));  \
      return BFQ_ECUDA;                                                             \
    }                                                                               \
  } while (0)

inline unsigned blocks_for(long long n, int bs) { return (unsigned)((n + bs - 1) / bs); }

int assemble(const bfr_desc& d, int device, double* r_out, double* halves_out, bfr_stats* st) {
  const int L = d.l_max, nk = d.k_max + 1, n_t = d.n_t;
  const int nlm = lm_index(L, L) + 1, nn = nk * nk, n3 = nn * nk;
  int ndev = 0;
  BFR_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) {
    set_error("device ordinal out of range");
    return BFQ_EINVAL;
  }
  // restore the caller's current device on every exit path (torch keeps its own)
  struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
      cudaGetDevice(&prev);
      if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
      int cur = -1;
      cudaGetDevice(&cur);
      if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
  } guard(device);
  int rc;
  if ((rc = set_ybar_constants())) return rc;
  DevBuf db;
  int32_t *d_trip, *d_swap;
  double *d_w3j, *d_scale, *d_eta, *d_we, *d_chix, *d_chiw, *d_epsc, *d_epss, *d_epsw, *d_norms, *d_me;
  (void)d_norms;
  if ((rc = upload(db, d.triplets, (size_t)3 * n_t, &d_trip))) return rc;
  if ((rc = upload(db, d.swap, (size_t)n_t, &d_swap))) return rc;
  if ((rc = upload(db, d.w3j, (size_t)n_t * (L + 1), &d_w3j))) return rc;
  if ((rc = upload(db, d.chan_scale, (size_t)n_t, &d_scale))) return rc;
  if ((rc = upload(db, d.e_x, (size_t)d.n_e, &d_eta))) return rc;
  if ((rc = upload(db, d.e_w, (size_t)d.n_e, &d_we))) return rc;
  if ((rc = upload(db, d.chi_x, (size_t)d.n_chi, &d_chix))) return rc;
  if ((rc = upload(db, d.chi_w, (size_t)d.n_chi, &d_chiw))) return rc;
  std::vector<double> ec(d.n_eps), es(d.n_eps);
  for (int i = 0; i < d.n_eps; ++i) {
    ec[i] = std::cos(d.eps_x[i]);
    es[i] = std::sin(d.eps_x[i]);
  }
  if ((rc = upload(db, ec.data(), ec.size(), &d_epsc))) return rc;
  if ((rc = upload(db, es.data(), es.size(), &d_epss))) return rc;
  if ((rc = upload(db, d.eps_w, (size_t)d.n_eps, &d_epsw))) return rc;
  if ((rc = upload(db, d.norms, (size_t)(L + 1) * nk, &d_norms))) return rc;
  // me[l][E][k][j] = fl(mono[l][k][j] * eta_E^j) and pf[l][E][k] = norms[l][k] * eta_E^(l/2):
  // the reference's own fp64 einsum operands (kinematic.py:466-471; numpy's path rounds
  // mono * eta^j first).  Measured: keeping that product exact moves R further from the
  // reference (N=12 1.2e-12 -> 2.3e-12), so the reference's rounding is reproduced.
  double* d_pf;
  {
    std::vector<double> me((size_t)(L + 1) * d.n_e * nn), pf((size_t)(L + 1) * d.n_e * nk);
    for (int l = 0; l <= L; ++l)
      for (int E = 0; E < d.n_e; ++E) {
        const double eta = d.e_x[E];
        const double eh = l == 0 ? 1.0 : std::pow(eta, 0.5 * l);
        for (int k = 0; k < nk; ++k) {
          pf[((size_t)l * d.n_e + E) * nk + k] = d.norms[l * nk + k] * eh;
          for (int j = 0; j < nk; ++j) {
            const double ep = j == 0 ? 1.0 : (j == 1 ? eta : std::pow(eta, (double)j));
            me[(((size_t)l * d.n_e + E) * nk + k) * nk + j] = d.mono[((size_t)l * nk + k) * nk + j] * ep;
          }
        }
      }
    if ((rc = upload(db, me.data(), me.size(), &d_me))) return rc;
    if ((rc = upload(db, pf.data(), pf.size(), &d_pf))) return rc;
  }
  double swc = 0.0;
  for (int i = 0; i < d.n_chi; ++i) swc += d.chi_w[i];
  swc = swc * 2.0 * PI;
  const double fgeo_c = 4.0 * std::pow(2.0 * PI, -3.0);

  double* halves = db.alloc<double>((size_t)3 * n_t * n3);
  double* full = db.alloc<double>((size_t)n_t * n3);
  double* rdev = db.alloc<double>((size_t)n_t * n3);
  if (!halves || !full || !rdev) {
    set_error("device allocation failed");
    return BFQ_ENOMEM;
  }
  BFR_TRY(cudaMemset(halves, 0, (size_t)3 * n_t * n3 * 8));

  // 8-row tiles per contraction block: 5 while the accumulators (MT x NPW x 2) keep
  // k_tri at <= 128 registers (two CTAs per SM), 3 for the wider n_k = 14..17 tiling
  int npw = ((nn + 7) / 8 + 7) / 8, tri_warps = 8;
  const int MT_BLK = npw <= 3 ? 5 : 3;
  TriKernel tri = pick_tri(MT_BLK, npw);
  // 17..22 column tiles (n_k = 12, 13): 11 warps x 2 tiles instead of 8 x 3
  if ((nn + 7) / 8 > 16 && (nn + 7) / 8 <= 22 && !std::getenv("BFR_TRI_8WARPS")) {
    npw = 2;
    tri_warps = 11;
    tri = k_tri<5, 2, 11>;
  }
  if (!tri) {
    set_error("n_k outside the contraction kernel's tiling (n_k <= 17)");
    return BFQ_EINVAL;
  }
  const int rows_max = 8 * MT_BLK;
  const size_t tri_smem = (size_t)3 * (rows_max + 2 * nk) * SROW * 8;
  BFR_TRY(cudaFuncSetAttribute(tri, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tri_smem));
  XrKernel xr = pick_xrows(nk);
  const size_t atab_sm = atab_smem(nlm, nk);
  {
    int optin = 0;
    BFR_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    if (atab_sm > (size_t)optin) {
      set_error("l_max too large for the angular-table kernel's shared memory");
      return BFQ_EINVAL;
    }
    BFR_TRY(cudaFuncSetAttribute(k_atab, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)atab_sm));
  }

  // per-patch sizes; every buffer is allocated once, before the timed region
  struct PatchDims {
    int n_o, n_t, n_ot, nq, PR, S;
    long long P, PS;
    double *ox, *ow, *tx, *tw;
  } pd[2];
  int max_ot = 0, max_nq = 0, max_S = 0;
  long long max_PS = 0;
  for (int patch = 0; patch < 2; ++patch) {
    PatchDims& q = pd[patch];
    q.n_o = d.n_outer[patch];
    q.n_t = d.n_inner[patch];
    q.n_ot = q.n_o * q.n_t;
    q.nq = patch == 0 ? q.n_o : q.n_ot;
    q.P = (long long)d.n_e * q.nq;
    q.PS = (q.P + 3) / 4 * 4;
    q.PR = q.P >= 16384 * 4 ? 16384 : (int)((q.P + PC - 1) / PC * PC);
    q.S = (int)((q.P + q.PR - 1) / q.PR);
    if ((rc = upload(db, d.outer_x[patch], (size_t)q.n_o, &q.ox))) return rc;
    if ((rc = upload(db, d.outer_w[patch], (size_t)q.n_o, &q.ow))) return rc;
    if ((rc = upload(db, d.inner_x[patch], (size_t)q.n_t, &q.tx))) return rc;
    if ((rc = upload(db, d.inner_w[patch], (size_t)q.n_t, &q.tw))) return rc;
    max_ot = std::max(max_ot, q.n_ot);
    max_nq = std::max(max_nq, q.nq);
    max_S = std::max(max_S, q.S);
    max_PS = std::max(max_PS, q.PS);
    if (st) st->n_points[patch] = q.P;
  }

  // channel batches = unions of unordered (l2, l3) pairs, integrand rows <= ~6 GB
  const size_t xrow_bytes = (size_t)3 * nk * max_PS * 8;
  const int cap = (int)std::max<size_t>(1, std::min<size_t>((size_t)n_t, ((size_t)6 << 30) / xrow_bytes));
  struct Batch {
    std::vector<int32_t> chan, rowtab, rowmap;
    std::vector<TriBlock> blocks;
  };
  std::vector<Batch> batches;
  {
    std::vector<std::vector<int>> by_pair((size_t)(L + 1) * (L + 1));
    for (int t = 0; t < n_t; ++t) by_pair[d.triplets[3 * t + 1] * (L + 1) + d.triplets[3 * t + 2]].push_back(t);
    Batch cur;
    auto flush = [&]() {
      if (cur.chan.empty()) return;
      // slots in (l1, tau) order: consecutive k_gstack CTAs then share one l1's A table in L2
      std::sort(cur.chan.begin(), cur.chan.end());  // channels are enumerated l1-major
      // slots, then the ordered-pair jobs of every pair present
      std::vector<int> slot(n_t, -1);
      for (size_t i = 0; i < cur.chan.size(); ++i) slot[cur.chan[i]] = (int)i;
      for (int x = 0; x <= L; ++x)
        for (int y = 0; y <= L; ++y) {
          const auto& fwd = by_pair[x * (L + 1) + y];  // gain + fast loss rows
          const auto& rev = by_pair[y * (L + 1) + x];  // slow loss rows, transposed
          if (fwd.empty() && rev.empty()) continue;
          if ((!fwd.empty() && slot[fwd[0]] < 0) || (!rev.empty() && slot[rev[0]] < 0)) continue;
          const int row0 = (int)cur.rowtab.size();
          for (int t : fwd)
            for (int h = 0; h < 2; ++h)
              for (int k = 0; k < nk; ++k) {
                cur.rowtab.push_back(slot[t] * 3 * nk + h * nk + k);
                cur.rowmap.push_back((t * 3 + h) * nk + k);
              }
          for (int t : rev)
            for (int k = 0; k < nk; ++k) {
              cur.rowtab.push_back(slot[t] * 3 * nk + 2 * nk + k);
              cur.rowmap.push_back(-1 - ((t * 3 + 2) * nk + k));
            }
          const int nrows = (int)cur.rowtab.size() - row0;
          const int ntile = (nrows + 7) / 8, nblk = (ntile + MT_BLK - 1) / MT_BLK;
          int r = 0;
          for (int bi = 0; bi < nblk; ++bi) {
            const int tiles = (ntile - bi * (ntile / nblk)) > 0 ? (ntile / nblk + (bi < ntile % nblk ? 1 : 0)) : 0;
            const int nr = std::min(tiles * 8, nrows - r);
            if (nr > 0) cur.blocks.push_back({x, y, row0 + r, nr});
            r += nr;
          }
        }
      batches.push_back(std::move(cur));
      cur = Batch();
    };
    for (int x = 0; x <= L; ++x)
      for (int y = x; y <= L; ++y) {
        std::vector<int> members = by_pair[x * (L + 1) + y];
        if (y != x) members.insert(members.end(), by_pair[y * (L + 1) + x].begin(), by_pair[y * (L + 1) + x].end());
        if (members.empty()) continue;
        if (!cur.chan.empty() && (int)(cur.chan.size() + members.size()) > cap) flush();
        cur.chan.insert(cur.chan.end(), members.begin(), members.end());
      }
    flush();
  }
  int max_chan = 0, max_rows = 0, max_blocks = 0;
  for (const Batch& bt : batches) {
    max_chan = std::max(max_chan, (int)bt.chan.size());
    max_rows = std::max(max_rows, (int)bt.rowtab.size());
    max_blocks = std::max(max_blocks, (int)bt.blocks.size());
  }
  double* geo = db.alloc<double>((size_t)G_NF * max_ot);
  double* yb = db.alloc<double>((size_t)nlm * max_ot);
  double* A = db.alloc<double>((size_t)2 * nlm * nk * max_ot);  // hi, lo
  double* env = db.alloc<double>((size_t)max_PS);
  double* phi = db.alloc<double>((size_t)(L + 1) * 2 * nk * max_PS);
  double* X = db.alloc<double>((size_t)max_chan * 3 * nk * max_PS);
  double* gq = db.alloc<double>((size_t)2 * max_chan * nk * max_nq);
  double* lq = db.alloc<double>((size_t)max_chan * max_nq);
  double* part = db.alloc<double>((size_t)max_blocks * max_S * rows_max * nn);
  if (!geo || !yb || !A || !env || !phi || !X || !gq || !lq || !part) {
    set_error("device allocation failed");
    return BFQ_ENOMEM;
  }
  // batch tables, uploaded once
  std::vector<int32_t*> d_chan(batches.size()), d_rowtab(batches.size()), d_rowmap(batches.size());
  std::vector<TriBlock*> d_blocks(batches.size());
  for (size_t bi = 0; bi < batches.size(); ++bi) {
    if ((rc = upload(db, batches[bi].chan.data(), batches[bi].chan.size(), &d_chan[bi]))) return rc;
    if ((rc = upload(db, batches[bi].rowtab.data(), batches[bi].rowtab.size(), &d_rowtab[bi]))) return rc;
    if ((rc = upload(db, batches[bi].rowmap.data(), batches[bi].rowmap.size(), &d_rowmap[bi]))) return rc;
    if ((rc = upload(db, batches[bi].blocks.data(), batches[bi].blocks.size(), &d_blocks[bi]))) return rc;
  }
  // Row tails [P, PS) are never read: k_tri zero-fills past the last point.

  const int n_batches = 2 * (int)batches.size();
  std::vector<cudaEvent_t> evs(2 + 2 * n_batches, nullptr);
  struct EvGuard {
    std::vector<cudaEvent_t>& e;
    ~EvGuard() {
      for (auto x : e)
        if (x) cudaEventDestroy(x);
    }
  } evg{evs};
  for (auto& e : evs) BFR_TRY(cudaEventCreate(&e));
  cudaEvent_t ev0 = evs[0], ev1 = evs[1];
  BFR_TRY(cudaEventRecord(ev0));
  double exec_macs = 0.0, alg_macs = 0.0, xbytes = 0.0;
  long long n_launch = 0;
  int ib = 0;

  for (int patch = 0; patch < 2; ++patch) {
    const PatchDims& q = pd[patch];
    const int n_o = q.n_o, n_tt = q.n_t, n_ot = q.n_ot, nq = q.nq, PR = q.PR, S = q.S;
    const long long P = q.P, PS = q.PS;
    k_geom<<<blocks_for(n_ot, 128), 128>>>(patch, q.ox, q.tx, n_o, n_tt, d.gamma, d.kernel_scale, fgeo_c, geo);
    BFR_LAUNCH_CHECK("k_geom");
    k_ybar_table<<<blocks_for(n_ot, 128), 128>>>(geo, n_ot, L, yb);
    BFR_LAUNCH_CHECK("k_ybar_table");
    {
      AtabParams ap{geo, n_ot, L, nk, d.n_chi, d.n_eps, d_chix, d_chiw, d_epsc, d_epss, d_epsw,
                    A, A + (size_t)nlm * nk * n_ot, std::getenv("BFR_ATAB_F64") ? 1 : 0};
      k_atab<<<n_ot, 256, atab_sm>>>(ap);
      BFR_LAUNCH_CHECK("k_atab");
    }
    {
      RadParams rp{geo, d_eta, d_we, q.ow, q.tw, d_norms, patch, d.n_e, n_o, n_tt, nq, L, nk, P, PS, phi, env};
      k_radial<<<blocks_for(P, 128), 128>>>(rp);
      BFR_LAUNCH_CHECK("k_radial");
    }
    for (size_t bi = 0; bi < batches.size(); ++bi, ++ib) {
      const Batch& bt = batches[bi];
      const int cb = (int)bt.chan.size(), nblk = (int)bt.blocks.size();
      GsParams gp{geo, A, A + (size_t)nlm * nk * n_ot, yb, q.tw, d_w3j, d_trip, d_chan[bi], cb, patch, n_o, n_tt,
                  nq, L, nk, swc, gq, lq};
      k_gstack<<<dim3(blocks_for((long long)nq * nk, 128), cb), 128>>>(gp);
      BFR_LAUNCH_CHECK("k_gstack");
      XrParams xp{gq, lq, d_me, d_pf, phi, env, d_trip, d_chan[bi], cb, d.n_e, nq, nk, L, P, PS, X};
      xr<<<dim3(blocks_for(P, 128), cb), 128>>>(xp);
      BFR_LAUNCH_CHECK("xr");
      BFR_TRY(cudaEventRecord(evs[2 + 2 * ib]));
      TriParams tp{X, phi, d_blocks[bi], d_rowtab[bi], nk, S, PR, rows_max, P, PS, part};
      tri<<<dim3(S, nblk), tri_warps * 32, tri_smem>>>(tp);
      BFR_LAUNCH_CHECK("tri");
      BFR_TRY(cudaEventRecord(evs[3 + 2 * ib]));
      k_reduce<<<blocks_for((long long)nblk * rows_max * nn, 256), 256>>>(part, d_blocks[bi], nblk, d_rowmap[bi],
                                                                             nk, S, rows_max, n_t, halves);
      BFR_LAUNCH_CHECK("k_reduce");
      for (const TriBlock& tb : bt.blocks)
        exec_macs += (double)S * PR * 64.0 * ((tb.nrows + 7) / 8) * ((nn + 7) / 8);
      alg_macs += (double)cb * P * 3.0 * nk * nn;
      xbytes += (double)cb * 3 * nk * P * 8.0 * 2.0;
    }
  }
  k_full<<<blocks_for((long long)n_t * n3, 256), 256>>>(halves, d_swap, n_t, nk, full);
  BFR_LAUNCH_CHECK("k_full");
  k_final<<<blocks_for((long long)n_t * n3, 256), 256>>>(full, d_swap, d_scale, n_t, nk, rdev);
  BFR_LAUNCH_CHECK("k_final");
  BFR_TRY(cudaEventRecord(ev1));
  BFR_TRY(cudaEventSynchronize(ev1));
  float ms_tot = 0.f;
  BFR_TRY(cudaEventElapsedTime(&ms_tot, ev0, ev1));
  double ms_contract = 0.0;
  for (int i = 0; i < ib; ++i) {
    float ms = 0.f;
    BFR_TRY(cudaEventElapsedTime(&ms, evs[2 + 2 * i], evs[3 + 2 * i]));
    ms_contract += ms;
  }
  BFR_TRY(cudaMemcpy(r_out, rdev, (size_t)n_t * n3 * 8, cudaMemcpyDeviceToHost));
  if (halves_out) BFR_TRY(cudaMemcpy(halves_out, halves, (size_t)3 * n_t * n3 * 8, cudaMemcpyDeviceToHost));
  if (st) {
    st->ms_total = ms_tot;
    st->ms_contract = ms_contract;
    st->contract_macs = exec_macs;
    st->alg_macs = alg_macs;
    st->x_bytes = xbytes;
    st->launches = n_launch;
  }
  return BFQ_OK;
}

}  // namespace

extern "C" int bfr_assemble(const bfr_desc* desc, int device, double* r_out, double* halves,
                            bfr_stats* stats) {
  if (!desc || !r_out) {
    set_error("null argument");
    return BFQ_EINVAL;
  }
  const bfr_desc& d = *desc;
  if (d.k_max < 0 || d.l_max < 0 || d.l_max > LMX || d.k_max + 1 > NK_MAX || d.n_t <= 0 || d.n_e <= 0 ||
      d.n_chi <= 0 || d.n_eps <= 0 || !d.triplets || !d.swap || !d.w3j || !d.chan_scale || !d.e_x ||
      !d.e_w || !d.chi_x || !d.chi_w || !d.eps_x || !d.eps_w || !d.mono || !d.norms) {
    set_error("invalid R-assembly descriptor (k_max+1 <= 17, l_max <= 24, all tables required)");
    return BFQ_EINVAL;
  }
  for (int p = 0; p < 2; ++p)
    if (d.n_outer[p] <= 0 || d.n_inner[p] <= 0 || !d.outer_x[p] || !d.outer_w[p] || !d.inner_x[p] ||
        !d.inner_w[p]) {
      set_error("invalid patch rule");
      return BFQ_EINVAL;
    }
  for (int t = 0; t < d.n_t; ++t) {
    const int* tr = d.triplets + 3 * t;
    if (tr[0] < 0 || tr[1] < 0 || tr[2] < 0 || tr[0] > d.l_max || tr[1] > d.l_max || tr[2] > d.l_max ||
        d.swap[t] < 0 || d.swap[t] >= d.n_t) {
      set_error("channel table out of range");
      return BFQ_EINVAL;
    }
  }
  if (stats) std::memset(stats, 0, sizeof(*stats));
  return assemble(d, device, r_out, halves, stats);
}
