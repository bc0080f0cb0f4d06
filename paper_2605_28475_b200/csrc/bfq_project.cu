// bfq_project.cu -- batched projection of drifting Maxwellians (include/bfq.h,
// bfq_project_maxwellians).  Replaces basis.project (basis.py:262-299) for the
// input generator of BASELINE configs 2-5: instead of sampling f on the
// reference's (radial x theta x phi) tensor grid, the angular integral is done
// in closed form,
//   exp(v.u/T) = 4 pi sum_lm i_l(v|u|/T) Y_lm(v^) Y_lm(u^),
// leaving a 1-D generalised Gauss-Laguerre sum per (l, k) and cell:
//   c_klm = (2/sqrt(pi)) e^{-|u|^2/2T} Y_lm(u^) sum_j w_j i_l(v_j|u|/T) phi_kl(v_j).
// One CTA per cell: (l, j-chunk) threads build the radial sums, one thread per
// m builds the real harmonics of u^, then all threads write the (k, q) block.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "bfq.h"
#include "bfq_internal.h"

using namespace bfq;

namespace {

constexpr int PJ_THREADS = 128;
constexpr int PJ_LMAX = 24;
constexpr int PJ_NKMAX = 32;

struct ProjParams {
  const double *x, *w;  // rule (device)
  int nr, nk, L;
  const double *u, *temp, *noise;
  double* out;
  long long n;
  const double* norms;  // [(L+1)][nk] radial norms
  const double* ynorm;  // [(L+1)(L+2)/2] N_lm = sqrt((2l+1)/(4pi) (l-m)!/(l+m)!)
};

// modified spherical Bessel i_l(x) by its power series (all terms positive)
__device__ double sph_in(int l, double x) {
  double pre = 1.0;
  for (int i = 1; i <= l; ++i) pre *= x / (2 * i + 1);
  const double y = 0.5 * x * x;
  double t = 1.0, s = 1.0;
  for (int k = 1; k < 400; ++k) {
    t *= y / (k * (2.0 * l + 2.0 * k + 1.0));
    s += t;
    if (t < 1e-18 * s) break;
  }
  return pre * s;
}

__global__ void __launch_bounds__(PJ_THREADS) k_project(ProjParams p) {
  const long long cell = blockIdx.x;
  if (cell >= p.n) return;
  const int L = p.L, nk = p.nk, nq = (L + 1) * (L + 1), tid = threadIdx.x;
  __shared__ double part[PJ_THREADS][PJ_NKMAX];  // per-thread radial partial sums
  __shared__ double ylm[(PJ_LMAX + 1) * (PJ_LMAX + 1)];
  const double ux = p.u[3 * cell], uy = p.u[3 * cell + 1], uz = p.u[3 * cell + 2], T = p.temp[cell];
  const double sp = sqrt(ux * ux + uy * uy + uz * uz);
  // threads (l, jb): l = tid % (L+1), j-chunk jb = tid / (L+1)
  const int nl = L + 1, njb = PJ_THREADS / nl;
  const int l = tid % nl, jb = tid / nl;
  for (int k = 0; k < nk; ++k) part[tid][k] = 0.0;
  if (jb < njb) {
    const double a = l + 0.5;
    for (int j = jb; j < p.nr; j += njb) {
      const double v = sqrt(2.0 * T * p.x[j]);
      const double wb = p.w[j] * sph_in(l, v * (sp / T));
      const double xx = 0.5 * v * v;
      const double vl = pow(v, (double)l);
      double lm1 = 1.0, lk = 1.0 + a - xx;
      part[tid][0] += p.norms[l * nk] * vl * 1.0 * wb;
      if (nk > 1) part[tid][1] += p.norms[l * nk + 1] * vl * lk * wb;
      for (int k = 1; k < nk - 1; ++k) {
        const double ln = ((2 * k + a + 1 - xx) * lk - (k + a) * lm1) / (k + 1);
        lm1 = lk;
        lk = ln;
        part[tid][k + 1] += p.norms[l * nk + k + 1] * vl * lk * wb;
      }
    }
  }
  // real harmonics of u^ (inputs.real_harmonics / basis.real_sph_harm)
  if (tid <= L) {
    const int m = tid;
    double cz = 1.0, phi = 0.0;
    if (sp > 0.0) {
      cz = fmin(fmax(uz / sp, -1.0), 1.0);
      phi = atan2(uy / sp, ux / sp);
    }
    const double sx = sqrt(fmax((1.0 - cz) * (1.0 + cz), 0.0));
    // unnormalised Ferrers functions with the Condon-Shortley phase, upward in l
    double pmm = 1.0;
    for (int i = 1; i <= m; ++i) pmm *= -(2.0 * i - 1.0) * sx;
    double p0 = 0.0, p1 = pmm;
    const double cm = cos(m * phi), sm = sin(m * phi), s2 = (m & 1) ? -1.4142135623730951 : 1.4142135623730951;
    for (int ll = m; ll <= L; ++ll) {
      double pl;
      if (ll == m) pl = pmm;
      else if (ll == m + 1) pl = cz * (2.0 * m + 1.0) * pmm;
      else pl = ((2.0 * ll - 1.0) * cz * p1 - (ll + m - 1.0) * p0) / (ll - m);
      if (ll > m) {
        p0 = p1;
        p1 = pl;
      }
      const double th = p.ynorm[ll * (ll + 1) / 2 + m] * pl;
      if (m == 0) {
        ylm[ll * ll + ll] = th;
      } else {
        ylm[ll * ll + ll + m] = s2 * th * cm;
        ylm[ll * ll + ll - m] = s2 * th * sm;
      }
    }
  }
  __syncthreads();
  const double pref = 1.1283791670955126 * exp(-0.5 * sp * sp / T);  // 2/sqrt(pi)
  double* out = p.out + cell * (long long)nk * nq;
  const double* noise = p.noise ? p.noise + cell * (long long)nk * nq : nullptr;
  for (int i = tid; i < nk * nq; i += PJ_THREADS) {
    const int k = i / nq, q = i - k * nq;
    const int lq = (int)sqrtf((float)q + 0.5f);
    double rad = 0.0;
    for (int b = 0; b < njb; ++b) rad += part[b * nl + lq][k];
    double v = (pref * rad) * ylm[q];
    if (noise) v += noise[i];
    out[i] = v;
  }
}

}  // namespace

extern "C" int bfq_project_maxwellians(int32_t k_max, int32_t l_max, const double* rule_x, const double* rule_w,
                                       int32_t n_rule, const double* u, const double* temp, const double* noise,
                                       double* out, int64_t n, void* stream) {
  if (k_max < 0 || l_max < 0 || l_max > PJ_LMAX || k_max + 1 > PJ_NKMAX || n_rule <= 0 || n < 0 ||
      !rule_x || !rule_w || (n > 0 && (!u || !temp || !out))) {
    set_error("invalid projection arguments (l_max <= 24, n_k <= 32)");
    return BFQ_EINVAL;
  }
  if (n == 0) return BFQ_OK;
  const int nk = k_max + 1, L = l_max;
  std::vector<double> norms((size_t)(L + 1) * nk), yn((size_t)(L + 1) * (L + 2) / 2);
  for (int l = 0; l <= L; ++l) {
    for (int k = 0; k < nk; ++k)
      norms[(size_t)l * nk + k] = std::exp(0.5 * (1.5 * std::log(2.0 * M_PI) + std::lgamma(k + 1.0) -
                                                  (l + 0.5) * std::log(2.0) - std::lgamma(k + l + 1.5)));
    for (int m = 0; m <= l; ++m)
      yn[(size_t)l * (l + 1) / 2 + m] = std::exp(0.5 * (std::log((2.0 * l + 1.0) / (4.0 * M_PI)) +
                                                        std::lgamma(l - m + 1.0) - std::lgamma(l + m + 1.0)));
  }
  cudaStream_t s = (cudaStream_t)stream;
  // small tables: one allocation, copied on the caller's stream, freed after the launch completes
  const size_t nbytes = (2 * (size_t)n_rule + norms.size() + yn.size()) * 8;
  double* tab = nullptr;
  if (cudaMallocAsync((void**)&tab, nbytes, s) != cudaSuccess) {
    set_error("device allocation failed");
    return BFQ_ENOMEM;
  }
  std::vector<double> host(nbytes / 8);
  std::copy(rule_x, rule_x + n_rule, host.begin());
  std::copy(rule_w, rule_w + n_rule, host.begin() + n_rule);
  std::copy(norms.begin(), norms.end(), host.begin() + 2 * n_rule);
  std::copy(yn.begin(), yn.end(), host.begin() + 2 * n_rule + norms.size());
  if (cudaMemcpyAsync(tab, host.data(), nbytes, cudaMemcpyHostToDevice, s) != cudaSuccess) {
    set_error("host-to-device copy failed");
    return BFQ_ECUDA;
  }
  ProjParams pp{tab, tab + n_rule, n_rule, nk, L, u, temp, noise, out, n, tab + 2 * n_rule,
                tab + 2 * n_rule + norms.size()};
  for (long long c0 = 0; c0 < n; c0 += 1LL << 30) {
    ProjParams q = pp;
    q.u = u + 3 * c0;
    q.temp = temp + c0;
    q.noise = noise ? noise + c0 * nk * (long long)(L + 1) * (L + 1) : nullptr;
    q.out = out + c0 * nk * (long long)(L + 1) * (L + 1);
    q.n = std::min<long long>(n - c0, 1LL << 30);
    k_project<<<(unsigned)q.n, PJ_THREADS, 0, s>>>(q);
  }
  cudaError_t e = cudaGetLastError();
  // the host staging vector must outlive the async copy
  cudaStreamSynchronize(s);
  cudaFreeAsync(tab, s);
  if (e != cudaSuccess) {
    set_error(std::string("projection kernel: ") + cudaGetErrorString(e));
    return BFQ_ECUDA;
  }
  return BFQ_OK;
}
