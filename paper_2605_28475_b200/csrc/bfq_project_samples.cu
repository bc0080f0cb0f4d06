// bfq_project_samples.cu -- batched general projection (include/bfq.h,
// bfq_projector_*).  Replaces basis.project(f, cfg, order) (basis.py:262-299)
// for f SAMPLED on the reference's product grid (radial node v slowest, polar
// node t, azimuth p fastest; basis.py:283-290):
//
//   c[k][q(l,m)] = sum_v Rv[v][l][k] sum_t P[l,|m|][t] sum_p f[v][t][p] W[p][col(m)]
//
// with the rule weights folded into the host tables: W = w_p {1, cos m phi,
// sin |m| phi} (col(0) = 0, col(-m) = 2m - 1, col(m) = 2m), P = w_t x the
// real-harmonic polar factor (sign (-1)^m sqrt2 for m != 0, basis.py:244-258),
// Rv = phi_kl(v) x the radial weight (basis.py:279-281, :292-298).
//
// B200 mapping.  The azimuthal sum is the only one with grid-sized work:
// G[t][col] = sum_p f[t][p] W[p][col] is a GEMM per (cell, v) slab with M = t,
// N = 2 l_max + 1, K = p, run on DMMA.8x8x4 (FP64 tensor pipe).  One CTA per
// cell walks its samples in t-chunks of 32 rows: the polar-table chunk stays in
// shared memory while the (v) slabs of that chunk stream through a ring of
// cp.async buffers (8-byte granules: rows of n_p doubles are not 16-byte
// aligned), so the HBM stream -- the roofline of this kernel at quadrature
// order ~64 -- overlaps the DMMAs.  The polar and radial sums (O(n_q n_t) and
// O(n_q n_k) per slab) run on DFMA out of shared memory, and the radial sum is
// applied per chunk (the whole map is linear), so no per-v intermediate is kept.
// The coefficient accumulator lives in shared memory: deterministic.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "bfq.h"
#include "bfq_device.cuh"
#include "bfq_internal.h"

using namespace bfq;

struct bfq_projector {
  int device = 0;
  int nk = 0, L = 0, nq = 0, nv = 0, nt = 0, np = 0;
  int ncol = 0, ntile = 0, ks = 0, sp = 0, nbuf = 0, nchunk = 0;
  size_t smem = 0;
  double* wfrag = nullptr;  // [ks][ntile][32] B fragments of W (zero padded)
  double* ptab = nullptr;   // [nchunk][(L+1)(L+2)/2][TC] polar table, t-chunked, zero padded
  double* rtab = nullptr;   // [nv][L+1][nk] radial table
};

namespace {

constexpr int TC = 32;        // polar rows per chunk (4 DMMA M-tiles)
constexpr int TCP = TC + 1;   // row stride of the polar-table chunk: odd, so the threads of
                              // the polar sum (one (l, |m|) row each) hit distinct banks
constexpr int PS_THREADS = 256;
constexpr int MAXT = 7;       // N tiles of the azimuthal GEMM: 2 l_max + 1 <= 56 (l_max <= 27)
constexpr int RAD_MAX = 24;   // coefficient entries per thread: n_k n_q <= 24 x 256 (bfq_projector_create)

struct PsParams {
  const double* f;
  double* out;
  long long n;
  int nk, L, nq, nv, nt, np, ncol, ntile, ks, sp, nbuf, nchunk, npl;
  const double* wfrag;
  const double* ptab;
  const double* rtab;
  int gs;  // row stride of the G tile (doubles)
};

__device__ __forceinline__ void cp_async8(uint32_t dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <int NT>  // N tiles of the azimuthal GEMM (ceil((2 l_max + 1) / 8)): no predicated-off DMMAs
__global__ void __launch_bounds__(PS_THREADS, 1) k_project_samples(const PsParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const long long cell = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, r0 = lane >> 2, kq = lane & 3;
  const int nrv = (p.L + 1) * p.nk;               // radial table of one v, staged with its slab
  const int slab = TC * p.sp + (nrv + 1) / 2 * 2;  // doubles per ring slot: samples | radial table
  double* buf = reinterpret_cast<double*>(smem_raw);  // [nbuf][TC][sp]
  double* wf = buf + (size_t)p.nbuf * slab;        // [ks][ntile][32]
  double* pt = wf + (size_t)p.ks * p.ntile * 32;   // [npl][TCP] polar chunk
  double* g = pt + (size_t)p.npl * TCP;            // [2][TC][gs] azimuthal sums of the chunk (two K halves)
  double* acc = g + (size_t)2 * TC * p.gs;         // [nk][nq]   coefficients of the cell
  double* aq = acc + (size_t)p.nk * p.nq;          // [nq]       polar sums of the chunk
  for (int i = tid; i < p.ks * p.ntile * 32; i += PS_THREADS) wf[i] = p.wfrag[i];
  for (int i = tid; i < p.nbuf * slab; i += PS_THREADS) buf[i] = 0.0;  // zero padding rows/columns
  for (int i = tid; i < p.nk * p.nq; i += PS_THREADS) acc[i] = 0.0;
  __syncthreads();

  const double* fc = p.f + cell * (long long)p.nv * p.nt * p.np;
  const int nsteps = p.nchunk * p.nv;  // (chunk outer, v inner)
  auto issue = [&](int s) {
    if (s < nsteps) {
      const int c = s / p.nv, v = s - c * p.nv;
      const int t0 = c * TC, rows = min(TC, p.nt - t0);
      const double* src = fc + ((long long)v * p.nt + t0) * p.np;
      const uint32_t dst = smem_u32(buf + (size_t)(s % p.nbuf) * slab);
      const double* rsrc = p.rtab + (size_t)v * nrv;
      for (int i = tid; i < nrv; i += PS_THREADS) cp_async8(dst + (uint32_t)(TC * p.sp + i) * 8u, rsrc + i);
      int r = tid / p.np, col = tid - r * p.np;  // walk (row, column) without a division per element
      const int dr = PS_THREADS / p.np, dc = PS_THREADS - dr * p.np;
      for (int i = tid; i < rows * p.np; i += PS_THREADS) {
        cp_async8(dst + (uint32_t)(r * p.sp + col) * 8u, src + i);
        r += dr;
        col += dc;
        if (col >= p.np) {
          col -= p.np;
          ++r;
        }
      }
    }
    cp_commit();  // possibly empty group: keeps the wait count uniform
  };
  for (int s = 0; s < p.nbuf - 1; ++s) issue(s);

  const int mt = warp & 3;  // M tile (8 polar rows) of this warp
  // this thread's entries (k, q) of the coefficient block, with l(q), for the radial sums
  int rad_i[RAD_MAX], rad_q[RAD_MAX], rad_lk[RAD_MAX];
#pragma unroll
  for (int j = 0; j < RAD_MAX; ++j) {
    const int i = tid + j * PS_THREADS;
    rad_i[j] = i < p.nk * p.nq ? i : -1;
    const int k = i / p.nq, q = i - k * p.nq;
    int l = (int)sqrtf((float)q);
    while (l * l > q) --l;
    while ((l + 1) * (l + 1) <= q) ++l;
    rad_q[j] = q;
    rad_lk[j] = l * p.nk + k;
  }
  for (int s = 0; s < nsteps; ++s) {
    const int c = s / p.nv, v = s - c * p.nv;
    if (v == 0) {  // new chunk: its polar table
      __syncthreads();
      for (int i = tid; i < p.npl * TC; i += PS_THREADS) {
        const int row = i / TC;
        pt[row * TCP + (i - row * TC)] = p.ptab[(size_t)c * p.npl * TC + i];
      }
    }
    issue(s + p.nbuf - 1);
    if (p.nbuf == 3) cp_wait<2>();
    else cp_wait<1>();
    __syncthreads();
    // ---- azimuthal GEMM: G[t][col] = sum_p f[t][p] W[p][col] (DMMA.8x8x4).
    // Warp (mt, kh): M tile mt (8 polar rows) x every N tile, half kh of the
    // k-steps -- each A fragment (the samples) feeds all N tiles, and the two
    // K halves land in separate G buffers that the polar sum adds.
    const double* bs = buf + (size_t)(s % p.nbuf) * slab;
    {
      const int kh = warp >> 2, kmid = (p.ks + 1) / 2;
      const int k0 = kh ? kmid : 0, k1 = kh ? p.ks : kmid;
      const uint32_t arow = smem_u32(bs + (size_t)(8 * mt + r0) * p.sp + kq);
      const uint32_t bw = smem_u32(wf + lane);
      double cacc[NT][2];
#pragma unroll
      for (int j = 0; j < NT; ++j) cacc[j][0] = cacc[j][1] = 0.0;
      // plain (non-volatile) shared loads: the slab and W are stable between the
      // barriers, so the compiler may hoist the next k-steps' loads over the DMMAs
#pragma unroll 4
      for (int k = k0; k < k1; ++k) {
        const double a = lds_ro(arow + (uint32_t)(4 * k) * 8u);
        const uint32_t bk = bw + (uint32_t)(k * p.ntile * 32) * 8u;
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma884(cacc[j][0], cacc[j][1], a, lds_ro(bk + (uint32_t)(j * 32) * 8u));
      }
      double* gr = g + (size_t)kh * TC * p.gs + (size_t)(8 * mt + r0) * p.gs + 2 * kq;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        gr[8 * j] = cacc[j][0];
        gr[8 * j + 1] = cacc[j][1];
      }
    }
    __syncthreads();
    // ---- polar sum of the chunk: aq[q] = sum_t P[l,|m|][t] G[t][col(m)]
    for (int q = tid; q < p.nq; q += PS_THREADS) {
      int l = (int)sqrtf((float)q);
      while (l * l > q) --l;
      while ((l + 1) * (l + 1) <= q) ++l;
      const int m = q - l * l - l, am = m < 0 ? -m : m;
      const int col = m == 0 ? 0 : (m < 0 ? 2 * am - 1 : 2 * am);
      const double* prow = pt + (size_t)(l * (l + 1) / 2 + am) * TCP;
      double a = 0.0;
#pragma unroll 8
      for (int t = 0; t < TC; ++t) a = fma(prow[t], g[(size_t)t * p.gs + col] + g[(size_t)(TC + t) * p.gs + col], a);
      aq[q] = a;
    }
    __syncthreads();
    // ---- radial sum of this (chunk, v): acc[k][q] += Rv[v][l][k] aq[q]
    const double* rv = bs + (size_t)TC * p.sp;  // staged with the slab (no global latency here)
#pragma unroll
    for (int j = 0; j < RAD_MAX; ++j)
      if (rad_i[j] >= 0) acc[rad_i[j]] = fma(rv[rad_lk[j]], aq[rad_q[j]], acc[rad_i[j]]);
    // the next iteration's __syncthreads (after its wait) orders these reads of
    // aq / g before they are rewritten; the ring slot s % nbuf is refilled only
    // by issue(s + nbuf), which follows that barrier
  }
  cp_wait<0>();
  __syncthreads();
  double* oc = p.out + cell * (long long)p.nk * p.nq;
  for (int i = tid; i < p.nk * p.nq; i += PS_THREADS) oc[i] = acc[i];
}

typedef void (*PsKernel)(const PsParams);
PsKernel ps_kernel(int ntile) {
  switch (ntile) {
    case 1: return k_project_samples<1>;
    case 2: return k_project_samples<2>;
    case 3: return k_project_samples<3>;
    case 4: return k_project_samples<4>;
    case 5: return k_project_samples<5>;
    case 6: return k_project_samples<6>;
    default: return k_project_samples<7>;
  }
}

int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DevGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace

extern "C" {

int bfq_projector_create(int32_t k_max, int32_t l_max, int32_t n_v, int32_t n_t, int32_t n_p, const double* phi_tab,
                         const double* theta_tab, const double* radial_tab, int device, bfq_projector** out) {
  if (!out || !phi_tab || !theta_tab || !radial_tab) return fail(BFQ_EINVAL, "null argument");
  *out = nullptr;
  if (k_max < 0 || l_max < 0 || n_v < 1 || n_t < 1 || n_p < 1) return fail(BFQ_EINVAL, "bad sizes");
  if (2 * l_max + 1 > 8 * MAXT) return fail(BFQ_EINVAL, "l_max above the projection kernel's limit (27)");
  if ((k_max + 1) * (l_max + 1) * (l_max + 1) > RAD_MAX * PS_THREADS)
    return fail(BFQ_EINVAL, "n_k n_q above the projection kernel's limit (6144)");
  if (n_t < l_max + 1 || n_p < 2 * l_max + 1)
    return fail(BFQ_EINVAL, "angular grid too small for l_max (basis.py:284-285)");
  DevGuard guard(device);
  auto* pj = new bfq_projector();
  pj->device = device;
  pj->nk = k_max + 1;
  pj->L = l_max;
  pj->nq = (l_max + 1) * (l_max + 1);
  pj->nv = n_v;
  pj->nt = n_t;
  pj->np = n_p;
  pj->ncol = 2 * l_max + 1;
  pj->ntile = (pj->ncol + 7) / 8;
  pj->ks = (n_p + 3) / 4;
  pj->sp = conflict_free_stride_dev(n_p);
  pj->nchunk = (n_t + TC - 1) / TC;
  const int npl = (l_max + 1) * (l_max + 2) / 2;
  const int gs = conflict_free_stride_dev(pj->ntile * 8);
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  auto smem_for = [&](int nbuf) {
    return (size_t)8 * ((size_t)nbuf * (TC * pj->sp + ((l_max + 1) * pj->nk + 1) / 2 * 2) + (size_t)pj->ks * pj->ntile * 32 + (size_t)npl * TC +
                        (size_t)2 * TC * gs + (size_t)pj->nk * pj->nq + pj->nq + (size_t)npl);
  };
  pj->nbuf = smem_for(3) <= (size_t)optin ? 3 : 2;
  pj->smem = smem_for(pj->nbuf);
  if (pj->smem > (size_t)optin) {
    delete pj;
    return fail(BFQ_ESMEM, "projection grid too large for shared memory (order / l_max)");
  }
  // W as DMMA B fragments: lane (r0, kq) of k-step ks, tile nt holds W[4 ks + kq][8 nt + r0]
  std::vector<double> wf((size_t)pj->ks * pj->ntile * 32, 0.0);
  for (int ks = 0; ks < pj->ks; ++ks)
    for (int nt = 0; nt < pj->ntile; ++nt)
      for (int lane = 0; lane < 32; ++lane) {
        const int pp = 4 * ks + (lane & 3), col = 8 * nt + (lane >> 2);
        if (pp < n_p && col < pj->ncol) wf[((size_t)ks * pj->ntile + nt) * 32 + lane] = phi_tab[(size_t)col * n_p + pp];
      }
  // polar table in t-chunks of TC rows: [chunk][(l, |m|)][t]
  std::vector<double> pt((size_t)pj->nchunk * npl * TC, 0.0);
  for (int l = 0; l <= l_max; ++l)
    for (int am = 0; am <= l; ++am) {
      const int row = l * (l + 1) / 2 + am;
      for (int t = 0; t < n_t; ++t)
        pt[((size_t)(t / TC) * npl + row) * TC + t % TC] = theta_tab[(size_t)row * n_t + t];
    }
  // radial table [v][l][k]
  std::vector<double> rt((size_t)n_v * (l_max + 1) * pj->nk);
  for (int l = 0; l <= l_max; ++l)
    for (int k = 0; k < pj->nk; ++k)
      for (int v = 0; v < n_v; ++v)
        rt[((size_t)v * (l_max + 1) + l) * pj->nk + k] = radial_tab[((size_t)l * pj->nk + k) * n_v + v];
  auto up = [&](const std::vector<double>& h, double** d) {
    if (cudaMalloc(d, h.size() * sizeof(double)) != cudaSuccess) return false;
    return cudaMemcpy(*d, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess;
  };
  if (!up(wf, &pj->wfrag) || !up(pt, &pj->ptab) || !up(rt, &pj->rtab)) {
    cudaFree(pj->wfrag);
    cudaFree(pj->ptab);
    cudaFree(pj->rtab);
    delete pj;
    return fail(BFQ_ENOMEM, "device allocation of the projection tables failed");
  }
  if (cudaFuncSetAttribute(ps_kernel(pj->ntile), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pj->smem) !=
      cudaSuccess) {
    bfq_projector_destroy(pj);
    return fail(BFQ_ECUDA, "cannot set the projection kernel's shared memory");
  }
  *out = pj;
  return BFQ_OK;
}

int bfq_projector_destroy(bfq_projector* pj) {
  if (!pj) return BFQ_OK;
  DevGuard guard(pj->device);
  cudaFree(pj->wfrag);
  cudaFree(pj->ptab);
  cudaFree(pj->rtab);
  delete pj;
  return BFQ_OK;
}

int bfq_project_samples(const bfq_projector* pj, const double* samples, double* out, int64_t n, void* stream) {
  if (!pj || (n > 0 && (!samples || !out))) return fail(BFQ_EINVAL, "null argument");
  if (n < 0) return fail(BFQ_EINVAL, "negative batch");
  if (n == 0) return BFQ_OK;
  if (n > 0x7fffffffLL) return fail(BFQ_EINVAL, "too many cells for one launch");
  DevGuard guard(pj->device);
  PsParams p;
  p.f = samples;
  p.out = out;
  p.n = n;
  p.nk = pj->nk;
  p.L = pj->L;
  p.nq = pj->nq;
  p.nv = pj->nv;
  p.nt = pj->nt;
  p.np = pj->np;
  p.ncol = pj->ncol;
  p.ntile = pj->ntile;
  p.ks = pj->ks;
  p.sp = pj->sp;
  p.nbuf = pj->nbuf;
  p.nchunk = pj->nchunk;
  p.npl = (pj->L + 1) * (pj->L + 2) / 2;
  p.wfrag = pj->wfrag;
  p.ptab = pj->ptab;
  p.rtab = pj->rtab;
  p.gs = conflict_free_stride_dev(pj->ntile * 8);
  ps_kernel(pj->ntile)<<<(unsigned)n, PS_THREADS, pj->smem, (cudaStream_t)stream>>>(p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(BFQ_ECUDA, std::string("projection launch: ") + cudaGetErrorString(e));
  return BFQ_OK;
}

int bfq_projector_work(const bfq_projector* pj, double* flops_per_cell, double* bytes_per_cell) {
  if (!pj) return fail(BFQ_EINVAL, "null projector");
  const double pts = (double)pj->nv * pj->nt * pj->np;
  // algorithmic: azimuthal sums (2 l_max + 1 per point) + polar (n_q per (v, t)) + radial (n_k n_q per v)
  if (flops_per_cell)
    *flops_per_cell = 2.0 * (pts * pj->ncol + (double)pj->nv * pj->nt * pj->nq + (double)pj->nv * pj->nk * pj->nq);
  if (bytes_per_cell) *bytes_per_cell = 8.0 * (pts + (double)pj->nk * pj->nq);
  return BFQ_OK;
}

}  // extern "C"
