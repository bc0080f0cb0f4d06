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
// cell walks its samples in t-chunks of 32 rows (chunk outer, v inner): the
// polar-table chunk stays in shared memory while the (v) slabs stream through
// a ring of cp.async buffers (8-byte granules: rows of n_p doubles are not
// 16-byte aligned), so the HBM stream overlaps the DMMAs.  The CTA is warp-
// specialized: 8 GEMM warps produce G (and copy the v's radial table) into one
// of two G buffers while 4 epilogue warps consume the other -- the polar sum
// (O(n_q n_t) per slab) and the radial sum (O(n_q n_k)), applied per chunk
// (the whole map is linear), each epilogue thread owning whole coefficient
// columns q in registers.  Deterministic and position independent.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
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
  double* ptab2 = nullptr;  // the same with |m|-major rows (v2 kernels)
  double* rtab = nullptr;   // [nv][L+1][nk] radial table
  // v2 kernel (k_project_v2): used when the shape fits its register tiles
  bool v2 = false;
  int kfull = 0, ks2 = 0, slot2 = 0, nbuf2 = 0, kb2 = 0;
  size_t smem2 = 0;
  double* wreg = nullptr;   // [ntile][ks2][32] A fragments of W^T, K permuted
  // mirror-folded v2 (FOLD): azimuth table even / odd under p <-> n_p - p (checked at create)
  int sms = 1;  // v2 kernels are persistent: one CTA per SM, cells strided over the grid
  bool fold = false, fold_whole = false;
  int kfull3 = 0, ks3 = 0, kb3 = 0, nbuf3 = 0;
  size_t smem3 = 0;
  double* wfold = nullptr;  // [|m| tile][cos, sin][ks3][32] A fragments of the folded W^T
};

namespace {

constexpr int TC = 32;        // polar rows per chunk (4 DMMA M-tiles)
constexpr int TCP = TC + 1;   // row stride of the polar-table chunk: odd, so the threads of
                              // the polar sum (one (l, |m|) row each) hit distinct banks
constexpr int PS_THREADS = 384;  // 8 GEMM warps + 4 epilogue warps
constexpr int MAXT = 7;       // N tiles of the azimuthal GEMM: 2 l_max + 1 <= 56 (l_max <= 27)

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

__device__ __forceinline__ void bar_sync(unsigned id, unsigned n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(unsigned id, unsigned n) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

// Warp roles: warps 0..7 stream the samples (cp.async ring) and run the
// azimuthal GEMM, writing G (and the v's radial table) into one of two G
// buffers; warps 8..11 run the polar and radial sums out of the other buffer.
// Named barriers: BAR_GEMM among the GEMM warps (ring), FULL[b] GEMM -> epilogue
// (buffer b written), EMPTY[b] epilogue -> GEMM (buffer b consumed), BAR_EPI
// among the epilogue warps.
// Azimuthal GEMM of one warp: M tile rows (arow), every k-step, the N tiles
// j = NH, NH + 2, ... (compile-time: no predicated-off DMMAs); `store` runs after
// the accumulation with the warp's C fragments.
template <int NT, int NH, class Store>
__device__ __forceinline__ void azim_gemm(uint32_t arow, uint32_t bw, int ks, int ntile, Store&& store) {
  constexpr int NJ = (NT - NH + 1) / 2;  // may be 0 (NT = 1): the store still runs (barrier)
  double c[NJ > 0 ? NJ : 1][2];
#pragma unroll
  for (int jj = 0; jj < NJ; ++jj) c[jj][0] = c[jj][1] = 0.0;
#pragma unroll 4
  for (int k = 0; k < ks; ++k) {
    const double a = lds_ro(arow + (uint32_t)(4 * k) * 8u);
    const uint32_t bk = bw + (uint32_t)(k * ntile * 32) * 8u;
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj) dmma884(c[jj][0], c[jj][1], a, lds_ro(bk + (uint32_t)((NH + 2 * jj) * 32) * 8u));
  }
  store(c, NH, NJ);
}

constexpr int GEMM_WARPS = 8, EPI_WARPS = 4;
constexpr unsigned BAR_GEMM = 1, BAR_FULL0 = 2, BAR_EMPTY0 = 4, BAR_EPI = 6;
constexpr unsigned NT_ALL = PS_THREADS, NT_GEMM = GEMM_WARPS * 32, NT_EPI = EPI_WARPS * 32;

constexpr int NKMAX_REG = 17;  // register accumulators in the epilogue: n_k <= 17, n_q <= 2 x 128

template <int NT, bool REGACC>  // N tiles of the azimuthal GEMM (ceil((2 l_max + 1) / 8)); coefficient
__global__ void __launch_bounds__(PS_THREADS, 1) k_project_samples(const PsParams p) {  // columns in registers
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const long long cell = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, r0 = lane >> 2, kq = lane & 3;
  const int nrv = (p.L + 1) * p.nk;               // radial table of one v, staged with its slab
  const int slab = TC * p.sp + (nrv + 1) / 2 * 2;  // doubles per ring slot: samples | radial table
  const int gsz = TC * p.gs + (nrv + 1) / 2 * 2;  // doubles per G buffer: G | radial table
  double* buf = reinterpret_cast<double*>(smem_raw);  // [nbuf][slab]
  double* wf = buf + (size_t)p.nbuf * slab;        // [ks][ntile][32]
  double* pt = wf + (size_t)p.ks * p.ntile * 32;   // [npl][TCP] polar chunk
  double* g = pt + (size_t)p.npl * TCP;            // [2][gsz]    G buffers
  double* acc = g + (size_t)2 * gsz;               // [nk][nq]   coefficients of the cell
  int* lq = reinterpret_cast<int*>(acc + (size_t)p.nk * p.nq);  // [nq] l(q)
  for (int i = tid; i < p.ks * p.ntile * 32; i += PS_THREADS) wf[i] = p.wfrag[i];
  for (int i = tid; i < p.nbuf * slab; i += PS_THREADS) buf[i] = 0.0;  // zero padding rows/columns
  for (int i = tid; i < p.nk * p.nq; i += PS_THREADS) acc[i] = 0.0;
  for (int q = tid; q < p.nq; q += PS_THREADS) {
    int l = (int)sqrtf((float)q);
    while (l * l > q) --l;
    while ((l + 1) * (l + 1) <= q) ++l;
    lq[q] = l;
  }
  __syncthreads();
  const int nsteps = p.nchunk * p.nv;  // (chunk outer, v inner)

  if (warp < GEMM_WARPS) {
    // ------------------------------------------------ producer: samples -> G
    const double* fc = p.f + cell * (long long)p.nv * p.nt * p.np;
    auto issue = [&](int s) {
      if (s < nsteps) {
        const int c = s / p.nv, v = s - c * p.nv;
        const int t0 = c * TC, rows = min(TC, p.nt - t0);
        const double* src = fc + ((long long)v * p.nt + t0) * p.np;
        const uint32_t dst = smem_u32(buf + (size_t)(s % p.nbuf) * slab);
        const double* rsrc = p.rtab + (size_t)v * nrv;
        for (int i = tid; i < nrv; i += NT_GEMM) cp_async8(dst + (uint32_t)(TC * p.sp + i) * 8u, rsrc + i);
        int r = tid / p.np, col = tid - r * p.np;  // walk (row, column) without a division per element
        const int dr = NT_GEMM / p.np, dc = NT_GEMM - dr * p.np;
        for (int i = tid; i < rows * p.np; i += NT_GEMM) {
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
    const int mt = warp & 3, nh = warp >> 2;
    const uint32_t bw = smem_u32(wf + lane);
    for (int s = 0; s < nsteps; ++s) {
      issue(s + p.nbuf - 1);
      if (p.nbuf == 3) cp_wait<2>();
      else cp_wait<1>();
      bar_sync(BAR_GEMM, NT_GEMM);  // slab s landed for every producer thread
      const double* bs = buf + (size_t)(s % p.nbuf) * slab;
      // azimuthal GEMM: G[t][col] = sum_p f[t][p] W[p][col] (DMMA.8x8x4); warp
      // (mt, nh): M tile mt (8 polar rows) x the N tiles nh, nh + 2, .., every k-step
      const uint32_t arow = smem_u32(bs + (size_t)(8 * mt + r0) * p.sp + kq);
      const int b = s & 1;
      double* gb = g + (size_t)b * gsz;
      auto store = [&](auto& c, int h, int nj) {
        if (s >= 2) bar_sync(BAR_EMPTY0 + b, NT_ALL);  // the epilogue has consumed buffer b
        double* gr = gb + (size_t)(8 * mt + r0) * p.gs + 2 * kq;
#pragma unroll
        for (int jj = 0; jj < (int)(sizeof(c) / sizeof(c[0])); ++jj)
          if (jj < nj) {
            gr[8 * (h + 2 * jj)] = c[jj][0];
            gr[8 * (h + 2 * jj) + 1] = c[jj][1];
          }
      };
      if (nh == 0) azim_gemm<NT, 0>(arow, bw, p.ks, p.ntile, store);
      else azim_gemm<NT, 1>(arow, bw, p.ks, p.ntile, store);
      for (int i = tid; i < nrv; i += NT_GEMM) gb[TC * p.gs + i] = bs[(size_t)TC * p.sp + i];
      __threadfence_block();
      bar_arrive(BAR_FULL0 + b, NT_ALL);
      // the ring slot s % nbuf is refilled by issue(s + nbuf) in the next
      // iteration, after every producer passed this step's BAR_GEMM and its reads
      bar_sync(BAR_GEMM, NT_GEMM);
    }
    cp_wait<0>();
  } else {
    // ------------------------------------------------ consumer: G -> coefficients
    // each epilogue thread owns whole coefficient columns q (every k): the polar
    // sum a = sum_t P[l,|m|][t] G[t][col(m)] (four partial chains), then the
    // radial sum c[k][q] += Rv[v][l][k] a, accumulated in registers (REGACC) or
    // in shared memory
    const int et = tid - NT_GEMM;
    double racc[REGACC ? 2 : 1][REGACC ? NKMAX_REG : 1];
#pragma unroll
    for (int u = 0; u < (REGACC ? 2 : 1); ++u)
#pragma unroll
      for (int k = 0; k < (REGACC ? NKMAX_REG : 1); ++k) racc[u][k] = 0.0;
    for (int s = 0; s < nsteps; ++s) {
      const int c = s / p.nv, b = s & 1;
      if (s % p.nv == 0) {  // new chunk: its polar table
        bar_sync(BAR_EPI, NT_EPI);
        for (int i = et; i < p.npl * TC; i += NT_EPI) {
          const int row = i / TC;
          pt[row * TCP + (i - row * TC)] = p.ptab[(size_t)c * p.npl * TC + i];
        }
      }
      bar_sync(BAR_FULL0 + b, NT_ALL);  // buffer b written (also orders the pt stores above)
      const double* gb = g + (size_t)b * gsz;
      const double* rv = gb + (size_t)TC * p.gs;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int q = et + u * NT_EPI;
        if (!REGACC && u > 0) break;
        for (int qq = q; qq < p.nq; qq += (REGACC ? p.nq : 2 * NT_EPI)) {  // REGACC: one pass
          const int l = lq[qq], m = qq - l * l - l, am = m < 0 ? -m : m;
          const int col = m == 0 ? 0 : (m < 0 ? 2 * am - 1 : 2 * am);
          const double* prow = pt + (size_t)(l * (l + 1) / 2 + am) * TCP;
          const double* g0 = gb + col;
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
          for (int t = 0; t < TC; t += 4) {
            a0 = fma(prow[t], g0[(size_t)t * p.gs], a0);
            a1 = fma(prow[t + 1], g0[(size_t)(t + 1) * p.gs], a1);
            a2 = fma(prow[t + 2], g0[(size_t)(t + 2) * p.gs], a2);
            a3 = fma(prow[t + 3], g0[(size_t)(t + 3) * p.gs], a3);
          }
          const double a = (a0 + a1) + (a2 + a3);
          const double* rvl = rv + l * p.nk;
          if constexpr (REGACC) {
#pragma unroll
            for (int k = 0; k < NKMAX_REG; ++k)
              if (k < p.nk) racc[u][k] = fma(rvl[k], a, racc[u][k]);
          } else {
            for (int k = 0; k < p.nk; ++k) acc[(size_t)k * p.nq + qq] = fma(rvl[k], a, acc[(size_t)k * p.nq + qq]);
          }
          if (!REGACC) continue;
        }
      }
      __threadfence_block();
      bar_arrive(BAR_EMPTY0 + b, NT_ALL);  // buffer b may be rewritten
    }
    double* oc = p.out + cell * (long long)p.nk * p.nq;
    if constexpr (REGACC) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int q = et + u * NT_EPI;
        if (q < p.nq)
#pragma unroll
          for (int k = 0; k < NKMAX_REG; ++k)
            if (k < p.nk) oc[(size_t)k * p.nq + q] = racc[u][k];
      }
    } else {
      bar_sync(BAR_EPI, NT_EPI);  // every column complete
      for (int i = et; i < p.nk * p.nq; i += NT_EPI) oc[i] = acc[i];
    }
  }
}

// ---------------------------------------------------------------- v2 kernel
// The same three sums with the operand traffic cut to what the FP64 tensor
// pipe needs (the v1 kernel above is shared-memory-wavefront bound, ncu ~60%):
//
// * azimuthal GEMM transposed, G^T[col][t] = sum_p W^T[col][p] f[t][p]: the A
//   operand W^T is the same for every slab, so each GEMM warp keeps the
//   fragments of ONE column tile and ONE part of the K axis in REGISTERS and
//   loads only the B fragments f[t][p] of the chunk's four polar tiles -- one
//   shared load per DMMA (v1: 1.5) and four independent accumulator chains per
//   warp.  The KP partial products of a column tile are added in a fixed order
//   (deterministic) by the part-0 warp, which stores G;
// * the slab (TC polar rows x n_p samples, contiguous in HBM) lands with one
//   cp.async.bulk + mbarrier per ring slot, unpadded (v1: 8-byte cp.async per
//   element into padded rows).  Conflict-free gathers without padding come
//   from the K order: inside every 16-sample block, k-step j of lane kq reads
//   sample 16 B + j + 4 kq, so a half-warp (rows r0 = 0..3, kq = 0..3) hits
//   r0 n_p + 4 kq (mod 16): distinct for odd n_p (n_p = 2 n_t + 1 always);
//   the W fragments are permuted the same way on the host.  The last partial
//   block keeps the natural order; its samples past n_p meet W = 0;
// * epilogue: a lane PAIR per (l, |m|) row instead of a thread per coefficient
//   column: each lane of the pair takes every other polar row of the chunk and
//   reads the (sin, cos) pair G[t][col(-m)], G[t][col(+m)] with one 16-byte
//   load (G is stored |m|-major), so P[l,|m|][t] is loaded once for both
//   signs of m; the halves meet by one shuffle, and the lanes split the radial
//   sums (k < h / k >= h) of both columns in registers.  Its DFMAs share the
//   FP64 pipe with the DMMA stream, so it runs on 8 warps with 4 G buffers of
//   slack behind the GEMM.
constexpr int V2_EPI_WARPS = 8;
constexpr int V2_GA = 2 * TC + 6;  // doubles per |m| block of a G buffer ([t][sin, cos]); = 6 (mod 16): the GEMM
                                   // warps' stores (lanes = 8 |m| x 4 t) spread over all banks (16-byte (sin, cos)
                                   // stores of the folded kernel: 4 wavefronts for 512 bytes), and the two or three
                                   // |m| blocks an epilogue warp reads (rows are |m|-major) do not collide
constexpr int V2_TCP = TC + 2;     // row stride of the polar chunk: = 2 (mod 16), the lane pairs
                                   // (row r, half h) of a half-warp read r V2_TCP + h: distinct banks
constexpr int V2_NKMAX = 17;       // n_k <= 17: radial accumulators (half of them per lane) in registers
constexpr int V2_KH = (V2_NKMAX + 1) / 2;
constexpr int V2_MAXBUF = 6;
constexpr int V2_NGB = 4;  // G buffers: the epilogue may lag the GEMM by three slabs
constexpr int V2_HDR = 256;  // mbarriers: full / empty [V2_MAXBUF], gfull / gempty [V2_NGB]
constexpr unsigned V2_BAR_FULL0 = 2, V2_BAR_EMPTY0 = 2 + V2_NGB, V2_BAR_EPI = 2 + 2 * V2_NGB,
                   V2_BAR_RED0 = 3 + 2 * V2_NGB;  // + column tile: the K-part reduction

struct Ps2Params {
  const double* f;
  double* out;
  long long n;
  int nk, L, nq, nv, nt, np, ncol, ks, kfull, nchunk, npl, nbuf, slot;
  const double* wreg;  // [ntile][ks][32] A fragments of W^T, K permuted as above
  const double* ptab;  // [nchunk][npl][TC], rows |m|-major: row(l, a) = a (L + 1) - a (a - 1) / 2 + l - a
  const double* rtab;  // [nv][L+1][nk]
};

// GEMM warps = column tiles x K parts (a multiple of 4: one per scheduler).
// The K axis is split in whole 16-sample blocks (4 k-steps each, immediate
// shared-memory offsets); the natural-order tail steps (n_p mod 16 samples)
// go to the last part, which does not reduce.
template <int NTILE>
struct V2Shape {
  static constexpr int KP = NTILE == 4 ? 2 : 4;
  static constexpr int GW = NTILE * KP;
  static constexpr int THREADS = (GW + V2_EPI_WARPS) * 32;
};
constexpr int V2_TAIL = 4;  // tail k-steps: ceil(15 / 4)

__device__ __forceinline__ void sts128_v(uint32_t addr, double x, double y) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(addr), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ double2 lds128_v(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(addr) : "memory");
  return v;
}

// FOLD (mirror-folded azimuth, NTILE = 4 warp layout): the trapezoid nodes phi_p = 2 pi p / n_p
// make cos(m phi) even and sin(m phi) odd under p <-> n_p - p, so the K axis runs
// over the (n_p - 1) / 2 sample PAIRS: fe = f[p] + f[n_p - p] meets the cos
// columns, fo = f[p] - f[n_p - p] the sin columns, and p = 0 is one extra
// k-step (cos only).  Per pair of samples that is 2 gathers + 2 DADD + 2 DMMA
// for a (cos, sin) tile pair instead of 4 gathers + 4 DMMA: half the tensor
// work and half the shared-memory reads.  A GEMM warp owns one |m| tile (its
// cos and its sin columns), one half of the chunk's polar rows and one K part.
// FOLD = 1: two K parts per (|m| tile, polar half) group, reduced through shared
// memory (any pair count in whole blocks).  FOLD = 2: no K split -- a warp owns
// one |m| tile, ONE polar tile and the whole K axis (<= 4 blocks: the cos and
// sin fragments fill 66 registers), two accumulator chains per warp, which is
// what two warps per scheduler need to keep the pipe fed; no partials, no
// reduction barrier, every GEMM warp stores its own G tile.
template <int NTILE, int KB, int FOLD = 0>  // KB: most 16-sample blocks of any K part (the others may have one fewer)
__global__ void __launch_bounds__(V2Shape<NTILE>::THREADS, 1) k_project_v2(const Ps2Params p) {
  static_assert(!FOLD || NTILE == 4, "the folded kernels use the 8-GEMM-warp layout");
  constexpr int KP = FOLD == 2 ? 1 : V2Shape<NTILE>::KP, GW = V2Shape<NTILE>::GW;
  constexpr int NGRP = GW / KP;  // groups = storing (part 0) warps
  constexpr int NPT = FOLD == 2 ? 1 : 2;  // FOLD: polar tiles per warp
  constexpr int NTH = V2Shape<NTILE>::THREADS, NT_G = GW * 32, NT_E = V2_EPI_WARPS * 32;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);  // [V2_MAXBUF] slab landed
  uint64_t* empty = full + V2_MAXBUF;                         // [V2_MAXBUF] slab released by every GEMM warp
  // G-buffer handoff through mbarriers (one arrival per warp): a GEMM warp waits
  // only for the epilogue's release of the buffer it is about to write, not for
  // its peers (the named FULL / EMPTY barriers re-synchronised all GEMM warps
  // every slab: 14% of their time, ncu)
  uint64_t* gfull = empty + V2_MAXBUF;                        // [V2_NGB] G buffer written by every storing warp
  uint64_t* gempty = gfull + V2_NGB;                          // [V2_NGB] G buffer read by every epilogue warp
  double* ring = reinterpret_cast<double*>(smem_raw + V2_HDR);  // [nbuf][slot]
  const int gsz = (p.L + 1) * V2_GA;
  double* gbuf = ring + (size_t)p.nbuf * p.slot;            // [NGB][L+1][GA]
  double* red = gbuf + (size_t)V2_NGB * gsz;                // [2][NTILE][KP-1][8][32] K-part partials
  double* pt = red + (size_t)2 * NGRP * (KP - 1) * 8 * 32;  // [npl][V2_TCP]
  // persistent: this CTA projects the cells blockIdx.x, blockIdx.x + gridDim.x, ... back to back;
  // the sample ring, the G buffers and every barrier phase run on across cell boundaries, so
  // the next cell's first slabs stream in while the epilogue finishes the current cell
  const long long cell0 = blockIdx.x, cstride = gridDim.x;
  const long long ncl = p.n > cell0 ? (p.n - cell0 + cstride - 1) / cstride : 0;  // cells of this CTA
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, r0 = lane >> 2, kq = lane & 3;
  // the ring starts zeroed: samples past a row (K padding) and the rows of a
  // partial polar chunk are read as finite values that meet W = 0 / P = 0
  for (int i = tid; i < p.nbuf * p.slot / 2; i += NTH) reinterpret_cast<double2*>(ring)[i] = make_double2(0.0, 0.0);
  if (tid == 0) {
    for (int b = 0; b < p.nbuf; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], GW);
    }
    for (int b = 0; b < V2_NGB; ++b) {
      mbar_init(&gfull[b], NGRP);
      mbar_init(&gempty[b], V2_EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // zeros before the bulk copies
  __syncthreads();
  const int nsteps = p.nchunk * p.nv;  // slabs per cell (chunk outer, v inner)
  const long long total = ncl * nsteps;  // slabs of this CTA
  const long long cell_elems = (long long)p.nv * p.nt * p.np;
  // slab (chunk c, radial node v), s = c n_v + v: element range [e0, e0 + cnt) of f;
  // smem index of element e is (e - e0) + m, m = 1 when f + e0 is not 16-byte
  // aligned.  Slab, ring-slot and buffer indices are carried as counters: the
  // integer divisions of s by run-time sizes were 21% of a GEMM warp's time (ncu)
  auto geom = [&](long long cell, int c, int v, long long& e0, int& cnt, int& m) {
    const int t0 = c * TC;
    e0 = cell * cell_elems + ((long long)v * p.nt + t0) * p.np;
    cnt = min(TC, p.nt - t0) * p.np;
    m = (int)((reinterpret_cast<uintptr_t>(p.f + e0) >> 3) & 1);
  };

  if (warp < GW) {
    // ------------------------------------------------ producer: samples -> G
    const int j = warp % NGRP, part = warp / NGRP;
    // this warp's blocks [b0, b0 + nb) of the n_p / 16 full blocks; the last
    // part also takes the tail k-steps [4 nfull, ks)
    const int nfull = p.kfull / 4, bq = nfull / KP, br = nfull - bq * KP;
    const int nb = bq + (part >= KP - br ? 1 : 0);  // the extra blocks go to the last parts
    const int b0 = part * bq + max(0, part - (KP - br));
    const int ntail = part == KP - 1 ? p.ks - p.kfull : 0;
    // FOLD: group j = (|m| tile jp, polar tiles pt0 .. pt0 + NPT - 1); W^T fragments of the cos and the
    // sin columns m = 8 jp + r0 ([jp][cos, sin][ks][32], K = pairs in 16-pair blocks,
    // then the p = 0 step)
    const int jp = j & 1, pt0 = NPT * (j >> 1);  // first polar tile of this warp
    double wc[FOLD ? KB * 4 : 1], wsn[FOLD ? KB * 4 : 1], w0 = 0.0;
    if constexpr (FOLD) {
      const double* wq = p.wreg + ((size_t)(2 * jp) * p.ks + 4 * b0) * 32 + lane;
#pragma unroll
      for (int k = 0; k < KB * 4; ++k) {
        wc[k] = k < 4 * nb ? __ldg(wq + k * 32) : 0.0;
        wsn[k] = k < 4 * nb ? __ldg(wq + (size_t)p.ks * 32 + k * 32) : 0.0;
      }
      if (ntail > 0) w0 = __ldg(p.wreg + ((size_t)(2 * jp) * p.ks + p.kfull) * 32 + lane);
    }
    double wr[FOLD ? 1 : KB * 4], wt[FOLD ? 1 : V2_TAIL];
    if constexpr (!FOLD) {
      const double* ws = p.wreg + ((size_t)j * p.ks + 4 * b0) * 32 + lane;
#pragma unroll
      for (int k = 0; k < KB * 4; ++k) wr[k] = k < 4 * nb ? __ldg(ws + k * 32) : 0.0;
      const double* wq = p.wreg + ((size_t)j * p.ks + p.kfull) * 32 + lane;
#pragma unroll
      for (int k = 0; k < V2_TAIL; ++k) wt[k] = k < ntail ? __ldg(wq + k * 32) : 0.0;
    }
    const bool full_kb = nb == KB;
    // one thread issues: head / tail elements by hand, the rest in one bulk
    // copy; a refilled slot waits for every GEMM warp's release of its
    // previous slab (empty[]); the mbarrier arrive publishes the generic stores
    long long is = 0, icell = cell0;     // next slab to issue: index, cell,
    int ic = 0, iv = 0, ib = 0, ir = 0;  // chunk, v, ring slot, round
    auto issue = [&]() {
      if (is >= total) return;
      long long e0;
      int cnt, m;
      geom(icell, ic, iv, e0, cnt, m);
      if (ir > 0) mbar_wait(&empty[ib], (unsigned)((ir - 1) & 1));
      double* dst = ring + (size_t)ib * p.slot;
      const int nin = (cnt - m) & ~1;
      if (m) dst[1] = __ldg(p.f + e0);
      if ((cnt - m) & 1) dst[m + cnt - 1] = __ldg(p.f + e0 + cnt - 1);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // earlier generic stores to the slot
      mbar_arrive_expect_tx(&full[ib], (unsigned)nin * 8u);
      if (nin > 0) bulk_g2s(dst + 2 * m, p.f + e0 + m, (unsigned)nin * 8u, &full[ib]);
      ++is;
      if (++iv == p.nv) {
        iv = 0;
        if (++ic == p.nchunk) {
          ic = 0;
          icell += cstride;
        }
      }
      if (++ib == p.nbuf) {
        ib = 0;
        ++ir;
      }
    };
    if (tid == 0)
      for (int k = 0; k < p.nbuf - 1; ++k) issue();
    const int col = 8 * j + r0;
    const int ga = (col + 1) >> 1, side = (col & 1) ? 0 : 1;  // col 2a-1: sin (m = -a), col 2a: cos (m = +a)
    long long ccell = cell0;            // this slab's cell,
    int cc = 0, cv = 0, b = 0, b2 = 0;  // chunk, v, ring slot, G buffer
    unsigned fph = 0, gph = 0;          // phase parity of full[b]; of G buffer b2's current round
    for (long long s = 0; s < total; ++s) {
      // slab s + nbuf - 2 into the slot of slab s - 2 (one slab of slack for its release)
      if (tid == 0 && s >= 1) issue();
      mbar_wait(&full[b], fph);
      long long e0;
      int cnt, m;
      geom(ccell, cc, cv, e0, cnt, m);
      // the B gathers are plain (reorderable) loads; this zero, produced after
      // the wait, keeps them from being hoisted above it
      uint32_t after_wait;
      asm volatile("mov.u32 %0, 0;\n" : "=r"(after_wait)::"memory");
      const uint32_t base = smem_u32(ring + (size_t)b * p.slot) + (uint32_t)(m + r0 * p.np) * 8u + after_wait;
      const uint32_t tstep = (uint32_t)(8 * p.np) * 8u;  // one polar tile
      double acc[4][2];
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0.0;
      if constexpr (FOLD) {
        // acc[2 i + cs]: polar tile pt0 + i, cs = 0 cos / 1 sin.  Pair kappa = 16 block + 4 kq + jj
        // is the samples p = kappa + 1 (forward) and n_p - 1 - kappa (mirror).
        uint32_t rowf[NPT], rowm[NPT];
#pragma unroll
        for (int i = 0; i < NPT; ++i) {
          const uint32_t r = base + (uint32_t)(8 * (pt0 + i)) * (uint32_t)p.np * 8u;
          rowf[i] = r + (uint32_t)(1 + 16 * b0 + 4 * kq) * 8u;
          rowm[i] = r + (uint32_t)(p.np - 1 - 16 * b0 - 4 * kq) * 8u;
        }
        auto kstep = [&](double c, double sn, uint32_t off) {
#pragma unroll
          for (int i = 0; i < NPT; ++i) {
            const double a = lds_ro(rowf[i] + off), bm = lds_ro(rowm[i] - off);
            dmma884(acc[2 * i][0], acc[2 * i][1], c, a + bm);
            dmma884(acc[2 * i + 1][0], acc[2 * i + 1][1], sn, a - bm);
          }
        };
#pragma unroll
        for (int blk = 0; blk < KB - 1; ++blk)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) kstep(wc[4 * blk + jj], wsn[4 * blk + jj], (uint32_t)(16 * blk + jj) * 8u);
        if (full_kb) {
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
            kstep(wc[4 * (KB - 1) + jj], wsn[4 * (KB - 1) + jj], (uint32_t)(16 * (KB - 1) + jj) * 8u);
        }
        if (ntail > 0) {  // p = 0: its own mirror image; the weight sits on the kq = 0 lanes
#pragma unroll
          for (int i = 0; i < NPT; ++i)
            dmma884(acc[2 * i][0], acc[2 * i][1], w0,
                    lds_ro(base + (uint32_t)(8 * (pt0 + i)) * (uint32_t)p.np * 8u));
        }
      } else {
      uint32_t rowb[4];  // block b0, lane offset 4 kq, polar tile i: k-step (block, jj) is +(16 block + jj) doubles
#pragma unroll
      for (int i = 0; i < 4; ++i) rowb[i] = base + (uint32_t)(16 * b0 + 4 * kq) * 8u + (uint32_t)i * tstep;
      auto kstep = [&](double w, uint32_t off) {
#pragma unroll
        for (int i = 0; i < 4; ++i) dmma884(acc[i][0], acc[i][1], w, lds_ro(rowb[i] + off));
      };
#pragma unroll
      for (int blk = 0; blk < KB - 1; ++blk)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) kstep(wr[4 * blk + jj], (uint32_t)(16 * blk + jj) * 8u);
      if (full_kb) {
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) kstep(wr[4 * (KB - 1) + jj], (uint32_t)(16 * (KB - 1) + jj) * 8u);
      }
      if (ntail > 0) {  // natural order: sample 16 nfull + 4 u + kq
        const uint32_t tb = (uint32_t)(16 * (nfull - b0) - 3 * kq) * 8u;
#pragma unroll
        for (int u = 0; u < V2_TAIL; ++u)
          if (u < ntail) kstep(wt[u], tb + (uint32_t)(4 * u) * 8u);
      }
      }
      // partials of the K parts, double-buffered by slab parity: a part writes
      // buffer (s & 1) again at slab s + 2, after the pair barrier of s + 1,
      // which part 0 reaches only after reading it at slab s
      double* rbuf = red + (size_t)(s & 1) * NGRP * (KP - 1) * 8 * 32;
      if (part > 0) {
        const uint32_t rw = smem_u32(rbuf + (size_t)(j * (KP - 1) + part - 1) * 8 * 32 + lane);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          sts_v(rw + (uint32_t)(64 * i) * 8u, acc[i][0]);
          sts_v(rw + (uint32_t)(64 * i + 32) * 8u, acc[i][1]);
        }
        bar_sync(V2_BAR_RED0 + j, KP * 32);
      } else {
        if constexpr (KP > 1) bar_sync(V2_BAR_RED0 + j, KP * 32);
        if constexpr (KP > 1) {
          // fixed order: ((p0 + p1) + p2) + p3
#pragma unroll
          for (int q = 0; q < KP - 1; ++q) {
            const uint32_t rq = smem_u32(rbuf + (size_t)(j * (KP - 1) + q) * 8 * 32 + lane);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              acc[i][0] += lds_v(rq + (uint32_t)(64 * i) * 8u);
              acc[i][1] += lds_v(rq + (uint32_t)(64 * i + 32) * 8u);
            }
          }
        }
        if (s >= V2_NGB) mbar_wait(&gempty[b2], gph ^ 1u);  // the epilogue released b2 (previous round)
        if constexpr (FOLD) {
          const int mm = 8 * jp + r0;  // |m| of this lane's cos and sin columns
          if (mm <= p.L) {
            const uint32_t gb = smem_u32(gbuf + (size_t)b2 * gsz + (size_t)mm * V2_GA);
#pragma unroll
            for (int i = 0; i < NPT; ++i)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const uint32_t t2 = (uint32_t)(2 * (8 * (pt0 + i) + 2 * kq + e)) * 8u;
                sts128_v(gb + t2, acc[2 * i + 1][e], acc[2 * i][e]);  // (sin, cos); m = 0: sin weights are 0
              }
          }
        } else if (col < p.ncol) {
          const uint32_t gb = smem_u32(gbuf + (size_t)b2 * gsz + (size_t)ga * V2_GA + side);
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int e = 0; e < 2; ++e) sts_v(gb + (uint32_t)(2 * (8 * i + 2 * kq + e)) * 8u, acc[i][e]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&gfull[b2]);  // release: the stores above are visible to the waiters
      }
      // release ring slot b: after the stores above, which consume every gather
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[b]);
      if (++cv == p.nv) {
        cv = 0;
        if (++cc == p.nchunk) {
          cc = 0;
          ccell += cstride;
        }
      }
      if (++b == p.nbuf) {
        b = 0;
        fph ^= 1u;
      }
      b2 = (b2 + 1) & (V2_NGB - 1);
      if (b2 == 0) gph ^= 1u;
    }
  } else {
    // ------------------------------------------------ consumer: G -> coefficients
    // (l, |m|) row of this lane pair, half.  Rows are |m|-major (all l of one |m|
    // consecutive): the 16 rows of a warp span two or three |m|, so their 16-byte
    // G loads are broadcasts of 2-3 distinct addresses per t (one wavefront
    // instead of four with l-major rows)
    const int et = tid - NT_G, r = et >> 1, hf = et & 1;
    int a = 0;
    while (a < p.L && (a + 1) * (p.L + 1) - (a + 1) * a / 2 <= r) ++a;
    const int l = a + (r - (a * (p.L + 1) - a * (a - 1) / 2));
    const bool live = r < p.npl;
    const int kh = (p.nk + 1) / 2, kb = hf ? kh : 0, ke = hf ? p.nk : kh;  // this lane's radial indices
    double racc[2][V2_KH];
#pragma unroll
    for (int k = 0; k < V2_KH; ++k) racc[0][k] = racc[1][k] = 0.0;
    const uint32_t prow = smem_u32(pt + (size_t)r * V2_TCP + hf);  // this lane's polar rows: t = 2 u + hf
    long long cell = cell0;
    int c = 0, v = 0, b2 = 0;
    unsigned gph = 0;
    for (long long s = 0; s < total; ++s) {
      // new chunk: its polar table (after every epilogue thread finished the old one);
      // with a single chunk the table of the first cell serves every cell
      if (v == 0 && (p.nchunk > 1 || s == 0)) {
        bar_sync(V2_BAR_EPI, NT_E);
        for (int i = et; i < p.npl * TC; i += NT_E) {
          const int row = i / TC;
          pt[row * V2_TCP + (i - row * TC)] = p.ptab[(size_t)c * p.npl * TC + i];
        }
        bar_sync(V2_BAR_EPI, NT_E);  // table complete before any epilogue warp reads it
      }
      // radial factors of this slab's v (global / L1; issued before the wait)
      double rk[V2_KH];
      const double* rv = p.rtab + ((size_t)v * (p.L + 1) + l) * p.nk + kb;
#pragma unroll
      for (int k = 0; k < V2_KH; ++k) rk[k] = (live && kb + k < ke) ? __ldg(rv + k) : 0.0;
      mbar_wait(&gfull[b2], gph);  // G buffer b2 written by every storing warp
      double as = 0.0, ac = 0.0;
      if (live) {
        // the pair interleaves its rows (t = 2 u + hf): the two lanes hit adjacent banks
        const uint32_t g = smem_u32(gbuf + (size_t)b2 * gsz + (size_t)a * V2_GA) + (uint32_t)(2 * hf) * 8u;
        double sa[4] = {0.0, 0.0, 0.0, 0.0}, ca[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int t = 0; t < TC / 2; t += 4) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double2 gv = lds128_v(g + (uint32_t)(4 * (t + u)) * 8u);
            const double pv = lds_v(prow + (uint32_t)(2 * (t + u)) * 8u);
            sa[u] = fma(pv, gv.x, sa[u]);
            ca[u] = fma(pv, gv.y, ca[u]);
          }
        }
        as = (sa[0] + sa[1]) + (sa[2] + sa[3]);
        ac = (ca[0] + ca[1]) + (ca[2] + ca[3]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&gempty[b2]);  // buffer b2 may be rewritten
      // both halves of the row, added in the same order on both lanes
      const double os = __shfl_xor_sync(0xffffffffu, as, 1), oc = __shfl_xor_sync(0xffffffffu, ac, 1);
      const double ts = hf ? os + as : as + os, tcv = hf ? oc + ac : ac + oc;
#pragma unroll
      for (int k = 0; k < V2_KH; ++k) {
        racc[0][k] = fma(rk[k], ts, racc[0][k]);
        racc[1][k] = fma(rk[k], tcv, racc[1][k]);
      }
      b2 = (b2 + 1) & (V2_NGB - 1);
      if (b2 == 0) gph ^= 1u;
      if (++v == p.nv) {
        v = 0;
        if (++c == p.nchunk) {  // the cell is complete: store its coefficients, start the next from zero
          c = 0;
          if (live) {
            double* oc = p.out + cell * (long long)p.nk * p.nq;
            const int qc = l * l + l + a, qs = l * l + l - a;  // cos side: m = +a (m = 0: column 0); sin side: m = -a
#pragma unroll
            for (int k = 0; k < V2_KH; ++k)
              if (kb + k < ke) {
                oc[(size_t)(kb + k) * p.nq + qc] = racc[1][k];
                if (a > 0) oc[(size_t)(kb + k) * p.nq + qs] = racc[0][k];
              }
          }
#pragma unroll
          for (int k = 0; k < V2_KH; ++k) racc[0][k] = racc[1][k] = 0.0;
          cell += cstride;
        }
      }
    }
  }
}

typedef void (*Ps2Kernel)(const Ps2Params);
template <int NTILE>
Ps2Kernel ps2_kernel_kb(int kb) {
  switch (kb) {
    case 1: return k_project_v2<NTILE, 1>;
    case 2: return k_project_v2<NTILE, 2>;
    case 3: return k_project_v2<NTILE, 3>;
    case 4: return k_project_v2<NTILE, 4>;
    default: return nullptr;
  }
}
// KB = ceil(full blocks / K parts); n_p <= 131 gives at most 8 blocks
Ps2Kernel ps2_kernel(int ntile, int kb) {
  switch (ntile) {
    case 1: return ps2_kernel_kb<1>(kb);
    case 2: return ps2_kernel_kb<2>(kb);
    case 3: return ps2_kernel_kb<3>(kb);
    case 4: return ps2_kernel_kb<4>(kb);
    default: return nullptr;
  }
}
// whole: no K split (kb = all blocks, <= 4); else two K parts (kb = blocks of the larger part, <= 3)
Ps2Kernel ps2_fold_kernel(int kb, bool whole) {
  if (whole) {
    switch (kb) {
      case 1: return k_project_v2<4, 1, 2>;
      case 2: return k_project_v2<4, 2, 2>;
      case 3: return k_project_v2<4, 3, 2>;
      case 4: return k_project_v2<4, 4, 2>;
      default: return nullptr;
    }
  }
  switch (kb) {
    case 1: return k_project_v2<4, 1, 1>;
    case 2: return k_project_v2<4, 2, 1>;
    case 3: return k_project_v2<4, 3, 1>;
    default: return nullptr;
  }
}
constexpr int FOLD_MAXKB = 3;
int ps2_kparts(int ntile) { return ntile == 4 ? 2 : 4; }
int ps2_threads(int ntile) {
  switch (ntile) {
    case 1: return V2Shape<1>::THREADS;
    case 2: return V2Shape<2>::THREADS;
    case 3: return V2Shape<3>::THREADS;
    default: return V2Shape<4>::THREADS;
  }
}
int ps2_red_doubles(int ntile) {
  const int kp = ntile == 4 ? 2 : 4;
  return 2 * ntile * (kp - 1) * 8 * 32;
}

typedef void (*PsKernel)(const PsParams);
template <bool R>
PsKernel ps_kernel_r(int ntile) {
  switch (ntile) {
    case 1: return k_project_samples<1, R>;
    case 2: return k_project_samples<2, R>;
    case 3: return k_project_samples<3, R>;
    case 4: return k_project_samples<4, R>;
    case 5: return k_project_samples<5, R>;
    case 6: return k_project_samples<6, R>;
    default: return k_project_samples<7, R>;
  }
}
bool ps_regacc(int nk, int nq) { return nk <= NKMAX_REG && nq <= 2 * (EPI_WARPS * 32); }
PsKernel ps_kernel(int ntile, int nk, int nq) {
  return ps_regacc(nk, nq) ? ps_kernel_r<true>(ntile) : ps_kernel_r<false>(ntile);
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
  cudaDeviceGetAttribute(&pj->sms, cudaDevAttrMultiProcessorCount, device);
  const int npl = (l_max + 1) * (l_max + 2) / 2;
  const int gs = conflict_free_stride_dev(pj->ntile * 8);
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  auto smem_for = [&](int nbuf) {
    const size_t rvp = ((size_t)(l_max + 1) * pj->nk + 1) / 2 * 2;  // radial table of one v, padded
    return (size_t)8 * ((size_t)nbuf * (TC * pj->sp + rvp) + (size_t)pj->ks * pj->ntile * 32 + (size_t)npl * TCP +
                        2 * ((size_t)TC * gs + rvp) + (size_t)pj->nk * pj->nq) +
           (size_t)4 * pj->nq;  // l(q) table
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
  if (cudaFuncSetAttribute(ps_kernel(pj->ntile, pj->nk, pj->nq), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pj->smem) !=
      cudaSuccess) {
    bfq_projector_destroy(pj);
    return fail(BFQ_ECUDA, "cannot set the projection kernel's shared memory");
  }
  // v2 (register W tiles, bulk-copied slabs, per-(l,|m|) epilogue): K = n_p in
  // 16-sample blocks (permuted order) plus a natural-order tail
  pj->kfull = 4 * (n_p / 16);
  pj->ks2 = pj->kfull + (n_p % 16 + 3) / 4;
  pj->slot2 = TC * n_p + 8;  // + the misalignment shift and the K-padding overrun of the last row
  pj->slot2 += pj->slot2 & 1;
  const int kp2 = ps2_kparts(pj->ntile), nfull2 = pj->kfull / 4;
  pj->kb2 = (nfull2 + kp2 - 1) / kp2;
  const bool v2_fits = pj->ntile <= 4 && npl <= V2_EPI_WARPS * 16 && pj->nk <= V2_NKMAX && pj->kb2 >= 1 &&
                       pj->kb2 <= 4 && !std::getenv("BFQ_PROJ_V1");
  if (v2_fits) {
    auto smem2_for = [&](int nbuf) {
      return (size_t)V2_HDR + (size_t)8 * ((size_t)nbuf * pj->slot2 + (size_t)V2_NGB * (l_max + 1) * V2_GA +
                                        (size_t)ps2_red_doubles(pj->ntile) + (size_t)npl * V2_TCP);
    };
    int nb = V2_MAXBUF;
    while (nb > 2 && smem2_for(nb) > (size_t)optin) --nb;
    if (smem2_for(nb) <= (size_t)optin) {
      // polar table with |m|-major rows: row(l, a) = a (L + 1) - a (a - 1) / 2 + l - a
      std::vector<double> pt2((size_t)pj->nchunk * npl * TC, 0.0);
      for (int l = 0; l <= l_max; ++l)
        for (int am = 0; am <= l; ++am) {
          const int row = l * (l + 1) / 2 + am, row2 = am * (l_max + 1) - am * (am - 1) / 2 + l - am;
          for (int t = 0; t < n_t; ++t)
            pt2[((size_t)(t / TC) * npl + row2) * TC + t % TC] = theta_tab[(size_t)row * n_t + t];
        }
      std::vector<double> wr((size_t)pj->ntile * pj->ks2 * 32, 0.0);
      for (int j = 0; j < pj->ntile; ++j)
        for (int k = 0; k < pj->ks2; ++k)
          for (int lane = 0; lane < 32; ++lane) {
            const int kq = lane & 3, col = 8 * j + (lane >> 2);
            const int pp = k < pj->kfull ? 16 * (k >> 2) + (k & 3) + 4 * kq : 4 * k + kq;
            if (pp < n_p && col < pj->ncol) wr[((size_t)j * pj->ks2 + k) * 32 + lane] = phi_tab[(size_t)col * n_p + pp];
          }
      pj->nbuf2 = nb;
      pj->smem2 = smem2_for(nb);
      if (!up(wr, &pj->wreg) || !up(pt2, &pj->ptab2) ||
          cudaFuncSetAttribute(ps2_kernel(pj->ntile, pj->kb2), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pj->smem2) !=
              cudaSuccess) {
        bfq_projector_destroy(pj);
        return fail(BFQ_ECUDA, "cannot set up the v2 projection kernel");
      }
      pj->v2 = true;
    }
  }
  // Mirror-folded kernel: n_p odd, the pairs (p, n_p - p) in whole 16-pair blocks,
  // two |m| tiles (8 <= l_max <= 14: the v2 epilogue holds 128 (l, |m|) rows), and a table that IS even (cos, m = 0
  // columns) / odd (sin columns) under the mirror to within a few ulp -- true of
  // the reference's trapezoid nodes phi_p = 2 pi p / n_p (basis.py:239-247);
  // numpy's cos(m phi_p) and cos(m phi_{n_p - p}) differ by rounding of m phi
  // (70 ulp of the column maximum at l_max = 12, n_p = 129; <= 128 ulp is
  // accepted and the folded weight is their mean, i.e. each weight moves by at
  // most 1.4e-14 of the column maximum, towards the exactly symmetric value).
  // Anything else keeps the unfolded kernel.
  if (pj->v2 && (n_p & 1) && l_max >= 8 && l_max <= 15 && npl <= V2_EPI_WARPS * 16 && !std::getenv("BFQ_PROJ_NOFOLD")) {
    const int H = (n_p - 1) / 2, nfull = H / 16;
    const bool whole = nfull <= 4 && !std::getenv("BFQ_PROJ_FOLD_SPLITK");  // K unsplit: order <= 64
    const int kb3 = whole ? nfull : (nfull + 1) / 2;
    bool ok = H % 16 == 0 && nfull >= (whole ? 1 : 2) && kb3 <= (whole ? 4 : FOLD_MAXKB);
    for (int col = 0; ok && col < pj->ncol; ++col) {
      const double* w = phi_tab + (size_t)col * n_p;
      double mx = 0.0;
      for (int pp = 0; pp < n_p; ++pp) mx = std::max(mx, std::fabs(w[pp]));
      const bool odd = col > 0 && (col & 1);  // col 2m-1: sin
      const double tol = 128.0 * 2.220446049250313e-16 * mx;
      if (odd && std::fabs(w[0]) > tol) ok = false;
      for (int pp = 1; ok && pp <= H; ++pp)
        if (std::fabs(w[pp] - (odd ? -w[n_p - pp] : w[n_p - pp])) > tol) ok = false;
    }
    if (ok) {
      pj->kfull3 = 4 * nfull;
      pj->ks3 = pj->kfull3 + 1;
      pj->kb3 = kb3;
      auto smem3_for = [&](int nbuf) {
        return (size_t)V2_HDR + (size_t)8 * ((size_t)nbuf * pj->slot2 + (size_t)V2_NGB * (l_max + 1) * V2_GA +
                                          (size_t)(whole ? 0 : ps2_red_doubles(4)) + (size_t)npl * V2_TCP);
      };
      int nb = V2_MAXBUF;
      if (const char* e = std::getenv("BFQ_PROJ_NBUF")) nb = std::max(3, std::min(V2_MAXBUF, std::atoi(e)));  // experiments
      while (nb > 2 && smem3_for(nb) > (size_t)optin) --nb;
      std::vector<double> wf3((size_t)2 * 2 * pj->ks3 * 32, 0.0);
      for (int jp = 0; jp < 2; ++jp)
        for (int k = 0; k < pj->ks3; ++k)
          for (int lane = 0; lane < 32; ++lane) {
            const int kq = lane & 3, mm = 8 * jp + (lane >> 2);
            if (mm > l_max) continue;
            const double* wc = phi_tab + (size_t)(2 * mm) * n_p;                    // cos m phi (m = 0: column 0)
            const double* ws = mm > 0 ? phi_tab + (size_t)(2 * mm - 1) * n_p : nullptr;  // sin m phi
            double c = 0.0, sn = 0.0;
            if (k < pj->kfull3) {
              const int pp = 16 * (k >> 2) + 4 * kq + (k & 3) + 1;
              c = 0.5 * (wc[pp] + wc[n_p - pp]);
              if (ws) sn = 0.5 * (ws[pp] - ws[n_p - pp]);
            } else if (kq == 0) {
              c = wc[0];  // p = 0 is its own mirror image; sin(0) = 0
            }
            wf3[((size_t)(2 * jp) * pj->ks3 + k) * 32 + lane] = c;
            wf3[((size_t)(2 * jp + 1) * pj->ks3 + k) * 32 + lane] = sn;
          }
      if (smem3_for(nb) <= (size_t)optin) {
        pj->nbuf3 = nb;
        pj->smem3 = smem3_for(nb);
        if (!up(wf3, &pj->wfold) ||
            cudaFuncSetAttribute(ps2_fold_kernel(kb3, whole), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pj->smem3) !=
                cudaSuccess) {
          bfq_projector_destroy(pj);
          return fail(BFQ_ECUDA, "cannot set up the folded projection kernel");
        }
        pj->fold = true;
        pj->fold_whole = whole;
      }
    }
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
  cudaFree(pj->wreg);
  cudaFree(pj->ptab2);
  cudaFree(pj->wfold);
  delete pj;
  return BFQ_OK;
}

int bfq_project_samples(const bfq_projector* pj, const double* samples, double* out, int64_t n, void* stream) {
  if (!pj || (n > 0 && (!samples || !out))) return fail(BFQ_EINVAL, "null argument");
  if (n < 0) return fail(BFQ_EINVAL, "negative batch");
  if (n == 0) return BFQ_OK;
  if (n > 0x7fffffffLL) return fail(BFQ_EINVAL, "too many cells for one launch");
  DevGuard guard(pj->device);
  if (pj->v2) {
    Ps2Params q;
    q.f = samples;
    q.out = out;
    q.n = n;
    q.nk = pj->nk;
    q.L = pj->L;
    q.nq = pj->nq;
    q.nv = pj->nv;
    q.nt = pj->nt;
    q.np = pj->np;
    q.ncol = pj->ncol;
    q.ks = pj->ks2;
    q.kfull = pj->kfull;
    q.nchunk = pj->nchunk;
    q.npl = (pj->L + 1) * (pj->L + 2) / 2;
    q.nbuf = pj->nbuf2;
    q.slot = pj->slot2;
    q.wreg = pj->wreg;
    q.ptab = pj->ptab2;
    q.rtab = pj->rtab;
    const unsigned grid = (unsigned)std::min<int64_t>(n, std::max(pj->sms, 1));
    if (pj->fold) {
      q.ks = pj->ks3;
      q.kfull = pj->kfull3;
      q.nbuf = pj->nbuf3;
      q.wreg = pj->wfold;
      ps2_fold_kernel(pj->kb3, pj->fold_whole)<<<grid, ps2_threads(4), pj->smem3, (cudaStream_t)stream>>>(q);
    } else {
      ps2_kernel(pj->ntile, pj->kb2)<<<grid, ps2_threads(pj->ntile), pj->smem2, (cudaStream_t)stream>>>(q);
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(BFQ_ECUDA, std::string("projection launch: ") + cudaGetErrorString(e));
    return BFQ_OK;
  }
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
  ps_kernel(pj->ntile, pj->nk, pj->nq)<<<(unsigned)n, PS_THREADS, pj->smem, (cudaStream_t)stream>>>(p);
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

int bfq_projector_kernel(const bfq_projector* pj) {
  if (!pj) return -1;
  return pj->fold ? 3 : (pj->v2 ? 2 : 1);
}

}  // extern "C"
