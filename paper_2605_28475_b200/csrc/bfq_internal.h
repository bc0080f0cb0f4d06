// Internal structures shared by the host-side plan builder (bfq_plan.cpp) and
// the device code (bfq_cuda.cu).  Not part of the ABI.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "bfq.h"

namespace bfq {

#ifdef __CUDACC__
#define BFQ_HD __host__ __device__
#else
#define BFQ_HD
#endif

// Stride rule for fp64 fragment gathers: lanes 0-15 of a DMMA operand load
// touch rows r0 in 0..3 at columns c in 0..3 (row*stride + c).  With
// stride = +-4 (mod 16) doubles those 16 addresses fall in 16 distinct
// 8-byte bank pairs, i.e. one wavefront per 16 lanes.
BFQ_HD constexpr int conflict_free_stride_dev(int n) {
  int s = (n + 3) / 4 * 4;
  while (s % 16 != 4 && s % 16 != 12) s += 4;
  return s;
}

// ---------------------------------------------------------------- K order
// The K axis of stage 2 (an index over the radial pairs (a, b) of Phi) may be
// numbered in any order as long as Phi and the R blocks agree.  It is numbered
// in the order the stage-1 epilogue STORES Phi: DMMA tile (A, B) = (a/8, b/8),
// accumulator half e = b&1, then lane (r0, kq) = (a&7, (b&7)>>1), skipping
// entries outside n_k (and, for self-symmetric channels, entries below the
// diagonal).  The valid lanes of each half-warp store then go to consecutive
// doubles -- conflict-free -- while K stays compact (n_k^2, or n_k(n_k+1)/2).
// phi_k / phid_k are used by the plan (R permutation) and by the kernels.
BFQ_HD constexpr int kq_count(int nk, int b, int e) {  // kq in 0..3 with 8b + 2kq + e < nk
  const int n = (nk - 8 * b - e + 1) / 2;
  return n < 0 ? 0 : (n > 4 ? 4 : n);
}
BFQ_HD constexpr int row_count(int nk, int a) {  // r0 in 0..7 with 8a + r0 < nk
  const int n = nk - 8 * a;
  return n < 0 ? 0 : (n > 8 ? 8 : n);
}
// first kq of row r0 on or above the diagonal of a self-symmetric tile (r0 <= 2kq + e)
BFQ_HD constexpr int kq_min_diag(int r0, int e) {
  const int d = r0 - e;
  return d <= 0 ? 0 : (d + 1) / 2;
}
// entries of the diagonal tile (A, A), half e, in rows before r0
BFQ_HD constexpr int diag_rows_before(int nk, int a, int e, int r0) {
  int s = 0;
  const int n = kq_count(nk, a, e);
  for (int r = 0; r < r0; ++r) {
    const int c = n - kq_min_diag(r, e);
    s += c > 0 ? c : 0;
  }
  return s;
}
// first K index of tile (A, B), half e
BFQ_HD constexpr int phi_base(int nk, int a, int b, int e) {
  const int mt = (nk + 7) / 8;
  int s = 0;
  for (int a2 = 0; a2 < mt; ++a2)
    for (int b2 = 0; b2 < mt; ++b2)
      for (int e2 = 0; e2 < 2; ++e2) {
        if (a2 == a && b2 == b && e2 == e) return s;
        s += row_count(nk, a2) * kq_count(nk, b2, e2);
      }
  return s;
}
BFQ_HD constexpr int phid_base(int nk, int a, int b, int e) {  // a <= b
  const int mt = (nk + 7) / 8;
  int s = 0;
  for (int a2 = 0; a2 < mt; ++a2)
    for (int b2 = a2; b2 < mt; ++b2)
      for (int e2 = 0; e2 < 2; ++e2) {
        if (a2 == a && b2 == b && e2 == e) return s;
        s += a2 < b2 ? row_count(nk, a2) * kq_count(nk, b2, e2) : diag_rows_before(nk, a2, e2, 8);
      }
  return s;
}
// K index of Phi[ia][ib] (ia, ib < nk)
BFQ_HD constexpr int phi_k(int nk, int ia, int ib) {
  return phi_base(nk, ia / 8, ib / 8, ib & 1) + (ia & 7) * kq_count(nk, ib / 8, ib & 1) + ((ib & 7) >> 1);
}
// K index of Phi[ia][ib] of a self-symmetric channel (ia <= ib < nk)
BFQ_HD constexpr int phid_k(int nk, int ia, int ib) {
  const int a = ia / 8, b = ib / 8, e = ib & 1, r0 = ia & 7, kq = (ib & 7) >> 1;
  if (a < b) return phid_base(nk, a, b, e) + r0 * kq_count(nk, b, e) + kq;
  return phid_base(nk, a, a, e) + diag_rows_before(nk, a, e, r0) + kq - kq_min_diag(r0, e);
}

// One COO row as the kernel reads it: 16 bytes, one LDG.128 per row.
struct alignas(16) Row {
  int32_t q2;
  int32_t q3;
  double g;
};

// Channel-program entry: which R block to stream and where its slices start.
struct alignas(16) ChanEntry {
  int32_t tau;         // R block index (0-based channel)
  int32_t slice_base;  // index into the expanded slice-start table; slice of m1 = base + m1
  int32_t weight2;     // 1: contribution doubled (fold, l2 < l3); resolved at plan time into a scaled R copy
  int32_t diag;        // 1: self-symmetric channel (l2 == l3), R block packed as the upper triangle
};

// Output-degree group: all channels sharing l1, i.e. one set of output columns.
struct alignas(16) Group {
  int32_t chan_off;  // first entry in the channel program
  int32_t n_chan;
  int32_t d1;        // 2*l1 + 1
  int32_t l1;
  int32_t unit_off;  // first entry of this group's units in Program::unit_m1 (x m1t)
  int32_t n_units;
  int32_t pad[2];
};

// One CTA's work inside a cell tile: up to MAX_TEAMS "teams" of units, each
// team walking the channel list of one l1 group in lockstep behind its own R
// ring.  Team t owns units [ubase[t], ubase[t] + nunits[t]) of group l1[t];
// the CTA's unit slots are assigned to teams in order.
constexpr int MAX_TEAMS = 4;
struct alignas(16) Item {
  int32_t l1[MAX_TEAMS];
  int32_t ubase[MAX_TEAMS];
  int32_t nunits[MAX_TEAMS];
  int32_t pad[MAX_TEAMS];
};

// Kernel shape chosen at plan time for one program (folded or full).
struct KernelConfig {
  int mt = 0;      // ceil(n_k / 8): 8x8 DMMA tiles per radial axis
  int cg = 0;      // cells per stage-1 register group
  int cells = 0;   // cells per CTA tile
  int m1t = 0;     // output m1 values per warp unit (cells * m1t == 8 DMMA rows)
  int nw = 0;      // compute warps per CTA
  int nstage = 0;  // R-block ring depth (per team; two teams per CTA)
  int nf = 1;      // f arrays staged per cell (2 for bilinear Q(f2,f3))
  int smem = 0;    // dynamic shared memory bytes
  int hdr = 0;     // bytes of the barrier/counter/channel-index header
  int pairsplit = 0;  // 1: two warps per unit (bfq_qkernel2), nw = 2 * units per CTA
  int nteams = 2;     // R rings (l1 groups) per CTA, <= MAX_TEAMS
  int upc = 0;        // units per CTA
  int max_chan = 0;
};

// Host image of one channel program (everything the kernel needs besides f and R).
struct Program {
  bool bilinear = false;
  KernelConfig cfg;
  std::vector<ChanEntry> chans;
  std::vector<Group> groups;  // indexed by l1
  std::vector<int16_t> unit_m1;  // [unit][m1t] output column m1 of each DMMA row group, -1 = none
  std::vector<Item> items;    // heavy first
  double exec_macs_per_cell = 0.0;
};

struct HostPlan {
  int n_k = 0, n_q = 0, l_max = 0, k_max = 0, n_t = 0;
  int64_t n_g = 0, n_s = 0;
  double gamma = 0.0;
  int qs = 0;   // smem row stride of f (doubles)
  int k2p = 0;  // n_k^2 rounded up to 4 (stage-2 K extent)
  int k2s = 0;  // row stride of Phi and R blocks (doubles)
  int k2pd = 0; // packed upper-triangle K of self-symmetric channels, rounded up to 4
  int k2sd = 0; // its row stride
  bool conservation = false, detailed_balance = false;
  bool folded = false;  // slot symmetry verified -> Q(f,f) uses the folded program
  std::vector<int32_t> triplets;  // [n_t*3]
  std::vector<Row> rows;          // [n_g] in table order
  std::vector<int32_t> sstart;    // expanded slice starts: per channel d1 slices (+1 end)
  std::vector<int32_t> chan_sbase;
  std::vector<double> rblocks;    // [n_t][n_k][k2s], rblocks[t][k1][a*n_k+b] = R[k1,a,b,t]
  Program sym;                    // Q(f,f) program (folded when `folded`)
  Program full;                   // Q(f2,f3) program (all channels, weight 1)
  double alg_flops_per_cell = 0.0, alg_bytes_per_cell = 0.0;
  double useful_macs_per_cell = 0.0;  // folded program, no tile / row padding
};

// Thread-local error detail.
void set_error(const std::string& msg);
const std::string& get_error();

// Validate a descriptor and build the host image.  Returns BFQ_OK or a code.
int build_host_plan(const bfq_desc& d, int smem_limit, HostPlan& hp);

// Read a BFCT cache file (cache.py:21-39,66-89) into owned vectors + desc.
struct BfctImage {
  int32_t k_max = 0, l_max = 0;
  double gamma = 0.0;
  uint32_t flags = 0;
  std::vector<int32_t> triplets, q1, q2, q3, tau, slice_tau, slice_q1;
  std::vector<int64_t> slice_starts;
  std::vector<double> g, r;
  bfq_desc desc{};
};
int read_bfct(const char* path, BfctImage& img);

uint32_t crc32_update(uint32_t crc, const unsigned char* data, size_t n);

}  // namespace bfq
