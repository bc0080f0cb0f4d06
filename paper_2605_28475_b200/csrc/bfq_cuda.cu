// B200 (sm_100a) kernels and C ABI of the Q(f,f) engine.
//
// Q[k1,q1] = sum_tau sum_{a,b} R[k1,a,b,tau] Phi_{tau,q1}[a,b]
// Phi_{tau,q1}[a,b] = sum_{z in slice(tau,q1)} g_z f2[a,q2_z] f3[b,q3_z]
// (the reference's angular-first order, contraction.py:293-317).
//
// One CTA = one cell tile (cells staged in shared memory) x one l1 group x a
// run of m1-units.  Every compute warp owns 8 output rows "pairs" = (m1, cell)
// and walks all channels tau of its l1 group:
//   stage 1  Phi_pair = A B^T over the slice rows, DMMA.8x8x4 (M=a, N=b, K=rows),
//            operands gathered from the staged f (the CG table read is
//            broadcast across the warp's cells),                   contraction.py:306-308
//   stage 2  out[pair,k1] += Phi[pair,(a,b)] R_tau[k1,(a,b)], DMMA.8x8x4
//            (M=pairs, N=k1, K=n_k^2), R_tau streamed into a shared
//            ring by cp.async.bulk + mbarrier from a producer warp,   contraction.py:309
//   scatter  the accumulator of the pair IS Q[cell][k1][q1]: written once at
//            the end, no atomics, deterministic;                    contraction.py:310-312
//   epilogue exact 0.0 on the five invariant slots                  kinematic.py:594-610
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>
#include <type_traits>

#include "bfq_device.cuh"
#include "bfq_internal.h"

namespace bfq {
typedef void (*QKernel)(const KParams);
// per-size instantiation units (bfq_inst_*.cu)
QKernel pick_n5(bool, bool, int, int);
QKernel pick_n9(bool, bool, int, int);
QKernel pick_n11(bool, bool, int, int);
QKernel pick_n13(bool, bool, int, int);
QKernel pick_n17(bool, bool, int, int);
QKernel pick_generic(bool, bool, int, int);
}  // namespace bfq

using namespace bfq;

#define BFQ_CUDA_TRY(expr)                                                          \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      set_error(std::string(#expr) + ": " + cudaGetErrorString(e_));               \
      return BFQ_ECUDA;                                                             \
    }                                                                               \
  } while (0)

namespace {

struct DevProgram {
  KernelConfig cfg;
  bool bilinear = false;
  ChanEntry* chans = nullptr;
  Group* groups = nullptr;
  int16_t* unit_m1 = nullptr;
  Item* items = nullptr;
  int n_items = 0;
  double exec_macs_per_cell = 0.0;
  QKernel kernel = nullptr;
};

unsigned long long* bfq_dbg_clk_ptr = nullptr;  // BFQ_DEBUG bit 3 only

QKernel pick_kernel(bool bilin, bool ps, int mt, int cells, int nk, int qs) {
  QKernel k = nullptr;
  if (!std::getenv("BFQ_GENERIC")) {
    if (nk == 13 && qs == 172) k = pick_n13(bilin, ps, mt, cells);
    else if (nk == 9 && qs == 84) k = pick_n9(bilin, ps, mt, cells);
    else if (nk == 11 && qs == 124) k = pick_n11(bilin, ps, mt, cells);
    else if (nk == 5 && qs == 28) k = pick_n5(bilin, ps, mt, cells);
    else if (nk == 17 && qs == 292) k = pick_n17(bilin, ps, mt, cells);
    if (k) return k;
  }
  return pick_generic(bilin, ps, mt, cells);
}

// ------------------------------------------------------------ small kernels
// basis.moments (basis.py:346-363): mass c[0,0]; momentum (c[0,3], c[0,1], c[0,2]);
// energy 0.5*(3*mass - sqrt(6)*c[1,0]).
__global__ void moments_kernel(const double* c, double* out, long long n_cells, int nk, int nq, int l_max) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n_cells) return;
  const double* v = c + i * (long long)nk * nq;
  const double mass = v[0];
  const double px = l_max >= 1 ? v[3] : 0.0, py = l_max >= 1 ? v[1] : 0.0, pz = l_max >= 1 ? v[2] : 0.0;
  const double e2 = nk >= 2 ? v[nq] : 0.0;
  double* o = out + i * 5;
  o[0] = mass;
  o[1] = px;
  o[2] = py;
  o[3] = pz;
  // separately rounded, in the reference's order (no FMA contraction): bitwise equal
  o[4] = __dmul_rn(0.5, __dadd_rn(__dmul_rn(3.0, mass), __dmul_rn(-2.449489742783178, e2)));
}

// RK4 stage helpers (harness.py:97-102).  Stage argument y + a*k is formed
// in one pass; the final combination also flags non-finite entries.
__global__ void axpy_kernel(const double* __restrict__ y, const double* __restrict__ k, double a,
                            double* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = __dadd_rn(y[i], __dmul_rn(a, k[i]));  // numpy order: y + (a*k)
}

// y += dt/6 (k1 + 2 k2 + 2 k3 + k4) with k1..k3 accumulated in `acc` as
// acc = k1 + 2k2 + 2k3 (built by rk4_accum) and k4 passed separately.
__global__ void rk4_accum_kernel(double* __restrict__ acc, const double* __restrict__ k, double w, long long n,
                                 int first) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    acc[i] = first ? k[i] : __dadd_rn(acc[i], __dmul_rn(w, k[i]));
}

__global__ void rk4_final_kernel(double* __restrict__ y, const double* __restrict__ acc,
                                 const double* __restrict__ k4, double dt, long long n, int* flag) {
  int bad = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    // same association as y + (dt/6)*(k1 + 2k2 + 2k3 + k4)
    const double v = __dadd_rn(y[i], __dmul_rn(dt / 6.0, __dadd_rn(acc[i], k4[i])));
    y[i] = v;
    bad |= !isfinite(v);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag, 1);
}

}  // namespace

// ------------------------------------------------------------ the plan
struct HostPathScratch {
  std::mutex mu;
  static constexpr int NB = 3;
  cudaStream_t st[NB] = {nullptr, nullptr, nullptr};
  double* buf[NB] = {nullptr, nullptr, nullptr};
  size_t cap = 0;  // doubles per buffer
  double* pin[NB] = {nullptr, nullptr, nullptr};  // pinned staging for pageable host buffers
  size_t pin_cap = 0;
};

struct bfq_plan {
  int device = 0;
  HostPlan hp;
  HostPathScratch* host = nullptr;  // lazily created by bfq_eval_host
  double* R = nullptr;
  Row* rows = nullptr;
  int* sstart = nullptr;
  DevProgram sym, full;
  size_t operator_bytes = 0;
  int* chk = nullptr;  // checked builds: violation record (KParams::chk)
};

namespace {

template <class T>
int upload(const std::vector<T>& v, T** out, size_t& total) {
  if (v.empty()) {
    *out = nullptr;
    return BFQ_OK;
  }
  BFQ_CUDA_TRY(cudaMalloc((void**)out, v.size() * sizeof(T)));
  BFQ_CUDA_TRY(cudaMemcpy(*out, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  total += v.size() * sizeof(T);
  return BFQ_OK;
}

int upload_program(const Program& pg, DevProgram& dp, size_t& total, int smem_optin, int nk, int qs) {
  dp.cfg = pg.cfg;
  dp.bilinear = pg.bilinear;
  dp.n_items = (int)pg.items.size();
  dp.exec_macs_per_cell = pg.exec_macs_per_cell;
  int rc;
  if ((rc = upload(pg.chans, &dp.chans, total))) return rc;
  if ((rc = upload(pg.groups, &dp.groups, total))) return rc;
  if ((rc = upload(pg.unit_m1, &dp.unit_m1, total))) return rc;
  if ((rc = upload(pg.items, &dp.items, total))) return rc;
  QKernel k = pick_kernel(pg.bilinear, pg.cfg.pairsplit != 0, pg.cfg.mt, pg.cfg.cells, nk, qs);
  if (!k) {
    set_error("no kernel instantiation for this tiling");
    return BFQ_EINVAL;
  }
  dp.kernel = k;
  // Kernel attributes are global per instantiation: always allow the device
  // maximum so plans of different sizes sharing a kernel never shrink it.
  BFQ_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin));
  return BFQ_OK;
}

void free_program(DevProgram& dp) {
  cudaFree(dp.chans);
  cudaFree(dp.groups);
  cudaFree(dp.unit_m1);
  dp.unit_m1 = nullptr;
  cudaFree(dp.items);
  dp.chans = nullptr;
  dp.groups = nullptr;
  dp.items = nullptr;
}

struct RkStage {  // fused RK4 stage consumed by the epilogue (KParams::rk_*, store_q)
  int stage = 0;
  double a = 0.0;
  double *y = nullptr, *arg = nullptr, *acc = nullptr;
  int* flag = nullptr;
};

int launch_q(const bfq_plan* plan, const DevProgram& dp, const double* f2, const double* f3, double* q,
             int64_t n_cells, cudaStream_t st, const RkStage& rk = RkStage()) {
  const HostPlan& hp = plan->hp;
  if (n_cells == 0) return BFQ_OK;
  KParams p;
  p.rk_stage = rk.stage;
  p.rk_a = rk.a;
  p.rk_y = rk.y;
  p.rk_arg = rk.arg;
  p.rk_acc = rk.acc;
  p.rk_flag = rk.flag;
  p.f2 = f2;
  p.f3 = f3 ? f3 : f2;
  p.q = q;
  p.n_cells = n_cells;
  p.n_tiles = (n_cells + dp.cfg.cells - 1) / dp.cfg.cells;
  p.n_items = dp.n_items;
  {
    // as many tiles per item-major chunk as keep their cells (f2 and f3)
    // within ~8 MB of L2, so every item of a tile reads its cells and merges
    // its Q columns while the lines are still resident: DRAM traffic of the
    // N=L=12 launch 47.4 -> 35.1 KB per cell (algorithmic 35.2) at equal speed
    // (profiles/r02_traffic_tile_chunk.txt; a 32 MB budget let lines be evicted
    // between the items of a tile); small batches stay fully heavy-first
    static const int forced = std::getenv("BFQ_TILE_CHUNK") ? std::max(1, std::atoi(std::getenv("BFQ_TILE_CHUNK"))) : 0;
    const long long tile_bytes = (long long)dp.cfg.cells * hp.n_k * hp.n_q * 8 * (dp.bilinear ? 2 : 1);
    // one-cell tiles (n_k = 17): chunks of 16 tiles measured 1.1% faster than
    // L2-sized ones (profiles/r02_tile_chunk.txt); other shapes are insensitive
    p.tile_chunk = forced ? forced
                          : dp.cfg.cells == 1 ? 16
                                               : (int)std::max<long long>(TILE_CHUNK, (8LL << 20) / std::max(tile_bytes, 1LL));
  }
  p.R = plan->R;
  p.rows = plan->rows;
  p.n_rows = (long long)hp.rows.size();
  p.chk = plan->chk;
  p.sstart = plan->sstart;
  p.chans = dp.chans;
  p.groups = dp.groups;
  p.unit_m1 = dp.unit_m1;
  p.items = dp.items;
  p.nk = hp.n_k;
  p.nq = hp.n_q;
  p.qs = hp.qs;
  p.k2s = hp.k2s;
  p.k2p = hp.k2p;
  p.k2sd = hp.k2sd;
  p.k2pd = hp.k2pd;
  p.cells = dp.cfg.cells;
  p.m1t = dp.cfg.m1t;
  p.nw = dp.cfg.nw;
  p.nstage = dp.cfg.nstage;
  p.conservation = hp.conservation ? 1 : 0;
  p.hdr = dp.cfg.hdr;
  p.max_chan = dp.cfg.max_chan;
  p.nteams = dp.cfg.nteams;
  {
    static const int dbg = std::getenv("BFQ_DEBUG") ? std::atoi(std::getenv("BFQ_DEBUG")) : 0;
    p.debug = dbg;
    static unsigned long long* clk = nullptr;
    if ((dbg & 8) && !clk) {
      cudaMalloc(&clk, 8 * sizeof(unsigned long long));
      cudaMemset(clk, 0, 8 * sizeof(unsigned long long));
    }
    p.dbg_clk = clk;
    if (dbg & 8) bfq_dbg_clk_ptr = clk;
  }
  const long long blocks = p.n_tiles * (long long)dp.n_items;
  if (blocks > 0x7fffffffLL) {
    set_error("too many cells for one launch");
    return BFQ_EINVAL;
  }
  QKernel k = dp.kernel;
  k<<<(unsigned)blocks, dp.cfg.nw * 32, dp.cfg.smem, st>>>(p);
  BFQ_CUDA_TRY(cudaGetLastError());
  return BFQ_OK;
}

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
};

// The output may not share bytes with an input: CTAs of one cell tile still
// read its cells while other CTAs of the tile already write Q.
bool io_overlap(const bfq_plan* plan, const double* f2, const double* f3, const double* q, int64_t n_cells) {
  if (n_cells <= 0) return false;
  const uintptr_t span = (uintptr_t)n_cells * plan->hp.n_k * plan->hp.n_q * sizeof(double);
  auto hit = [&](const double* in) {
    if (!in) return false;
    const uintptr_t a = (uintptr_t)in, b = (uintptr_t)q;
    return a < b + span && b < a + span;
  };
  if (hit(f2) || hit(f3)) {
    set_error("q must not overlap f2 or f3 (in-place evaluation is not supported)");
    return true;
  }
  return false;
}

int plan_from_desc(const bfq_desc* desc, int device, bfq_plan** out) {
  if (!desc || !out) {
    set_error("null argument");
    return BFQ_EINVAL;
  }
  *out = nullptr;
  int ndev = 0;
  BFQ_CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) {
    set_error("device ordinal out of range");
    return BFQ_EINVAL;
  }
  DeviceGuard guard(device);
  int smem_optin = 0;
  BFQ_CUDA_TRY(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  std::unique_ptr<bfq_plan> plan(new (std::nothrow) bfq_plan());
  if (!plan) {
    set_error("host allocation failed");
    return BFQ_ENOMEM;
  }
  plan->device = device;
  int rc = build_host_plan(*desc, smem_optin, plan->hp);
  if (rc) return rc;
  size_t total = 0;
  if ((rc = upload(plan->hp.rblocks, &plan->R, total)) || (rc = upload(plan->hp.rows, &plan->rows, total)) ||
      (rc = upload(plan->hp.sstart, &plan->sstart, total)) ||
      (rc = upload_program(plan->hp.sym, plan->sym, total, smem_optin, plan->hp.n_k, plan->hp.qs)) ||
      (rc = upload_program(plan->hp.full, plan->full, total, smem_optin, plan->hp.n_k, plan->hp.qs))) {
    bfq_plan_destroy(plan.release());
    return rc;
  }
  plan->operator_bytes = total;
  if (kChecked) {
    BFQ_CUDA_TRY(cudaMalloc(&plan->chk, 8 * sizeof(int)));
    BFQ_CUDA_TRY(cudaMemset(plan->chk, 0, 8 * sizeof(int)));
  }
  // host copies of the bulk data are no longer needed
  std::vector<double>().swap(plan->hp.rblocks);
  *out = plan.release();
  return BFQ_OK;
}

}  // namespace

// ------------------------------------------------------------ C ABI
extern "C" {

int bfq_plan_create(const bfq_desc* desc, int device, bfq_plan** out) { return plan_from_desc(desc, device, out); }

int bfq_plan_create_bfct(const char* path, int device, bfq_plan** out) {
  if (!path || !out) {
    set_error("null argument");
    return BFQ_EINVAL;
  }
  BfctImage img;
  int rc = read_bfct(path, img);
  if (rc) return rc;
  return plan_from_desc(&img.desc, device, out);
}

int bfq_plan_destroy(bfq_plan* plan) {
  if (!plan) return BFQ_OK;
  {
    DeviceGuard guard(plan->device);
    cudaFree(plan->R);
    cudaFree(plan->rows);
    cudaFree(plan->sstart);
    cudaFree(plan->chk);
    free_program(plan->sym);
    free_program(plan->full);
    if (plan->host) {
      for (int b = 0; b < HostPathScratch::NB; ++b) {
        cudaFree(plan->host->buf[b]);
        cudaFreeHost(plan->host->pin[b]);
        if (plan->host->st[b]) cudaStreamDestroy(plan->host->st[b]);
      }
      delete plan->host;
    }
  }
  delete plan;
  return BFQ_OK;
}

int bfq_plan_get_info(const bfq_plan* plan, bfq_plan_info* info) {
  if (!plan || !info) {
    set_error("null argument");
    return BFQ_EINVAL;
  }
  const HostPlan& hp = plan->hp;
  info->n_k = hp.n_k;
  info->n_q = hp.n_q;
  info->n_t = hp.n_t;
  info->n_g = hp.n_g;
  info->n_s = hp.n_s;
  info->folded = hp.folded ? 1 : 0;
  info->cells_per_cta = plan->sym.cfg.cells;
  info->warps_per_cta = plan->sym.cfg.nw;
  info->stages = plan->sym.cfg.nstage;
  info->smem_bytes = plan->sym.cfg.smem;
  info->items_per_tile = plan->sym.n_items;
  info->exec_macs_per_cell = plan->sym.exec_macs_per_cell;
  info->useful_macs_per_cell = plan->hp.useful_macs_per_cell;
  info->operator_bytes = (double)plan->operator_bytes;
  return BFQ_OK;
}

int bfq_plan_work(const bfq_plan* plan, double* flops_per_cell, double* bytes_per_cell) {
  if (!plan) {
    set_error("null plan");
    return BFQ_EINVAL;
  }
  if (flops_per_cell) *flops_per_cell = plan->hp.alg_flops_per_cell;
  if (bytes_per_cell) *bytes_per_cell = plan->hp.alg_bytes_per_cell;
  return BFQ_OK;
}

int bfq_eval(const bfq_plan* plan, const double* f2, const double* f3, double* q, int64_t n_cells, void* stream) {
  if (!plan || n_cells < 0) {
    set_error("invalid plan or cell count");
    return BFQ_EINVAL;
  }
  if (n_cells > 0 && (!f2 || !q)) {
    set_error("null buffer");
    return BFQ_EINVAL;
  }
  if (io_overlap(plan, f2, f3, q, n_cells)) return BFQ_EINVAL;
  DeviceGuard guard(plan->device);
  const bool same = (f3 == nullptr || f3 == f2);
  return launch_q(plan, same ? plan->sym : plan->full, f2, same ? f2 : f3, q, n_cells, (cudaStream_t)stream);
}

int bfq_eval_host(const bfq_plan* plan, const double* f2, const double* f3, double* q, int64_t n_cells) {
  if (!plan || n_cells < 0 || (n_cells > 0 && (!f2 || !q))) {
    set_error("invalid argument");
    return BFQ_EINVAL;
  }
  if (n_cells == 0) return BFQ_OK;
  if (io_overlap(plan, f2, f3, q, n_cells)) return BFQ_EINVAL;
  DeviceGuard guard(plan->device);
  const bool same = (f3 == nullptr || f3 == f2);
  const size_t ndof = (size_t)plan->hp.n_k * plan->hp.n_q;
  // chunked pipeline over NB streams: H2D(i+1), Q(i), D2H(i-1) overlap; the
  // streams and device buffers persist in the plan (serialised by a mutex)
  static const int64_t forced_chunk = std::getenv("BFQ_HOST_CHUNK") ? std::atoll(std::getenv("BFQ_HOST_CHUNK")) : 0;
  // 256-cell chunks: the exposed first H2D / last D2H shrink to one small
  // chunk and the launches of the three streams overlap each other's tails
  // (measured e2e / device: 0.97 -> 1.00 at N=L=12, 0.79 -> 0.96 at N=L=8)
  const int64_t chunk = std::min<int64_t>(n_cells, forced_chunk > 0 ? forced_chunk : 256);
  HostPathScratch*& hs = const_cast<bfq_plan*>(plan)->host;
  static std::mutex create_mu;
  {
    std::lock_guard<std::mutex> lk(create_mu);
    if (!hs) hs = new (std::nothrow) HostPathScratch();
    if (!hs) {
      set_error("host allocation failed");
      return BFQ_ENOMEM;
    }
  }
  std::lock_guard<std::mutex> lk(hs->mu);
  const int NB = HostPathScratch::NB;
  const size_t per = chunk * ndof, need = per * 3;
  if (hs->cap < need) {
    for (int b = 0; b < NB; ++b) {
      cudaFree(hs->buf[b]);
      hs->buf[b] = nullptr;
    }
    hs->cap = 0;
    for (int b = 0; b < NB; ++b)
      if (cudaMalloc(&hs->buf[b], need * sizeof(double)) != cudaSuccess) {
        set_error("device allocation failed");
        return BFQ_ENOMEM;
      }
    hs->cap = need;
  }
  for (int b = 0; b < NB; ++b)
    if (!hs->st[b] && cudaStreamCreateWithFlags(&hs->st[b], cudaStreamNonBlocking) != cudaSuccess) {
      set_error("stream creation failed");
      return BFQ_ECUDA;
    }
  // Pageable host buffers cannot be copied asynchronously: stage them through
  // pinned buffers owned by the plan, so the host memcpy of chunk i+1 (and the
  // copy-out of chunk i-NB) overlaps the device work of the chunks in flight.
  auto pinned = [](const void* p) {
    if (!p) return true;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return at.type == cudaMemoryTypeHost;
  };
  const bool stage_in = !pinned(f2) || (!same && !pinned(f3));
  const bool stage_out = !pinned(q);
  if ((stage_in || stage_out) && hs->pin_cap < need) {
    for (int b = 0; b < NB; ++b) {
      cudaFreeHost(hs->pin[b]);
      hs->pin[b] = nullptr;
    }
    hs->pin_cap = 0;
    for (int b = 0; b < NB; ++b)
      if (cudaMallocHost(&hs->pin[b], need * sizeof(double)) != cudaSuccess) {
        set_error("pinned host allocation failed");
        return BFQ_ENOMEM;
      }
    hs->pin_cap = need;
  }
  int rc = BFQ_OK;
  std::vector<int64_t> pending(NB, -1);  // chunk start whose staged Q is still in pin[b]
  auto drain = [&](int b) {
    if (pending[b] < 0) return;
    if (cudaStreamSynchronize(hs->st[b]) != cudaSuccess) {
      set_error(cudaGetErrorString(cudaGetLastError()));
      rc = BFQ_ECUDA;
    } else {
      const int64_t n = std::min<int64_t>(chunk, n_cells - pending[b]);
      std::memcpy(q + pending[b] * ndof, hs->pin[b] + 2 * per, n * ndof * sizeof(double));
    }
    pending[b] = -1;
  };
  for (int64_t c0 = 0, i = 0; c0 < n_cells && rc == BFQ_OK; c0 += chunk, ++i) {
    const int b = (int)(i % NB);
    cudaStream_t st = hs->st[b];
    const int64_t n = std::min<int64_t>(chunk, n_cells - c0);
    double* d2 = hs->buf[b];
    double* dq = d2 + per;
    double* d3 = same ? d2 : dq + per;
    const size_t bytes = n * ndof * sizeof(double);
    if (stage_out) drain(b);
    else if (stage_in && i >= NB && cudaStreamSynchronize(st) != cudaSuccess) {  // pin[b] still being read
      set_error(cudaGetErrorString(cudaGetLastError()));
      rc = BFQ_ECUDA;
    }
    if (rc) break;
    const double* s2 = f2 + c0 * ndof;
    const double* s3 = same ? s2 : f3 + c0 * ndof;
    if (stage_in) {  // pin[b] = [f2 chunk | f3 chunk | Q chunk]
      std::memcpy(hs->pin[b], s2, bytes);
      if (!same) std::memcpy(hs->pin[b] + per, s3, bytes);
      s2 = hs->pin[b];
      s3 = same ? s2 : hs->pin[b] + per;
    }
    if (cudaMemcpyAsync(d2, s2, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        (!same && cudaMemcpyAsync(d3, s3, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess)) {
      set_error("host-to-device copy failed");
      rc = BFQ_ECUDA;
      break;
    }
    rc = launch_q(plan, same ? plan->sym : plan->full, d2, d3, dq, n, st);
    if (rc) break;
    double* dst = stage_out ? hs->pin[b] + 2 * per : q + c0 * ndof;
    if (cudaMemcpyAsync(dst, dq, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess) {
      set_error("device-to-host copy failed");
      rc = BFQ_ECUDA;
    }
    if (stage_out) pending[b] = c0;
  }
  for (int b = 0; b < NB; ++b) {
    if (stage_out && rc == BFQ_OK) drain(b);
    if (cudaStreamSynchronize(hs->st[b]) != cudaSuccess && rc == BFQ_OK) {
      set_error(cudaGetErrorString(cudaGetLastError()));
      rc = BFQ_ECUDA;
    }
  }
  return rc;
}

int bfq_rk4_step(const bfq_plan* plan, double* y, double* work, int64_t n_cells, double dt, int32_t* flag,
                 void* stream) {
  if (!plan || !y || !work || !flag || n_cells < 0) {
    set_error("invalid argument");
    return BFQ_EINVAL;
  }
  if (n_cells == 0) return BFQ_OK;
  DeviceGuard guard(plan->device);
  cudaStream_t st = (cudaStream_t)stream;
  const long long n = n_cells * (long long)plan->hp.n_k * plan->hp.n_q;
  int rc;
  // Fused (BFQ_RK4_FUSED=1): four Q launches whose epilogues form
  // the next stage argument, the weighted sum k1 + 2k2 + 2k3 and, at stage 4,
  // the new state (store_q in bfq_device.cuh); the prologue of stage s+1 stages
  // the argument buffer stage s wrote (ping-pong A / B, so no launch reads what
  // it writes).  Bit-identical to the unfused sequence, but measured 0.7% slower
  // at config 5 (844k vs 850k Q/s, profiles/r02_rk4_fused_ab.txt): the epilogue's
  // scattered 8-byte read-modify-writes from the 12 CTAs of a tile cost more
  // than the seven streaming elementwise passes they replace, so the unfused
  // sequence stays the default.
  static const bool fused = std::getenv("BFQ_RK4_FUSED") != nullptr && std::atoi(std::getenv("BFQ_RK4_FUSED")) != 0;
  if (fused) {
    double* argA = work;
    double* argB = work + n;
    double* acc = work + 2 * n;
    RkStage s1{1, 0.5 * dt, y, argA, acc, flag}, s2{2, 0.5 * dt, y, argB, acc, flag},
        s3{3, dt, y, argA, acc, flag}, s4{4, dt / 6.0, y, nullptr, acc, flag};
    if ((rc = launch_q(plan, plan->sym, y, y, nullptr, n_cells, st, s1))) return rc;        // k1 = Q(y)
    if ((rc = launch_q(plan, plan->sym, argA, argA, nullptr, n_cells, st, s2))) return rc;  // k2 = Q(y + dt/2 k1)
    if ((rc = launch_q(plan, plan->sym, argB, argB, nullptr, n_cells, st, s3))) return rc;  // k3 = Q(y + dt/2 k2)
    return launch_q(plan, plan->sym, argA, argA, nullptr, n_cells, st, s4);                 // k4 = Q(y + dt k3)
  }
  // Unfused sequence (default): Q launches plus elementwise stage kernels in
  // numpy's association (harness.py:97-102).
  double* k = work;         // current stage derivative
  double* arg = work + n;   // stage argument
  double* acc = work + 2 * n;
  const int tb = 256;
  const int gb = (int)std::min<long long>((n + tb - 1) / tb, 148LL * 16);
  // k1 = Q(y)
  if ((rc = launch_q(plan, plan->sym, y, y, k, n_cells, st))) return rc;
  rk4_accum_kernel<<<gb, tb, 0, st>>>(acc, k, 1.0, n, 1);
  axpy_kernel<<<gb, tb, 0, st>>>(y, k, 0.5 * dt, arg, n);
  // k2 = Q(y + dt/2 k1)
  if ((rc = launch_q(plan, plan->sym, arg, arg, k, n_cells, st))) return rc;
  rk4_accum_kernel<<<gb, tb, 0, st>>>(acc, k, 2.0, n, 0);
  axpy_kernel<<<gb, tb, 0, st>>>(y, k, 0.5 * dt, arg, n);
  // k3 = Q(y + dt/2 k2)
  if ((rc = launch_q(plan, plan->sym, arg, arg, k, n_cells, st))) return rc;
  rk4_accum_kernel<<<gb, tb, 0, st>>>(acc, k, 2.0, n, 0);
  axpy_kernel<<<gb, tb, 0, st>>>(y, k, dt, arg, n);
  // k4 = Q(y + dt k3)
  if ((rc = launch_q(plan, plan->sym, arg, arg, k, n_cells, st))) return rc;
  rk4_final_kernel<<<gb, tb, 0, st>>>(y, acc, k, dt, n, flag);
  BFQ_CUDA_TRY(cudaGetLastError());
  return BFQ_OK;
}

int bfq_moments(const bfq_plan* plan, const double* c, double* out, int64_t n_cells, void* stream) {
  if (!plan || n_cells < 0 || (n_cells > 0 && (!c || !out))) {
    set_error("invalid argument");
    return BFQ_EINVAL;
  }
  if (n_cells == 0) return BFQ_OK;
  DeviceGuard guard(plan->device);
  const int tb = 128;
  moments_kernel<<<(unsigned)((n_cells + tb - 1) / tb), tb, 0, (cudaStream_t)stream>>>(
      c, out, n_cells, plan->hp.n_k, plan->hp.n_q, plan->hp.l_max);
  BFQ_CUDA_TRY(cudaGetLastError());
  return BFQ_OK;
}

int bfq_host_plan_info(const bfq_desc* desc, int smem_limit, bfq_plan_info* info) {
  if (!desc || !info) {
    set_error("null argument");
    return BFQ_EINVAL;
  }
  HostPlan hp;
  int rc = build_host_plan(*desc, smem_limit, hp);
  if (rc) return rc;
  info->n_k = hp.n_k;
  info->n_q = hp.n_q;
  info->n_t = hp.n_t;
  info->n_g = hp.n_g;
  info->n_s = hp.n_s;
  info->folded = hp.folded ? 1 : 0;
  info->cells_per_cta = hp.sym.cfg.cells;
  info->warps_per_cta = hp.sym.cfg.nw;
  info->stages = hp.sym.cfg.nstage;
  info->smem_bytes = hp.sym.cfg.smem;
  info->items_per_tile = (int)hp.sym.items.size();
  info->exec_macs_per_cell = hp.sym.exec_macs_per_cell;
  info->useful_macs_per_cell = hp.useful_macs_per_cell;
  info->operator_bytes = (double)(hp.rblocks.size() * sizeof(double) + hp.rows.size() * sizeof(Row) +
                                  hp.sstart.size() * sizeof(int32_t));
  return BFQ_OK;
}

const char* bfq_strerror(int code) {
  switch (code) {
    case BFQ_OK: return "success";
    case BFQ_EINVAL: return "invalid argument or operator";
    case BFQ_EUNSORTED: return "COO rows must be sorted and grouped by (tau, q1)";
    case BFQ_ECUDA: return "CUDA error";
    case BFQ_ENOMEM: return "out of memory";
    case BFQ_ESMEM: return "no kernel configuration fits in shared memory";
    case BFQ_EIO: return "I/O error";
    case BFQ_EFORMAT: return "unrecognized or incompatible cache layout";
    case BFQ_EINTEGRITY: return "cache payload does not match its checksum or advertised sizes";
    case BFQ_EDIVERGED: return "integration diverged";
    default: return "unknown error";
  }
}

const char* bfq_last_error(void) { return get_error().c_str(); }

// Checked builds only (libbfq_checked.so): copy out and reset the first
// recorded violation {code, block, thread, aux, count}; returns BFQ_EINVAL in
// an unchecked build.  Synchronises the plan's device.
extern "C" int bfq_debug_check_status(const bfq_plan* plan, int* out5);
int bfq_debug_check_status(const bfq_plan* plan, int* out5) {
  if (!plan || !out5 || !plan->chk) return BFQ_EINVAL;
  DeviceGuard guard(plan->device);
  BFQ_CUDA_TRY(cudaDeviceSynchronize());
  BFQ_CUDA_TRY(cudaMemcpy(out5, plan->chk, 5 * sizeof(int), cudaMemcpyDeviceToHost));
  BFQ_CUDA_TRY(cudaMemset(plan->chk, 0, 8 * sizeof(int)));
  return BFQ_OK;
}

// Debug only (BFQ_DEBUG bit 3): copy out and reset the per-phase cycle totals.
extern "C" int bfq_debug_phase_clocks(unsigned long long* out8);
int bfq_debug_phase_clocks(unsigned long long* out8) {
  if (!bfq_dbg_clk_ptr) return BFQ_EINVAL;
  cudaDeviceSynchronize();
  cudaMemcpy(out8, bfq_dbg_clk_ptr, 64, cudaMemcpyDeviceToHost);
  cudaMemset(bfq_dbg_clk_ptr, 0, 64);
  return BFQ_OK;
}

}  // extern "C"
