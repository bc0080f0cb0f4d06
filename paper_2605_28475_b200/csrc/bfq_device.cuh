// Device-side building blocks of the Q(f,f) kernels, shared by the per-size
// instantiation units (bfq_inst_*.cu) and the launcher (bfq_cuda.cu):
// the launch parameter block, the CTA -> (item, tile) map and the PTX
// wrappers (DMMA, shared loads/stores, mbarrier, bulk copy, table rows).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "bfq_internal.h"

namespace bfq {

struct KParams {
  const double* f2;
  const double* f3;
  double* q;
  long long n_cells;
  long long n_tiles;
  int n_items;     // CTAs (items) per cell tile
  int tile_chunk;  // tiles per item-major chunk of the grid
  const double* R;
  const Row* rows;
  const int* sstart;
  const ChanEntry* chans;
  const Group* groups;
  const int16_t* unit_m1;
  const Item* items;
  int nk, nq, qs, k2s, k2p, k2sd, k2pd;
  int cells, m1t, nw, nstage;
  int conservation;
  int hdr, max_chan, nteams;
  int debug;  // timing experiments only (BFQ_DEBUG): bit0 skip stage 1, bit1 skip stage 2, bit3 phase clocks
  unsigned long long* dbg_clk;  // [8] phase cycle totals when bit3 set
  long long n_rows;  // table rows (incl. padding) -- bounds of the row stream
  int* chk;          // BFQ_CHECKED builds: first violation {code, block, thread, aux, count}
  // fused RK4 stage (bfq_rk4_step, harness.py:93-107): 0 = plain Q(f2, f3) into q
  int rk_stage;
  double rk_a;       // stage factor: dt/2 (stages 1, 2), dt (3), dt/6 (4)
  double* rk_y;      // state y (read; written at stage 4)
  double* rk_arg;    // next stage argument y + a k (stages 1-3)
  double* rk_acc;    // k1 + 2 k2 + 2 k3
  int* rk_flag;      // set when the new state is not finite
};

// Epilogue store of one Q element at flat offset `off` = (cell, k1, q1).  A
// plain evaluation writes Q.  The fused RK4 stages consume the element in place
// with numpy's association and rounding (no FMA contraction), so the fused step
// equals the unfused one bit for bit:
//   stage 1  acc = k1            arg = y + (dt/2) k1
//   stage 2  acc = acc + 2 k2    arg = y + (dt/2) k2
//   stage 3  acc = acc + 2 k3    arg = y + dt k3
//   stage 4  y = y + (dt/6) (acc + k4), flag if not finite   (harness.py:97-107)
// Every element is owned by exactly one lane of one CTA, and the prologues read
// only the previous stage's argument buffer (stage 1: y), so no launch reads an
// element another CTA of the same launch writes.
__device__ __forceinline__ void store_q(const KParams& p, long long off, double v) {
  switch (p.rk_stage) {
    case 0:
      p.q[off] = v;
      return;
    case 1:
      p.rk_acc[off] = v;
      p.rk_arg[off] = __dadd_rn(p.rk_y[off], __dmul_rn(p.rk_a, v));
      return;
    case 2:
    case 3:
      p.rk_acc[off] = __dadd_rn(p.rk_acc[off], __dmul_rn(2.0, v));
      p.rk_arg[off] = __dadd_rn(p.rk_y[off], __dmul_rn(p.rk_a, v));
      return;
    default: {
      const double yn = __dadd_rn(p.rk_y[off], __dmul_rn(p.rk_a, __dadd_rn(p.rk_acc[off], v)));
      p.rk_y[off] = yn;
      if (!isfinite(yn)) atomicExch(p.rk_flag, 1);
    }
  }
}

// ------------------------------------------------------------ checked build
// -DBFQ_CHECKED (libbfq_checked.so, tests/test_gpu_checked.py): every shared
// memory access of the Q kernel is checked against the sub-buffer it belongs
// to (staged cells of this warp, this unit's Phi rows, this team's R slot),
// every table row index against the table, every Q store against the
// output; mbarrier waits time out instead of hanging; the first violation is
// recorded in p.chk (and the access clamped into its buffer, so the kernel
// finishes and the host can read the record).  The race canaries (R-slot and
// Phi poisoning, randomized delays) live in the kernel itself.
enum CheckCode {
  CHK_F2 = 1,      // stage-1 gather of g f2[a, q2] outside this warp's staged cells
  CHK_F3 = 2,      // stage-1 gather of f3[b, q3]
  CHK_PHI_ST = 3,  // Phi store outside this warp's Phi row
  CHK_PHI_LD = 4,  // stage-2 Phi load outside this unit's Phi buffer
  CHK_RING = 5,    // stage-2 R load outside this team's ring slot
  CHK_XCH = 6,     // epilogue exchange outside this unit's buffer
  CHK_ROW = 7,     // table row index outside the table
  CHK_Q = 8,       // Q store outside the output
  CHK_ZERO = 9,    // an invariant slot computed non-zero before the epilogue forced it
  CHK_HANG = 10,   // mbarrier wait timed out (ring never filled)
};

#ifdef BFQ_CHECKED
static __device__ __noinline__ void chk_fail(const KParams& p, int code, long long aux) {
  if (atomicAdd(p.chk + 4, 1) == 0) {
    p.chk[0] = code;
    p.chk[1] = (int)blockIdx.x;
    p.chk[2] = (int)threadIdx.x;
    p.chk[3] = (int)aux;
  }
}
__device__ __forceinline__ uint32_t chk_range(const KParams& p, uint32_t addr, uint32_t lo, uint32_t hi, int code) {
  if (addr < lo || addr + 8u > hi || (addr & 7u)) {
    chk_fail(p, code, (long long)addr);
    return lo;
  }
  return addr;
}
__device__ __forceinline__ long long chk_index(const KParams& p, long long i, long long n, int code) {
  if (i < 0 || i >= n) {
    chk_fail(p, code, i);
    return 0;
  }
  return i;
}
// pseudo-random delay (0..1023 ns) of a warp at a schedule point
__device__ __forceinline__ void chk_jitter(unsigned salt) {
  unsigned h = (blockIdx.x * 0x9E3779B9u) ^ ((threadIdx.x >> 5) * 0x85EBCA6Bu) ^ (salt * 0xC2B2AE35u);
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  __nanosleep(h & 1023u);
}
#define BFQ_CHK(addr, lo, hi, code) chk_range(p, (addr), (lo), (hi), (code))
#define BFQ_CHK_IDX(i, n, code) chk_index(p, (i), (n), (code))
#define BFQ_JITTER(salt) chk_jitter(salt)
constexpr bool kChecked = true;
#else
#define BFQ_CHK(addr, lo, hi, code) (addr)
#define BFQ_CHK_IDX(i, n, code) (i)
#define BFQ_JITTER(salt) ((void)0)
constexpr bool kChecked = false;
#endif

// CTA -> (item, tile).  Tiles are taken in chunks of TILE_CHUNK; inside a
// chunk the CTAs run item-major (heavy items first), so all items of a tile
// are resident within a few waves and the tile's cells are read from HBM
// once (L2 serves the other items), while only the last chunk's tail sees
// the light items last.
constexpr int TILE_CHUNK = 64;  // minimum; BFQ_TILE_CHUNK overrides (experiments)
__device__ __forceinline__ void cta_item_tile(const long long b, const long long n_tiles, const int n_items,
                                              const int chunk, long long& item, long long& tile) {
  const long long full = n_tiles / chunk, per = (long long)chunk * n_items;
  if (b < full * per) {
    const long long ch = b / per, r = b - ch * per;
    item = r / chunk;
    tile = ch * chunk + (r - item * chunk);
  } else {
    const long long rem = n_tiles - full * chunk, r = b - full * per;
    item = r / rem;
    tile = full * chunk + (r - item * rem);
  }
}

// ------------------------------------------------------------ PTX helpers
// Not volatile: the scheduler may move shared loads across DMMAs.
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// Gather from the staged cells: read-only after the staging barrier, so a
// plain (non-volatile) asm the compiler may schedule freely.
__device__ __forceinline__ double lds_ro(uint32_t addr) {
  double v;
  asm("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}

// Loads/stores of buffers rewritten inside the kernel (Phi, R ring): volatile
// so they stay ordered with the warp syncs and mbarrier waits.
__device__ __forceinline__ double lds_v(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr) : "memory");
  return v;
}

__device__ __forceinline__ void named_bar_sync(unsigned id, unsigned count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

__device__ __forceinline__ void sts_v(uint32_t addr, double v) {
  asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(addr), "d"(v) : "memory");
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// try_wait with a suspend-time hint: the waiting warp sleeps in hardware
// until the phase flips (or the hint expires) instead of spinning on issue slots.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Checked builds: a bounded wait (~seconds) that records CHK_HANG instead of
// hanging the GPU when a ring slot is never filled.
__device__ __forceinline__ void mbar_wait_chk(const KParams& p, uint64_t* bar, unsigned parity) {
#ifdef BFQ_CHECKED
  for (long long it = 0;; ++it) {
    uint32_t ok;
    asm volatile(
        "{\n"
        " .reg .pred q;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2, 100000;\n"
        " selp.u32 %0, 1, 0, q;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    if (it > (1LL << 22)) {
      chk_fail(p, CHK_HANG, (long long)parity);
      return;
    }
  }
#else
  (void)p;
  mbar_wait(bar, parity);
#endif
}

// Non-blocking probe of an mbarrier phase.
__device__ __forceinline__ bool mbar_test(uint64_t* bar, unsigned parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      " mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// volatile: the compiler must issue the table-row load where it is written
// (early, as a prefetch), not sink it next to its first use.
__device__ __forceinline__ Row load_row(const Row* rows, int z) {
  int4 v;
  asm volatile("ld.global.nc.v4.s32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(reinterpret_cast<const int4*>(rows) + z));
  Row r;
  r.q2 = v.x;
  r.q3 = v.y;
  r.g = __hiloint2double(v.w, v.z);
  return r;
}

__device__ __forceinline__ Row fetch_row(const Row* rows, int z, int ze) {
  if (z < ze) return load_row(rows, z);
  Row r;
  r.q2 = 0;
  r.q3 = 0;
  r.g = 0.0;
  return r;
}

// Branch-free fetch of row z of a range ending at ze: always loads a valid
// row (clamped into [0, ze-1], row 0 for an empty range) and zeroes g when z
// is past the end, so padding lanes and exhausted streams contribute 0.
__device__ __forceinline__ Row fetch_row_bf(const Row* rows, int z, int ze) {
  Row r = load_row(rows, max(min(z, ze - 1), 0));
  r.g = z < ze ? r.g : 0.0;
  return r;
}

__device__ __forceinline__ Row fetch_row_clamped(const Row* rows, int z, int ze) {
  Row r = load_row(rows, min(z, ze - 1));
  if (z >= ze) r.g = 0.0;  // padding lane of the last k-step: contributes 0
  return r;
}

// ------------------------------------------------------------ the Q kernel

}  // namespace bfq
