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
};

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
