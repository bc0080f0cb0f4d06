// Kernel instantiation helpers: every bfq_inst_*.cu unit instantiates the
// pair-split Q kernel (bfq_qkernel2.cuh) for one compile-time size, so the
// sizes compile in parallel and a change to one size recompiles one unit.
#pragma once
#include "bfq_device.cuh"

namespace bfq {

#include "bfq_qkernel.cuh"
#include "bfq_qkernel2.cuh"

typedef void (*QKernel)(const KParams);

// Single-warp-per-unit kernel (fallback shapes, see choose_config).
template <bool BILIN, int NK, int QS>
QKernel pick_fixed1(int mt, int cells) {
  constexpr int MT = (NK + 7) / 8;
  if (mt != MT) return nullptr;
  if constexpr (MT == 1) {
    if (cells == 8) return bfq_q_kernel<1, 8, BILIN, NK, QS>;
    if (cells == 4) return bfq_q_kernel<1, 4, BILIN, NK, QS>;
  } else if constexpr (MT == 2) {
    if (cells == 4) return bfq_q_kernel<2, 4, BILIN, NK, QS>;
    if (cells == 2) return bfq_q_kernel<2, 2, BILIN, NK, QS>;
  } else {
    if (cells == 2) return bfq_q_kernel<MT, 2, BILIN, NK, QS>;
    if (cells == 1) return bfq_q_kernel<MT, 1, BILIN, NK, QS>;
  }
  return nullptr;
}

// Compile-time-size instantiations for the BASELINE configurations (all
// gathers then use immediate offsets); NK = 0 is the generic kernel.
template <bool BILIN, int NK, int QS>
QKernel pick_fixed2(int mt, int cells) {
  constexpr int MT = (NK + 7) / 8;
  if (mt != MT) return nullptr;
  if constexpr (MT == 1) {
    if (cells == 8) return bfq_q_kernel2<1, 8, BILIN, NK, QS>;
    if (cells == 4) return bfq_q_kernel2<1, 4, BILIN, NK, QS>;
  } else if constexpr (MT == 2) {
    if constexpr (NK == 9) {
      if (cells == 8) return bfq_q_kernel2<2, 8, BILIN, NK, QS>;  // X1: one DMMA tile per cell
    }
    if (cells == 4) return bfq_q_kernel2<2, 4, BILIN, NK, QS>;
    if (cells == 2) return bfq_q_kernel2<2, 2, BILIN, NK, QS>;
  } else {
    if (cells == 2) return bfq_q_kernel2<MT, 2, BILIN, NK, QS>;
    if constexpr (NK == 17) {
      if (cells == 1) return bfq_q_kernel2<MT, 1, BILIN, NK, QS>;  // SPLITM
    }
  }
  return nullptr;
}

}  // namespace bfq

// One instantiation unit: QKernel pick_<tag>(bilinear, pairsplit, mt, cells).
#define BFQ_DEFINE_PICK(tag, NK, QS)                                                              \
  namespace bfq {                                                                                 \
  QKernel pick_##tag(bool bilin, bool pairsplit, int mt, int cells) {                             \
    if (pairsplit)                                                                                \
      return bilin ? pick_fixed2<true, NK, QS>(mt, cells) : pick_fixed2<false, NK, QS>(mt, cells); \
    return bilin ? pick_fixed1<true, NK, QS>(mt, cells) : pick_fixed1<false, NK, QS>(mt, cells);   \
  }                                                                                               \
  }
