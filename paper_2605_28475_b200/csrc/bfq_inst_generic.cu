// Generic Q kernel instantiations (n_k and the row stride at run time).
#include "bfq_inst.cuh"

namespace bfq {
QKernel pick_generic(bool bilin, bool pairsplit, int mt, int cells) {
  auto pick1 = [&](auto b) -> QKernel {  // single-warp-per-unit fallback
    constexpr bool B = decltype(b)::value;
    if (mt == 1) {
      if (cells == 8) return bfq_q_kernel<1, 8, B, 0, 0>;
      if (cells == 4) return bfq_q_kernel<1, 4, B, 0, 0>;
      if (cells == 2) return bfq_q_kernel<1, 2, B, 0, 0>;
      if (cells == 1) return bfq_q_kernel<1, 1, B, 0, 0>;
    }
    if (mt == 2) {
      if (cells == 4) return bfq_q_kernel<2, 4, B, 0, 0>;
      if (cells == 2) return bfq_q_kernel<2, 2, B, 0, 0>;
      if (cells == 1) return bfq_q_kernel<2, 1, B, 0, 0>;
    }
    if (mt == 3) {
      if (cells == 2) return bfq_q_kernel<3, 2, B, 0, 0>;
      if (cells == 1) return bfq_q_kernel<3, 1, B, 0, 0>;
    }
    return nullptr;
  };
  if (!pairsplit) return bilin ? pick1(std::true_type{}) : pick1(std::false_type{});
  auto pick = [&](auto b) -> QKernel {
    constexpr bool B = decltype(b)::value;
    if (mt == 1) {
      if (cells == 8) return bfq_q_kernel2<1, 8, B, 0, 0>;
      if (cells == 4) return bfq_q_kernel2<1, 4, B, 0, 0>;
      if (cells == 2) return bfq_q_kernel2<1, 2, B, 0, 0>;
    }
    if (mt == 2) {
      if (cells == 4) return bfq_q_kernel2<2, 4, B, 0, 0>;
      if (cells == 2) return bfq_q_kernel2<2, 2, B, 0, 0>;
    }
    if (mt == 3 && cells == 2) return bfq_q_kernel2<3, 2, B, 0, 0>;
    return nullptr;
  };
  return bilin ? pick(std::true_type{}) : pick(std::false_type{});
}
}  // namespace bfq
