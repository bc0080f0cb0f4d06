// Q kernel instantiations for n_k = 11 (row stride 124 doubles).
#include "bfq_inst.cuh"
BFQ_DEFINE_PICK(n11, 11, 124)
