// Q kernel instantiations for n_k = 17 (row stride 292 doubles).
#include "bfq_inst.cuh"
BFQ_DEFINE_PICK(n17, 17, 292)
