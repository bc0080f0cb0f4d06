// Q kernel instantiations for n_k = 5 (row stride 28 doubles).
#include "bfq_inst.cuh"
BFQ_DEFINE_PICK(n5, 5, 28)
