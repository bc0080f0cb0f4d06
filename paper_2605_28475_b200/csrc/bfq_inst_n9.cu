// Q kernel instantiations for n_k = 9 (row stride 84 doubles).
#include "bfq_inst.cuh"
BFQ_DEFINE_PICK(n9, 9, 84)
