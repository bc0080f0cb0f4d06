// Q kernel instantiations for n_k = 13 (row stride 172 doubles).
#include "bfq_inst.cuh"
BFQ_DEFINE_PICK(n13, 13, 172)
