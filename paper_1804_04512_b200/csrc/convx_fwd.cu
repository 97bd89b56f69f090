// convx_fwd.cu -- instantiates the exact (reference-order FFMA) conv forward (convx.cuh).
#define B2N_CONVX_INSTANTIATE
#include "convx.cuh"
