// sm_100a tensor-core (tcgen05 + TMEM + TMA) kernels of the contraction
// family.  Each returns NTB_ERR_UNSUPPORTED (without launching) when the
// operands fall outside its layout contract so the dispatcher can take the
// generic CUDA-core path.
#pragma once
#include "k_generic.cuh"

namespace ntb {

int gemm_sm100(const GemmDesc& g, int dtype, cudaStream_t s);
int conv_sm100(const ConvDesc& c, int dtype, cudaStream_t s);
int attn_sm100(const AttnDesc& a, int dtype, cudaStream_t s);

}  // namespace ntb
