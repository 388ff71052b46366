// placeholder: tcgen05 GEMM lands in the next commit
#include "common.cuh"
#include "k_sm100.cuh"
namespace ntb {
int gemm_sm100(const GemmDesc&, int, cudaStream_t) { return NTB_ERR_UNSUPPORTED; }
int conv_sm100(const ConvDesc&, int, cudaStream_t) { return NTB_ERR_UNSUPPORTED; }
int attn_sm100(const AttnDesc&, int, cudaStream_t) { return NTB_ERR_UNSUPPORTED; }
}  // namespace ntb
