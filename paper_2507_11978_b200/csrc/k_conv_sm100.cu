// placeholder until the tcgen05 implicit-GEMM conv kernel lands
#include "common.cuh"
#include "k_sm100.cuh"
namespace ntb {
int conv_sm100(const ConvDesc&, int, cudaStream_t) { return NTB_ERR_UNSUPPORTED; }
}  // namespace ntb
