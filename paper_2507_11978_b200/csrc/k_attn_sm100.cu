// placeholder until the tcgen05 attention kernel lands
#include "common.cuh"
#include "k_sm100.cuh"
namespace ntb {
int attn_sm100(const AttnDesc&, int, cudaStream_t) { return NTB_ERR_UNSUPPORTED; }
}  // namespace ntb
