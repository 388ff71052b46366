// sm_100a tensor-core (tcgen05 + TMEM + TMA) kernels of the contraction
// family.  Each returns NTB_ERR_UNSUPPORTED (without launching) when the
// operands fall outside its layout contract so the dispatcher can take the
// generic CUDA-core path.
#pragma once
#include "k_generic.cuh"

namespace ntb {

int gemm_sm100(const GemmDesc& g, int dtype, cudaStream_t s);
// fp32 operands: 3xTF32 (hi*hi + hi*lo + lo*hi) on kind::tf32, CTA pairs.
int gemm_tf32_sm100(const GemmDesc& g, cudaStream_t s);
// fp32 conv2d: the same kernel as an implicit GEMM over a pixel-major copy.
int conv_tf32_sm100(const ConvDesc& c, cudaStream_t s);
int conv_sm100(const ConvDesc& c, int dtype, cudaStream_t s);
// Query-side rotary tables for sdpa_rope: {rows, cols, row_stride,
// col_stride} in elements.  The kernel rotates Q tiles in shared memory; K
// arrives already rotated (launch_sdpa_rope's pre-pass).
struct RopeTables {
  const void *sin_q, *cos_q;
  int64_t sq[4], cq[4];
};
// Half-split rotary embedding of `rows` contiguous rows of 2*half elements
// (position of row r = (r / pos_div) % S; tables (S, half), row stride half).
int rope_rows_vec(const void* x, const void* sn, const void* cs, void* out, int64_t rows,
                  int64_t S, int64_t pos_div, int half, int dtype, cudaStream_t s);
// dry_run: validate the layout contract (and build the tensor maps) without launching.
int attn_sm100(const AttnDesc& a, int dtype, cudaStream_t s, const RopeTables* rope = nullptr,
               bool dry_run = false);

}  // namespace ntb
