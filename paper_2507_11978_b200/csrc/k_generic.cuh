// Descriptors of the contraction families (element strides throughout).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ntb {

// C[b] (c_m x c_n) = A[b] (a_m x k) * B[b] (k x b_n); optional epilogue
// C = beta * D + alpha * acc with D (d_m x d_n) (addmm).
struct GemmDesc {
  const void* a; const void* b; void* c; const void* d;
  int64_t batch, k;
  int64_t a_m, a_sb, a_sm, a_sk;
  int64_t b_n, b_sb, b_sk, b_sn;
  int64_t c_m, c_n, c_sb, c_sm, c_sn;
  int64_t d_m, d_n, d_sm, d_sn;
  float alpha, beta;
};

// Stride-1, no-padding cross-correlation, NCHW x KCRS -> NKPQ.
struct ConvDesc {
  const void* x; const void* w; void* y;
  int64_t N, C, H, W, K, R, S, P, Q;
  int64_t xs[4], ws[4], ys[4];
};

// O = softmax(Q K^T * scale) V over (B, H, S, D) tensors.
struct AttnDesc {
  const void* q; const void* k; const void* v; void* o;
  int64_t B, H, Sq, Sk, D;
  int64_t qs[4], ks[4], vs[4], os[4];
  float scale;
};

int gemm_generic(const GemmDesc& g, int dtype, cudaStream_t s);
int conv_generic(const ConvDesc& c, int dtype, cudaStream_t s);
int attn_generic(const AttnDesc& a, int dtype, cudaStream_t s);

}  // namespace ntb
