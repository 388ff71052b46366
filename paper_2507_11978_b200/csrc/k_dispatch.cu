// Argument unpacking and path selection for the contraction families
// (mm / bmm / addmm, conv2d, sdpa).  Fast sm_100a tcgen05 kernels take the
// layouts they support; everything else runs the generic CUDA-core kernels
// (k_generic.cu).  Nothing here ever computes on the host.
#include "common.cuh"
#include "k_generic.cuh"
#include "k_sm100.cuh"

namespace ntb {

int launch_gemm(const LaunchArgs& A) {
  GemmDesc g = {};
  const bool addmm = A.kernel == NTB_K_ADDMM;
  const bool bmm = A.kernel == NTB_K_BMM;
  const int n_t = addmm ? 4 : 3;
  if (A.n_ptrs != n_t) return fail(NTB_ERR_ARG, "gemm: wrong parameter count");
  const int rank = bmm ? 3 : 2;
  const int ia = addmm ? 1 : 0, ib = addmm ? 2 : 1, ic = addmm ? 3 : 2;
  for (int i = 0; i < n_t; ++i)
    if (A.ranks[i] != (addmm && i == 0 ? 2 : rank)) return fail(NTB_ERR_ARG, "gemm: bad rank");
  const int64_t* S = A.sizes;
  const int64_t* T = A.strides;
  const int64_t a0 = A.base[ia], b0 = A.base[ib], c0 = A.base[ic];
  const int o = bmm ? 1 : 0;  // leading batch dim offset
  g.a = A.ptrs[ia];
  g.b = A.ptrs[ib];
  g.c = A.ptrs[ic];
  g.batch = bmm ? S[c0] : 1;
  g.a_m = S[a0 + o];
  g.a_sm = T[a0 + o];
  g.a_sk = T[a0 + o + 1];
  g.a_sb = bmm ? T[a0] : 0;
  g.b_n = S[b0 + o + 1];
  g.b_sk = T[b0 + o];
  g.b_sn = T[b0 + o + 1];
  g.b_sb = bmm ? T[b0] : 0;
  g.k = S[a0 + o + 1] < S[b0 + o] ? S[a0 + o + 1] : S[b0 + o];  // masks: min(K_a, K_b)
  g.c_m = S[c0 + o];
  g.c_n = S[c0 + o + 1];
  g.c_sm = T[c0 + o];
  g.c_sn = T[c0 + o + 1];
  g.c_sb = bmm ? T[c0] : 0;
  if (bmm && (S[a0] < g.batch || S[b0] < g.batch))
    return fail(NTB_ERR_UNSUPPORTED, "bmm: operand batch smaller than the output batch");
  g.alpha = 1.f;
  g.beta = 0.f;
  if (addmm) {
    if (A.n_scalars != 2) return fail(NTB_ERR_ARG, "addmm: needs beta and alpha");
    const int64_t d0 = A.base[0];
    g.d = A.ptrs[0];
    g.d_m = S[d0];
    g.d_n = S[d0 + 1];
    g.d_sm = T[d0];
    g.d_sn = T[d0 + 1];
    g.beta = (float)A.scalars[0];
    g.alpha = (float)A.scalars[1];
  }
  if (A.dtype == NTB_F16 || A.dtype == NTB_BF16) {
    int rc = gemm_sm100(g, A.dtype, A.stream);
    if (rc != NTB_ERR_UNSUPPORTED) return rc;
  }
  return gemm_generic(g, A.dtype, A.stream);
}

int launch_conv2d(const LaunchArgs& A) {
  if (A.n_ptrs != 3 || A.ranks[0] != 4 || A.ranks[1] != 4 || A.ranks[2] != 4)
    return fail(NTB_ERR_ARG, "conv2d: expects input(4), filter(4), output(4)");
  ConvDesc c = {};
  const int64_t* S = A.sizes;
  const int64_t* T = A.strides;
  const int64_t x0 = A.base[0], w0 = A.base[1], y0 = A.base[2];
  c.x = A.ptrs[0];
  c.w = A.ptrs[1];
  c.y = A.ptrs[2];
  c.N = S[x0];
  c.C = S[x0 + 1];
  c.H = S[x0 + 2];
  c.W = S[x0 + 3];
  c.K = S[w0];
  c.R = S[w0 + 2];
  c.S = S[w0 + 3];
  c.P = c.H - c.R + 1;
  c.Q = c.W - c.S + 1;
  for (int d = 0; d < 4; ++d) {
    c.xs[d] = T[x0 + d];
    c.ws[d] = T[w0 + d];
    c.ys[d] = T[y0 + d];
  }
  if (c.P < 1 || c.Q < 1) return fail(NTB_ERR_ARG, "conv2d: filter larger than image");
  if (S[w0 + 1] < c.C)
    return fail(NTB_ERR_UNSUPPORTED, "conv2d: filter has fewer channels than the image");
  if (S[y0] != c.N || S[y0 + 1] != c.K || S[y0 + 2] != c.P || S[y0 + 3] != c.Q)
    return fail(NTB_ERR_UNSUPPORTED, "conv2d: output extent differs from (N, K, H-R+1, W-S+1)");
  if (A.dtype == NTB_F16 || A.dtype == NTB_BF16) {
    int rc = conv_sm100(c, A.dtype, A.stream);
    if (rc != NTB_ERR_UNSUPPORTED) return rc;
  }
  return conv_generic(c, A.dtype, A.stream);
}

int launch_sdpa(const LaunchArgs& A) {
  if (A.n_ptrs != 4) return fail(NTB_ERR_ARG, "sdpa: expects q, k, v, o");
  for (int i = 0; i < 4; ++i)
    if (A.ranks[i] != 4) return fail(NTB_ERR_ARG, "sdpa: rank-4 (B, H, S, D) tensors");
  AttnDesc a = {};
  const int64_t* S = A.sizes;
  const int64_t* T = A.strides;
  const int64_t q0 = A.base[0], k0 = A.base[1], v0 = A.base[2], o0 = A.base[3];
  a.q = A.ptrs[0];
  a.k = A.ptrs[1];
  a.v = A.ptrs[2];
  a.o = A.ptrs[3];
  a.B = S[q0];
  a.H = S[q0 + 1];
  a.Sq = S[q0 + 2];
  a.D = S[q0 + 3];
  a.Sk = S[k0 + 2];
  for (int d = 0; d < 4; ++d) {
    a.qs[d] = T[q0 + d];
    a.ks[d] = T[k0 + d];
    a.vs[d] = T[v0 + d];
    a.os[d] = T[o0 + d];
  }
  if (S[v0 + 2] != a.Sk || S[k0 + 3] != a.D || S[v0 + 3] != a.D || S[o0 + 2] != a.Sq ||
      S[o0 + 3] != a.D)
    return fail(NTB_ERR_UNSUPPORTED, "sdpa: inconsistent K/V/O extents");
  a.scale = 1.0f / sqrtf((float)a.D);
  if (A.dtype == NTB_F16 || A.dtype == NTB_BF16) {
    int rc = attn_sm100(a, A.dtype, A.stream);
    if (rc != NTB_ERR_UNSUPPORTED) return rc;
  }
  return attn_generic(a, A.dtype, A.stream);
}

}  // namespace ntb
