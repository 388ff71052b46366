// Argument unpacking and path selection for the contraction families
// (mm / bmm / addmm, conv2d, sdpa).  Fast sm_100a tcgen05 kernels take the
// layouts they support; everything else runs the generic CUDA-core kernels
// (k_generic.cu).  Nothing here ever computes on the host.
#include <stdlib.h>

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
  } else if (A.dtype == NTB_F32) {
    // the reference catalog's own dtype (catalog.py:125-129): 3xTF32 on the
    // tensor cores; NTB_GEMM_F32_FMA=1 forces the CUDA-core kernel (A/B only)
    static const bool fma_only = getenv("NTB_GEMM_F32_FMA") != nullptr;
    if (!fma_only) {
      int rc = gemm_tf32_sm100(g, A.stream);
      if (rc != NTB_ERR_UNSUPPORTED) return rc;
    }
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
  } else if (A.dtype == NTB_F32) {
    static const bool fma_only = getenv("NTB_GEMM_F32_FMA") != nullptr;
    if (!fma_only) {
      int rc = conv_tf32_sm100(c, A.stream);
      if (rc != NTB_ERR_UNSUPPORTED) return rc;
    }
  }
  return conv_generic(c, A.dtype, A.stream);
}

static int fill_attn(const LaunchArgs& A, int qi, int ki, int vi, int oi, AttnDesc& a) {
  for (int i : {qi, ki, vi, oi})
    if (A.ranks[i] != 4) return fail(NTB_ERR_ARG, "sdpa: rank-4 (B, H, S, D) tensors");
  const int64_t* S = A.sizes;
  const int64_t* T = A.strides;
  const int64_t q0 = A.base[qi], k0 = A.base[ki], v0 = A.base[vi], o0 = A.base[oi];
  a.q = A.ptrs[qi];
  a.k = A.ptrs[ki];
  a.v = A.ptrs[vi];
  a.o = A.ptrs[oi];
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
  return NTB_OK;
}

// read per call (tests vary it): NTB_ROPE_WS_MB, default 512
static int64_t rope_ws_cap() {
  const char* e = getenv("NTB_ROPE_WS_MB");
  const long long mb = e ? atoll(e) : 512;
  return (int64_t)(mb > 0 ? mb : 1) << 20;
}

// sdpa(rope(q), rope(k), v): params q, k, v, sin_q, cos_q, sin_k, cos_k, o
// (catalog.spec_sdpa_rope).  Q is rotated inside the attention kernel (in
// shared memory between its TMA load and the first MMA, once per query
// tile); K is rotated once per (b, h) by a vectorised pre-pass into library
// workspace (same layout as k), because in-kernel K rotation is redone by
// every query block that shares the K tile.
int launch_sdpa_rope(const LaunchArgs& A) {
  if (A.n_ptrs != 8) return fail(NTB_ERR_ARG, "sdpa_rope: expects q, k, v, sin_q, cos_q, sin_k, cos_k, o");
  AttnDesc a = {};
  int rc = fill_attn(A, 0, 1, 2, 7, a);
  if (rc) return rc;
  for (int i = 3; i < 7; ++i)
    if (A.ranks[i] != 2) return fail(NTB_ERR_ARG, "sdpa_rope: rotary tables are (S, D/2)");
  if (A.dtype != NTB_F16 && A.dtype != NTB_BF16)
    return fail(NTB_ERR_UNSUPPORTED, "sdpa_rope: fp16 / bf16 only");
  const char* layout_msg =
      "sdpa_rope: the fused path needs D in {64, 128}, q/k/v 16-byte aligned with unit inner "
      "stride, k contiguous as (B, S, H, D) or (B, H, S, D), and contiguous (S, D/2) tables "
      "covering every position; run rope_launch + sdpa_launch for other layouts";
  // K pre-pass
  const int64_t B = a.B, H = a.H, S = a.Sk, D = a.D;
  const int64_t* ks = a.ks;
  int64_t pos_div;
  if (ks[3] == 1 && ks[1] == D && ks[2] == H * D && (B == 1 || ks[0] == S * H * D)) pos_div = H;
  else if (ks[3] == 1 && ks[2] == D && ks[1] == S * D && (B == 1 || ks[0] == H * S * D)) pos_div = 1;
  else return fail(NTB_ERR_UNSUPPORTED, layout_msg);
  const int64_t sb = A.base[5], cb = A.base[6];
  if (A.sizes[sb] < S || A.sizes[cb] < S || A.sizes[sb + 1] != D / 2 || A.sizes[cb + 1] != D / 2 ||
      A.strides[sb] != D / 2 || A.strides[cb] != D / 2 || A.strides[sb + 1] != 1 ||
      A.strides[cb + 1] != 1 || !aligned16(A.ptrs[5]) || !aligned16(A.ptrs[6]) ||
      !aligned16(a.k) || (D != 64 && D != 128))
    return fail(NTB_ERR_UNSUPPORTED, layout_msg);
  // The rotated K lives in workspace one batch chunk at a time (at most
  // rope_ws_cap() bytes, default 512 MB): the pre-pass and the attention
  // alternate per chunk, so the workspace is bounded, not O(B H S D).
  const int64_t per_batch = H * S * D * 2;
  int64_t bc = rope_ws_cap() / per_batch;
  if (bc < 1) bc = 1;
  if (bc > B) bc = B;
  const int64_t n_chunks = (B + bc - 1) / bc;
  bc = (B + n_chunks - 1) / n_chunks;
  void* krot = workspace((size_t)(bc * per_batch), A.stream);
  if (!krot) return fail(NTB_ERR_CUDA, "sdpa_rope: workspace allocation failed");
  RopeTables rt;
  rt.sin_q = A.ptrs[3];
  rt.cos_q = A.ptrs[4];
  for (int d = 0; d < 2; ++d) {
    rt.sq[d] = A.sizes[A.base[3] + d];
    rt.cq[d] = A.sizes[A.base[4] + d];
    rt.sq[2 + d] = A.strides[A.base[3] + d];
    rt.cq[2 + d] = A.strides[A.base[4] + d];
  }
  // the attention kernel validates q / v / o and the query tables without
  // launching; only then run the K pre-pass
  AttnDesc ak = a;
  ak.k = krot;
  rc = attn_sm100(ak, A.dtype, A.stream, &rt, /*dry_run=*/true);
  if (rc == NTB_ERR_UNSUPPORTED) return fail(NTB_ERR_UNSUPPORTED, layout_msg);
  if (rc) return rc;
  for (int64_t b0 = 0; b0 < B; b0 += bc) {
    const int64_t nb = B - b0 < bc ? B - b0 : bc;
    AttnDesc ac = ak;
    ac.B = nb;
    ac.q = static_cast<const uint16_t*>(a.q) + b0 * a.qs[0];
    ac.v = static_cast<const uint16_t*>(a.v) + b0 * a.vs[0];
    ac.o = static_cast<uint16_t*>(a.o) + b0 * a.os[0];
    rc = rope_rows_vec(static_cast<const uint16_t*>(a.k) + b0 * ks[0], A.ptrs[5], A.ptrs[6], krot,
                       nb * H * S, S, pos_div, (int)(D / 2), A.dtype, A.stream);
    if (rc) return rc;
    rc = attn_sm100(ac, A.dtype, A.stream, &rt);
    if (rc) return rc;
  }
  return NTB_OK;
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
