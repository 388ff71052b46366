// Generic (any-stride, any-dtype) CUDA-core paths of the contraction family:
// mm / bmm / addmm, implicit-GEMM conv2d and attention.  These are the GPU
// path for fp32 operands (the reference computes in f32) and for
// layouts the tcgen05/TMA kernels do not take (non-unit inner strides,
// misaligned bases); there is no CPU fallback anywhere in the library.
//
// Semantics follow the reference maps exactly (mm.py.golden:34-45):
//   acc[m, n] = sum_{k < K_eff} A[m, k] * B[k, n],  K_eff = min(K_a, K_b)
// with A rows masked to A's own M, B columns to B's own N (fill 0) and the
// store masked to the output extent; addmm adds beta*input + alpha*acc with
// the addend masked to its own extent (addmm.py.golden:44-54).
#include "common.cuh"
#include "k_generic.cuh"

namespace ntb {

constexpr int GT = 64;   // tile edge
constexpr int GK = 16;   // k step

template <typename T>
__global__ void __launch_bounds__(256) gemm_generic_kernel(GemmDesc g) {
  __shared__ float As[GK][GT + 1];
  __shared__ float Bs[GK][GT + 1];
  const int64_t b = blockIdx.z;
  const int64_t m0 = (int64_t)blockIdx.y * GT, n0 = (int64_t)blockIdx.x * GT;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const T* A = (const T*)g.a + b * g.a_sb;
  const T* B = (const T*)g.b + b * g.b_sb;
  float acc[4][4] = {};
  for (int64_t k0 = 0; k0 < g.k; k0 += GK) {
    for (int i = threadIdx.x; i < GK * GT; i += blockDim.x) {
      int kk = i % GK, mm = i / GK;
      int64_t m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < g.a_m && k < g.k) ? Elem<T>::to_f(A[m * g.a_sm + k * g.a_sk]) : 0.f;
      int nn = i % GT, kb = i / GT;
      int64_t n = n0 + nn, k2 = k0 + kb;
      Bs[kb][nn] = (n < g.b_n && k2 < g.k) ? Elem<T>::to_f(B[k2 * g.b_sk + n * g.b_sn]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  T* C = (T*)g.c + b * g.c_sb;
  const T* D = (const T*)g.d;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t m = m0 + ty * 4 + i;
    if (m >= g.c_m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t n = n0 + tx * 4 + j;
      if (n >= g.c_n) continue;
      float v = acc[i][j];
      if (D) {
        float addend = (m < g.d_m && n < g.d_n) ? Elem<T>::to_f(D[m * g.d_sm + n * g.d_sn]) : 0.f;
        v = g.beta * addend + g.alpha * v;
      }
      C[m * g.c_sm + n * g.c_sn] = Elem<T>::from_f(v);
    }
  }
}

template <typename T>
static int gemm_generic_t(const GemmDesc& g, cudaStream_t s) {
  dim3 grid((unsigned)cdiv64(g.c_n, GT), (unsigned)cdiv64(g.c_m, GT), (unsigned)g.batch);
  gemm_generic_kernel<T><<<grid, 256, 0, s>>>(g);
  return check_launch("gemm generic", NTB_PATH_GEMM_GENERIC);
}

int gemm_generic(const GemmDesc& g, int dtype, cudaStream_t s) {
  if (g.batch == 0 || g.c_m == 0 || g.c_n == 0) return NTB_OK;
  switch (dtype) {
    case NTB_F32: return gemm_generic_t<float>(g, s);
    case NTB_F16: return gemm_generic_t<__half>(g, s);
    case NTB_BF16: return gemm_generic_t<__nv_bfloat16>(g, s);
  }
  return fail(NTB_ERR_UNSUPPORTED, "gemm: unsupported dtype");
}

// ---- conv2d: direct implicit GEMM over NCHW with arbitrary strides ------
template <typename T>
__global__ void __launch_bounds__(256) conv_generic_kernel(ConvDesc c) {
  __shared__ float As[GK][GT + 1];
  __shared__ float Bs[GK][GT + 1];
  const int64_t m0 = (int64_t)blockIdx.y * GT, n0 = (int64_t)blockIdx.x * GT;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const T* X = (const T*)c.x;
  const T* W = (const T*)c.w;
  const int64_t PQ = c.P * c.Q, RS = c.R * c.S, M = c.N * PQ, KK = c.C * RS;
  float acc[4][4] = {};
  for (int64_t k0 = 0; k0 < KK; k0 += GK) {
    for (int i = threadIdx.x; i < GK * GT; i += blockDim.x) {
      int kk = i % GK, mm = i / GK;
      int64_t m = m0 + mm, k = k0 + kk;
      float v = 0.f;
      if (m < M && k < KK) {
        int64_t n = m / PQ, p = (m / c.Q) % c.P, q = m % c.Q;
        int64_t ch = k / RS, r = (k / c.S) % c.R, s = k % c.S;
        v = Elem<T>::to_f(X[n * c.xs[0] + ch * c.xs[1] + (p + r) * c.xs[2] + (q + s) * c.xs[3]]);
      }
      As[kk][mm] = v;
      int nn = i % GT, kb = i / GT;
      int64_t ko = n0 + nn, k2 = k0 + kb;
      float u = 0.f;
      if (ko < c.K && k2 < KK) {
        int64_t ch = k2 / RS, r = (k2 / c.S) % c.R, s = k2 % c.S;
        u = Elem<T>::to_f(W[ko * c.ws[0] + ch * c.ws[1] + r * c.ws[2] + s * c.ws[3]]);
      }
      Bs[kb][nn] = u;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  T* Y = (T*)c.y;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t m = m0 + ty * 4 + i;
    if (m >= M) continue;
    int64_t n = m / PQ, p = (m / c.Q) % c.P, q = m % c.Q;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t ko = n0 + tx * 4 + j;
      if (ko >= c.K) continue;
      Y[n * c.ys[0] + ko * c.ys[1] + p * c.ys[2] + q * c.ys[3]] = Elem<T>::from_f(acc[i][j]);
    }
  }
}

int conv_generic(const ConvDesc& c, int dtype, cudaStream_t s) {
  const int64_t M = c.N * c.P * c.Q;
  if (M == 0 || c.K == 0) return NTB_OK;
  dim3 grid((unsigned)cdiv64(c.K, GT), (unsigned)cdiv64(M, GT), 1);
  switch (dtype) {
    case NTB_F32: conv_generic_kernel<float><<<grid, 256, 0, s>>>(c); break;
    case NTB_F16: conv_generic_kernel<__half><<<grid, 256, 0, s>>>(c); break;
    case NTB_BF16: conv_generic_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(c); break;
    default: return fail(NTB_ERR_UNSUPPORTED, "conv2d: unsupported dtype");
  }
  return check_launch("conv2d generic", NTB_PATH_CONV_GENERIC);
}

// ---- attention: one warp per query row, online softmax in fp32 ----------
template <typename T, int DPL>
__global__ void __launch_bounds__(128) attn_generic_kernel(AttnDesc a) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int64_t total = a.B * a.H * a.Sq;
  if (row >= total) return;
  const int64_t i = row % a.Sq, h = (row / a.Sq) % a.H, b = row / (a.Sq * a.H);
  const T* Q = (const T*)a.q + b * a.qs[0] + h * a.qs[1] + i * a.qs[2];
  const T* K = (const T*)a.k + b * a.ks[0] + h * a.ks[1];
  const T* V = (const T*)a.v + b * a.vs[0] + h * a.vs[1];
  float q[DPL], acc[DPL];
#pragma unroll
  for (int t = 0; t < DPL; ++t) {
    int d = lane + 32 * t;
    q[t] = d < a.D ? Elem<T>::to_f(Q[d * a.qs[3]]) * a.scale : 0.f;
    acc[t] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  for (int64_t j = 0; j < a.Sk; ++j) {
    float s = 0.f;
#pragma unroll
    for (int t = 0; t < DPL; ++t) {
      int d = lane + 32 * t;
      if (d < a.D) s = fmaf(q[t], Elem<T>::to_f(K[j * a.ks[2] + d * a.ks[3]]), s);
    }
    s = warp_sum(s);
    float mn = fmaxf(m, s);
    float corr = expf(m - mn), p = expf(s - mn);
    l = l * corr + p;
#pragma unroll
    for (int t = 0; t < DPL; ++t) {
      int d = lane + 32 * t;
      float vv = d < a.D ? Elem<T>::to_f(V[j * a.vs[2] + d * a.vs[3]]) : 0.f;
      acc[t] = acc[t] * corr + p * vv;
    }
    m = mn;
  }
  T* O = (T*)a.o + b * a.os[0] + h * a.os[1] + i * a.os[2];
#pragma unroll
  for (int t = 0; t < DPL; ++t) {
    int d = lane + 32 * t;
    if (d < a.D) O[d * a.os[3]] = Elem<T>::from_f(acc[t] / l);
  }
}

template <typename T>
static int attn_generic_t(const AttnDesc& a, cudaStream_t s) {
  const int64_t rows = a.B * a.H * a.Sq;
  const unsigned blocks = (unsigned)cdiv64(rows, 4);
  if (a.D <= 32) attn_generic_kernel<T, 1><<<blocks, 128, 0, s>>>(a);
  else if (a.D <= 64) attn_generic_kernel<T, 2><<<blocks, 128, 0, s>>>(a);
  else if (a.D <= 128) attn_generic_kernel<T, 4><<<blocks, 128, 0, s>>>(a);
  else if (a.D <= 256) attn_generic_kernel<T, 8><<<blocks, 128, 0, s>>>(a);
  else return fail(NTB_ERR_UNSUPPORTED, "sdpa: head dim > 256");
  return check_launch("sdpa generic", NTB_PATH_ATTN_GENERIC);
}

int attn_generic(const AttnDesc& a, int dtype, cudaStream_t s) {
  if (a.B * a.H * a.Sq == 0) return NTB_OK;
  switch (dtype) {
    case NTB_F32: return attn_generic_t<float>(a, s);
    case NTB_F16: return attn_generic_t<__half>(a, s);
    case NTB_BF16: return attn_generic_t<__nv_bfloat16>(a, s);
  }
  return fail(NTB_ERR_UNSUPPORTED, "sdpa: unsupported dtype");
}

}  // namespace ntb
