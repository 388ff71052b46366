// softmax / rms_norm: the row-tiled reduction family
// (reference catalog.py:155-223; softmax.py.golden, rms_norm.py.golden).
//
// softmax: program (r, j) loads columns [j*CP, j*CP + CP) of row r with -inf
// fill (catalog.py:170), m = max, e = exp(x - m), s = sum(e), out = e / s
// (store masked to the output width).  CP < C therefore yields a per-chunk
// softmax, exactly like the reference.
// rms_norm: program r loads the whole row (launch check cdiv(C, CP) == 1),
// out = x / sqrt(sum(x^2) / C + 1e-6) * w with C the TRUE width
// (catalog.py:209) and eps = 1e-6 (catalog.py:38).
//
// Fast path: one warp per row, the row held in registers as 128-bit packs
// (VPL packs per lane), warp-shuffle reductions, fp32 math, one HBM read and
// one HBM write per element.  HBM roofline: 2 x R x C x sizeof(T) (+ C for
// the rms_norm weight, L2-resident across rows).
// Generic path: one CTA per (row, chunk) over arbitrary element strides.
#include <math.h>

#include "common.cuh"

namespace ntb {

constexpr float kRmsEps = 1e-6f;

template <typename T, int VPL, bool kSoftmax>
__global__ void __launch_bounds__(256) row_vec_kernel(const T* __restrict__ in, int64_t in_rs,
                                                      const T* __restrict__ w,
                                                      T* __restrict__ out, int64_t out_rs,
                                                      int64_t rows, int cols) {
  using P = Pack<T>;
  const int lane = threadIdx.x & 31;
  const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int n_vec = cols / P::N;
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows;
       r += warps_total) {
    const T* src = in + r * in_rs;
    P v[VPL];
#pragma unroll
    for (int u = 0; u < VPL; ++u) {
      int c = lane + u * 32;
      if (c < n_vec) v[u].raw = ld_stream(src + (int64_t)c * P::N);
    }
    float red = kSoftmax ? -INFINITY : 0.f;
#pragma unroll
    for (int u = 0; u < VPL; ++u) {
      int c = lane + u * 32;
      if (c < n_vec) {
        float f[P::N];
        v[u].to_float(f);
#pragma unroll
        for (int k = 0; k < P::N; ++k) red = kSoftmax ? fmaxf(red, f[k]) : fmaf(f[k], f[k], red);
      }
    }
    float scale;
    if (kSoftmax) {
      const float m = warp_max(red);
      float s = 0.f;
#pragma unroll
      for (int u = 0; u < VPL; ++u) {
        int c = lane + u * 32;
        if (c < n_vec) {
          float f[P::N];
          v[u].to_float(f);
#pragma unroll
          for (int k = 0; k < P::N; ++k) s += expf(f[k] - m);
        }
      }
      s = warp_sum(s);
      scale = 1.0f / s;
      T* dst = out + r * out_rs;
#pragma unroll
      for (int u = 0; u < VPL; ++u) {
        int c = lane + u * 32;
        if (c < n_vec) {
          float f[P::N];
          v[u].to_float(f);
#pragma unroll
          for (int k = 0; k < P::N; ++k) f[k] = expf(f[k] - m) * scale;
          P o;
          o.from_float(f);
          st_stream(dst + (int64_t)c * P::N, o.raw);
        }
      }
    } else {
      const float ss = warp_sum(red);
      scale = 1.0f / sqrtf(ss / (float)cols + kRmsEps);
      T* dst = out + r * out_rs;
#pragma unroll
      for (int u = 0; u < VPL; ++u) {
        int c = lane + u * 32;
        if (c < n_vec) {
          float f[P::N], g[P::N];
          v[u].to_float(f);
          P wp;
          wp.raw = ld_keep(w + (int64_t)c * P::N);
          wp.to_float(g);
#pragma unroll
          for (int k = 0; k < P::N; ++k) f[k] = f[k] * scale * g[k];
          P o;
          o.from_float(f);
          st_stream(dst + (int64_t)c * P::N, o.raw);
        }
      }
    }
  }
}

// ---- generic strided path -------------------------------------------------
__device__ __forceinline__ float block_reduce(float v, bool is_max, float* sh) {
  v = is_max ? warp_max(v) : warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  float r = is_max ? -INFINITY : 0.f;
  for (int i = 0; i < nw; ++i) r = is_max ? fmaxf(r, sh[i]) : r + sh[i];
  return r;
}

template <typename T>
__global__ void softmax_generic_kernel(const T* in, int64_t in_r, int64_t in_c, int64_t in_rs,
                                       int64_t in_cs, T* out, int64_t out_c, int64_t out_rs,
                                       int64_t out_cs, int64_t cp, int64_t chunks) {
  __shared__ float sh[32];
  const int64_t r = blockIdx.x / chunks, j = blockIdx.x % chunks;
  const int64_t c0 = j * cp;
  float m = -INFINITY;
  for (int64_t t = threadIdx.x; t < cp; t += blockDim.x) {
    int64_t c = c0 + t;
    if (c < in_c) m = fmaxf(m, Elem<T>::to_f(in[r * in_rs + c * in_cs]));
  }
  m = block_reduce(m, true, sh);
  float s = 0.f;
  for (int64_t t = threadIdx.x; t < cp; t += blockDim.x) {
    int64_t c = c0 + t;
    float x = c < in_c ? Elem<T>::to_f(in[r * in_rs + c * in_cs]) : -INFINITY;
    s += expf(x - m);
  }
  s = block_reduce(s, false, sh);
  for (int64_t t = threadIdx.x; t < cp; t += blockDim.x) {
    int64_t c = c0 + t;
    if (c >= out_c) continue;
    float x = c < in_c ? Elem<T>::to_f(in[r * in_rs + c * in_cs]) : -INFINITY;
    out[r * out_rs + c * out_cs] = Elem<T>::from_f(expf(x - m) / s);
  }
  (void)in_r;
}

template <typename T>
__global__ void rms_generic_kernel(const T* in, int64_t in_c, int64_t in_rs, int64_t in_cs,
                                   const T* w, int64_t w_n, int64_t w_s, T* out, int64_t out_c,
                                   int64_t out_rs, int64_t out_cs, int64_t cp) {
  __shared__ float sh[32];
  const int64_t r = blockIdx.x;
  float ss = 0.f;
  for (int64_t c = threadIdx.x; c < cp; c += blockDim.x) {
    float x = c < in_c ? Elem<T>::to_f(in[r * in_rs + c * in_cs]) : 0.f;
    ss = fmaf(x, x, ss);
  }
  ss = block_reduce(ss, false, sh);
  const float rinv = 1.0f / sqrtf(ss / (float)in_c + kRmsEps);
  for (int64_t c = threadIdx.x; c < cp; c += blockDim.x) {
    if (c >= out_c) continue;
    float x = c < in_c ? Elem<T>::to_f(in[r * in_rs + c * in_cs]) : 0.f;
    float g = c < w_n ? Elem<T>::to_f(w[c * w_s]) : 0.f;
    out[r * out_rs + c * out_cs] = Elem<T>::from_f(x * rinv * g);
  }
}

template <typename T, bool kSoftmax, int VPL>
static void launch_vec(const T* in, int64_t in_rs, const T* w, T* out, int64_t out_rs,
                       int64_t rows, int cols, cudaStream_t s) {
  const int warps = 8;
  int64_t blocks = cdiv64(rows, warps);
  row_vec_kernel<T, VPL, kSoftmax><<<(unsigned)blocks, warps * 32, 0, s>>>(in, in_rs, w, out,
                                                                           out_rs, rows, cols);
}

template <typename T, bool kSoftmax>
static bool try_vec(const T* in, int64_t in_rs, const T* w, T* out, int64_t out_rs, int64_t rows,
                    int64_t cols, cudaStream_t s) {
  constexpr int N = Pack<T>::N;
  if (cols % N || in_rs % N || out_rs % N || !aligned16(in) || !aligned16(out) ||
      (w && !aligned16(w)))
    return false;
  int64_t per_lane = cdiv64(cols / N, 32);
  if (per_lane <= 1) launch_vec<T, kSoftmax, 1>(in, in_rs, w, out, out_rs, rows, (int)cols, s);
  else if (per_lane <= 2) launch_vec<T, kSoftmax, 2>(in, in_rs, w, out, out_rs, rows, (int)cols, s);
  else if (per_lane <= 4) launch_vec<T, kSoftmax, 4>(in, in_rs, w, out, out_rs, rows, (int)cols, s);
  else if (per_lane <= 8) launch_vec<T, kSoftmax, 8>(in, in_rs, w, out, out_rs, rows, (int)cols, s);
  else if (per_lane <= 16) launch_vec<T, kSoftmax, 16>(in, in_rs, w, out, out_rs, rows, (int)cols, s);
  else return false;
  return true;
}

template <typename T>
static int run_rows(const LaunchArgs& A) {
  const bool softmax = A.kernel == NTB_K_SOFTMAX;
  const int n_t = softmax ? 2 : 3;
  if (A.n_ptrs != n_t) return fail(NTB_ERR_ARG, "rowwise: wrong parameter count");
  if (A.n_meta != 1 || A.meta[0] < 1) return fail(NTB_ERR_ARG, "rowwise: needs COLS_PADDED");
  const int64_t cp = A.meta[0];
  const T* in = (const T*)A.ptrs[0];
  const int64_t ib = A.base[0];
  const int64_t R = A.sizes[ib], C = A.sizes[ib + 1], irs = A.strides[ib], ics = A.strides[ib + 1];
  const int oi = softmax ? 1 : 2;
  T* out = (T*)A.ptrs[oi];
  const int64_t ob = A.base[oi];
  const int64_t OC = A.sizes[ob + 1], ors = A.strides[ob], ocs = A.strides[ob + 1];
  if (A.ranks[0] != 2 || A.ranks[oi] != 2) return fail(NTB_ERR_ARG, "rowwise: rank-2 input/output");
  if (R == 0 || OC == 0) return NTB_OK;
  const T* w = nullptr;
  int64_t wn = 0, ws = 0;
  if (!softmax) {
    if (A.ranks[1] != 1) return fail(NTB_ERR_ARG, "rms_norm: weight must be rank 1");
    w = (const T*)A.ptrs[1];
    wn = A.sizes[A.base[1]];
    ws = A.strides[A.base[1]];
  }
  bool fast = ics == 1 && ocs == 1 && C == OC && cp >= C && (softmax || (ws == 1 && wn == C));
  if (fast) {
    bool ok = softmax ? try_vec<T, true>(in, irs, nullptr, out, ors, R, C, A.stream)
                      : try_vec<T, false>(in, irs, w, out, ors, R, C, A.stream);
    if (ok) return check_launch("rowwise vec", NTB_PATH_ROW_VEC);
  }
  int threads = 256;
  if (softmax) {
    int64_t chunks = cdiv64(C > OC ? C : OC, cp);
    if (chunks < 1) chunks = 1;
    softmax_generic_kernel<T><<<(unsigned)(R * chunks), threads, 0, A.stream>>>(
        in, R, C, irs, ics, out, OC, ors, ocs, cp, chunks);
  } else {
    rms_generic_kernel<T><<<(unsigned)R, threads, 0, A.stream>>>(in, C, irs, ics, w, wn, ws, out,
                                                                 OC, ors, ocs, cp);
  }
  return check_launch("rowwise generic", NTB_PATH_ROW_GENERIC);
}

int launch_rowwise(const LaunchArgs& A) {
  switch (A.dtype) {
    case NTB_F32: return run_rows<float>(A);
    case NTB_F16: return run_rows<__half>(A);
    case NTB_BF16: return run_rows<__nv_bfloat16>(A);
    default: return fail(NTB_ERR_UNSUPPORTED, "rowwise: unsupported dtype");
  }
}

}  // namespace ntb
