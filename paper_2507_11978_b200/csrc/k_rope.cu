// rope: half-split rotary position embedding (builder-defined; the
// reference declares rope out of scope, catalog.py:36; paper signature
// rope((B,S,H,D), (S,D/2), (S,D/2))).
//
// Logical grid (S, B*H) from catalog.spec_rope: program (s, bh) rotates the
// D-vector x[b, s, h, :] with c = cos[s, :], s_ = sin[s, :]:
//   out[..., :HALF] = x0*c - x1*s_ ;  out[..., HALF:] = x0*s_ + x1*c
// x0/x1 = the two HALF_D halves (loads masked to D, fill 0; table loads
// masked to the table width).
// Fast path: contiguous tensors, 128-bit packs of the first half paired with
// the same packs of the second half; tables (S x HALF) stay L2-resident.
// HBM roofline: 2 x B*S*H*D*sizeof(T) (+ the tables once).
#include "common.cuh"
#include "k_sm100.cuh"

namespace ntb {

template <typename T>
__global__ void __launch_bounds__(256) rope_vec_kernel(const T* __restrict__ x,
                                                       const T* __restrict__ sn,
                                                       const T* __restrict__ cs,
                                                       T* __restrict__ out, int64_t rows,
                                                       int64_t S, int64_t H, int half) {
  using P = Pack<T>;
  pdl_wait();
  pdl_trigger();
  const int vpr = half / P::N;  // packs per half-row
  const int64_t n = rows * vpr;
  const int64_t D = 2 * (int64_t)half;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / vpr;
    const int v = (int)(i - row * vpr);
    const int64_t s = (row / H) % S;
    const T* xr = x + row * D + (int64_t)v * P::N;
    P a, b, c, t;
    a.raw = ld_stream(xr);
    b.raw = ld_stream(xr + half);
    c.raw = ld_keep(cs + s * half + (int64_t)v * P::N);
    t.raw = ld_keep(sn + s * half + (int64_t)v * P::N);
    float fa[P::N], fb[P::N], fc[P::N], ft[P::N], o0[P::N], o1[P::N];
    a.to_float(fa);
    b.to_float(fb);
    c.to_float(fc);
    t.to_float(ft);
#pragma unroll
    for (int k = 0; k < P::N; ++k) {
      o0[k] = fa[k] * fc[k] - fb[k] * ft[k];
      o1[k] = fa[k] * ft[k] + fb[k] * fc[k];
    }
    P r0, r1;
    r0.from_float(o0);
    r1.from_float(o1);
    T* orow = out + row * D + (int64_t)v * P::N;
    st_stream(orow, r0.raw);
    st_stream(orow + half, r1.raw);
  }
}

struct Strides4 { int64_t n[4], s[4]; };

template <typename T>
__global__ void rope_generic_kernel(const T* x, Strides4 xs, const T* sn, int64_t sn_s0,
                                    int64_t sn_s1, int64_t sn_w, const T* cs, int64_t cs_s0,
                                    int64_t cs_s1, int64_t cs_w, T* out, Strides4 os,
                                    int64_t half) {
  // one thread per (s, bh, lane) point of the logical grid
  const int64_t S = xs.n[1], BH = xs.n[0] * xs.n[2];
  const int64_t n = S * BH * half;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = i % half;
    const int64_t bh = (i / half) % BH;
    const int64_t s = i / (half * BH);
    const int64_t xb = bh / xs.n[2], xh = bh % xs.n[2];
    const int64_t ob = bh / os.n[2], oh = bh % os.n[2];
    const T* xr = x + xb * xs.s[0] + s * xs.s[1] + xh * xs.s[2];
    float x0 = l < xs.n[3] ? Elem<T>::to_f(xr[l * xs.s[3]]) : 0.f;
    float x1 = half + l < xs.n[3] ? Elem<T>::to_f(xr[(half + l) * xs.s[3]]) : 0.f;
    float sv = l < sn_w ? Elem<T>::to_f(sn[s * sn_s0 + l * sn_s1]) : 0.f;
    float cv = l < cs_w ? Elem<T>::to_f(cs[s * cs_s0 + l * cs_s1]) : 0.f;
    T* orow = out + ob * os.s[0] + s * os.s[1] + oh * os.s[2];
    if (l < os.n[3]) orow[l * os.s[3]] = Elem<T>::from_f(x0 * cv - x1 * sv);
    if (half + l < os.n[3]) orow[(half + l) * os.s[3]] = Elem<T>::from_f(x0 * sv + x1 * cv);
  }
}

template <typename T>
static int run_rope(const LaunchArgs& A) {
  if (A.n_ptrs != 4 || A.ranks[0] != 4 || A.ranks[1] != 2 || A.ranks[2] != 2 || A.ranks[3] != 4)
    return fail(NTB_ERR_ARG, "rope: expects input(4), sin(2), cos(2), output(4)");
  if (A.n_meta != 1 || A.meta[0] < 1) return fail(NTB_ERR_ARG, "rope: needs HALF_D");
  const int64_t half = A.meta[0];
  Strides4 xs, os;
  for (int d = 0; d < 4; ++d) {
    xs.n[d] = A.sizes[A.base[0] + d];
    xs.s[d] = A.strides[A.base[0] + d];
    os.n[d] = A.sizes[A.base[3] + d];
    os.s[d] = A.strides[A.base[3] + d];
  }
  const int64_t* sz = A.sizes;
  const int64_t* st = A.strides;
  const int64_t sb = A.base[1], cb = A.base[2];
  const T* x = (const T*)A.ptrs[0];
  const T* sn = (const T*)A.ptrs[1];
  const T* cs = (const T*)A.ptrs[2];
  T* out = (T*)A.ptrs[3];
  const int64_t rows = xs.n[0] * xs.n[1] * xs.n[2];
  if (rows == 0) return NTB_OK;
  constexpr int N = Pack<T>::N;
  bool contig_x = xs.s[3] == 1 && xs.s[2] == xs.n[3] && xs.s[1] == xs.n[2] * xs.n[3] &&
                  xs.s[0] == xs.n[1] * xs.s[1];
  bool same = true;
  for (int d = 0; d < 4; ++d) same = same && xs.n[d] == os.n[d] && xs.s[d] == os.s[d];
  bool fast = contig_x && same && xs.n[3] == 2 * half && half % N == 0 && sz[sb + 1] == half &&
              sz[cb + 1] == half && st[sb + 1] == 1 && st[cb + 1] == 1 && st[sb] == half &&
              st[cb] == half && aligned16(x) && aligned16(out) && aligned16(sn) &&
              aligned16(cs) && sz[sb] >= xs.n[1] && sz[cb] >= xs.n[1];
  const int sms = sm_count();
  if (fast) {
    int64_t items = rows * (half / N);
    int64_t blocks = cdiv64(items, 256);
    if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
    launch_pdl(rope_vec_kernel<T>, dim3((unsigned)blocks), dim3(256), 0, A.stream, x, sn, cs, out,
               rows, xs.n[1], xs.n[2], (int)half);
    return check_launch("rope", NTB_PATH_ROPE_VEC);
  } else {
    int64_t items = xs.n[1] * xs.n[0] * xs.n[2] * half;
    int64_t blocks = cdiv64(items, 256);
    if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
    rope_generic_kernel<T><<<(unsigned)blocks, 256, 0, A.stream>>>(
        x, xs, sn, st[sb], st[sb + 1], sz[sb + 1], cs, st[cb], st[cb + 1], sz[cb + 1], out, os,
        half);
  }
  return check_launch("rope", NTB_PATH_ROPE_GENERIC);
}

int rope_rows_vec(const void* x, const void* sn, const void* cs, void* out, int64_t rows,
                  int64_t S, int64_t pos_div, int half, int dtype, cudaStream_t s) {
  const int sms = sm_count();
  auto go = [&](auto tag) {
    using T = decltype(tag);
    constexpr int N = Pack<T>::N;
    int64_t items = rows * (half / N);
    int64_t blocks = cdiv64(items, 256);
    if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
    if (blocks < 1) blocks = 1;
    launch_pdl(rope_vec_kernel<T>, dim3((unsigned)blocks), dim3(256), 0, s, (const T*)x,
               (const T*)sn, (const T*)cs, (T*)out, rows, S, pos_div, half);
    return check_launch("rope (sdpa_rope K pre-pass)", NTB_PATH_ROPE_VEC);
  };
  if (dtype == NTB_F16) return go(__half());
  if (dtype == NTB_BF16) return go(__nv_bfloat16());
  return NTB_ERR_UNSUPPORTED;
}

int launch_rope(const LaunchArgs& A) {
  switch (A.dtype) {
    case NTB_F32: return run_rope<float>(A);
    case NTB_F16: return run_rope<__half>(A);
    case NTB_BF16: return run_rope<__nv_bfloat16>(A);
    default: return fail(NTB_ERR_UNSUPPORTED, "rope: unsupported dtype");
  }
}

}  // namespace ntb
