// add / silu: the tile((BLOCK_SIZE,)) elementwise family
// (reference catalog.py:121-152; emitted add.py.golden / silu.py.golden).
//
// Logical program p of the reference grid covers elements [p*B, p*B + B) of
// every parameter, each load masked against its own size (fill 0) and the
// store masked against the output size (add.py.golden:26-30).  The union of
// the logical programs is [0, grid*B), so the whole op is
//     out[i] = f(in[i] (i < n_in else 0), other[i] (i < n_other else 0))
// for i < n_out.  BLOCK_SIZE only shapes the logical grid; the physical
// launch is a grid-stride loop of 128-bit vectors sized to the SM count.
//
// HBM roofline: add moves 3 x n x sizeof(T) bytes, silu 2 x n x sizeof(T).
#include "common.cuh"

#ifndef NTB_EW_UNROLL
#define NTB_EW_UNROLL 0   // 0: per element type (see run_ew)
#endif

namespace ntb {

struct AddOp {
  static constexpr int kIn = 2;
  __device__ __forceinline__ float operator()(float a, float b) const { return a + b; }
};
struct SiluOp {
  static constexpr int kIn = 1;
  __device__ __forceinline__ float operator()(float x, float) const {
    return __fdividef(x, 1.0f + exp2f(-x * 1.4426950408889634f));
  }
};

template <typename T, typename Op, int UNROLL>
__global__ void __launch_bounds__(256) ew_vec_kernel(const T* __restrict__ a,
                                                     const T* __restrict__ b,
                                                     T* __restrict__ out, int64_t n_vec) {
  using P = Pack<T>;
  Op op;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
#if !NTB_EW_NO_PREFETCH
  // this CTA's first-iteration inputs: UNROLL runs of 256 vectors each,
  // when the whole first wave fits in L2 next to the previous kernel's data
  // (add fp32 2^24 = 78 MB of first wave measured 0.97 -> 0.93 with it)
  const int64_t wave_vec = n_vec < stride * UNROLL ? n_vec : stride * UNROLL;
  if (wave_vec * 16 * Op::kIn <= (32ll << 20) && threadIdx.x < UNROLL * Op::kIn) {
    const int u = threadIdx.x % UNROLL;
    const int64_t v0 = (int64_t)blockIdx.x * blockDim.x + u * stride;
    if (v0 < n_vec) {
      const int64_t nv = n_vec - v0 < (int64_t)blockDim.x ? n_vec - v0 : (int64_t)blockDim.x;
      prefetch_l2_bulk((threadIdx.x < UNROLL ? a : b) + v0 * P::N, (uint32_t)(nv * 16));
    }
  }
#endif
  pdl_wait();
  pdl_trigger();
  // every iteration keeps UNROLL vectors per input in flight; the last one
  // is predicated per vector (no serial one-vector tail loop)
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_vec;
       i += UNROLL * stride) {
    P va[UNROLL], vb[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      if (i + u * stride < n_vec) {
        va[u].raw = ld_stream(a + (i + u * stride) * P::N);
        if (Op::kIn == 2) vb[u].raw = ld_stream(b + (i + u * stride) * P::N);
      }
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      if (i + u * stride >= n_vec) break;
      float fa[P::N], fb[P::N];
      va[u].to_float(fa);
      if (Op::kIn == 2) vb[u].to_float(fb);
#pragma unroll
      for (int k = 0; k < P::N; ++k) fa[k] = op(fa[k], Op::kIn == 2 ? fb[k] : 0.f);
      P r;
      r.from_float(fa);
      st_stream(out + (i + u * stride) * P::N, r.raw);
    }
  }
}

// Generic path: any element strides / mismatched sizes / unaligned bases.
template <typename T, typename Op>
__global__ void ew_generic_kernel(const T* a, int64_t na, int64_t sa, const T* b, int64_t nb,
                                  int64_t sb, T* out, int64_t no, int64_t so) {
  Op op;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < no;
       i += (int64_t)gridDim.x * blockDim.x) {
    float x = i < na ? Elem<T>::to_f(a[i * sa]) : 0.f;
    float y = (Op::kIn == 2 && i < nb) ? Elem<T>::to_f(b[i * sb]) : 0.f;
    out[i * so] = Elem<T>::from_f(op(x, y));
  }
}

template <typename T, typename Op>
static int run_ew(const LaunchArgs& A) {
  const int nin = Op::kIn;
  const T* a = (const T*)A.ptrs[0];
  const T* b = nin == 2 ? (const T*)A.ptrs[1] : nullptr;
  T* out = (T*)A.ptrs[nin];
  int64_t na = A.sizes[A.base[0]], sa = A.strides[A.base[0]];
  int64_t nb = nin == 2 ? A.sizes[A.base[1]] : 0, sb = nin == 2 ? A.strides[A.base[1]] : 0;
  int64_t no = A.sizes[A.base[nin]], so = A.strides[A.base[nin]];
  if (no == 0) return NTB_OK;
  constexpr int N = Pack<T>::N;
  bool fast = sa == 1 && so == 1 && na == no && aligned16(a) && aligned16(out) && no % N == 0 &&
              (nin == 1 || (sb == 1 && nb == no && aligned16(b)));
  const int sms = sm_count();
  if (fast) {
    int64_t n_vec = no / N;
    // one wave of 8 resident 256-thread CTAs per SM, each thread U vectors
    // per input in flight per iteration (measured: 8 for fp32 add 2^24 =
    // 0.97 of HBM, 4 for the 16-bit silu 2^24 = 0.80)
    constexpr int U = NTB_EW_UNROLL ? NTB_EW_UNROLL : (sizeof(T) == 4 ? 8 : 4);
    int64_t blocks = cdiv64(n_vec, 256 * U);
    int64_t cap = (int64_t)sms * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    launch_pdl(ew_vec_kernel<T, Op, U>, dim3((unsigned)blocks), dim3(256), 0, A.stream, a, b, out,
               n_vec);
    return check_launch("elementwise", NTB_PATH_EW_VEC);
  } else {
    int64_t blocks = cdiv64(no, 256);
    if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
    ew_generic_kernel<T, Op><<<(unsigned)blocks, 256, 0, A.stream>>>(a, na, sa, b, nb, sb, out,
                                                                      no, so);
  }
  return check_launch("elementwise", NTB_PATH_EW_GENERIC);
}

int launch_elementwise(const LaunchArgs& A) {
  const bool is_add = A.kernel == NTB_K_ADD;
  if (A.n_ptrs != (is_add ? 3 : 2)) return fail(NTB_ERR_ARG, "elementwise: wrong parameter count");
  for (int i = 0; i < A.n_ptrs; ++i)
    if (A.ranks[i] != 1) return fail(NTB_ERR_ARG, "elementwise: parameters must be rank 1");
  switch (A.dtype) {
    case NTB_F32: return is_add ? run_ew<float, AddOp>(A) : run_ew<float, SiluOp>(A);
    case NTB_F16: return is_add ? run_ew<__half, AddOp>(A) : run_ew<__half, SiluOp>(A);
    case NTB_BF16:
      return is_add ? run_ew<__nv_bfloat16, AddOp>(A) : run_ew<__nv_bfloat16, SiluOp>(A);
    default: return fail(NTB_ERR_UNSUPPORTED, "elementwise: unsupported dtype");
  }
}

}  // namespace ntb
