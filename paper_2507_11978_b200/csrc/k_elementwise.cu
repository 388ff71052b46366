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
#include <stdlib.h>

#include "common.cuh"

#ifndef NTB_EW_UNROLL
#define NTB_EW_UNROLL 0   // 0: per element type (see run_ew)
#endif

namespace ntb {

// Each op maps a pack of n fp32 values in place (b: the second input).
struct AddOp {
  static constexpr int kIn = 2;
  template <int n>
  __device__ __forceinline__ void apply(float (&a)[n], const float (&b)[n]) const {
#pragma unroll
    for (int e = 0; e < n; ++e) a[e] += b[e];
  }
};
// silu(x) = x / (1 + 2^(-x log2 e)).  Two elements share one reciprocal:
// 1/d0 = d1 / (d0 d1) and 1/d1 = d0 / (d0 d1) while d0 d1 < 2^126 (both
// reciprocals then stay normal fp32); otherwise (x < -43 in one of the two,
// or a NaN) each gets its own.  3 SFU ops per pair instead of 4: at 2^24
// 16-bit elements, 2 SFU ops per element are 7.4 us of SFU time per SMSP
// against 10.3 us of HBM time.
#ifndef NTB_SILU_FMA_EVERY
// 16-bit outputs: every k-th pair's 2^t on the FMA pipe (0: all on the SFU).
// fp32 outputs always use the SFU (the cubic's 7.5e-5 is above fp32's 1e-5
// silu tolerance).  Measured silu fp16 2^24: k = 2 12.2-12.3 us, SFU only
// 12.4-12.7 us.
#define NTB_SILU_FMA_EVERY 2
#endif
struct SiluOp {
  static constexpr int kIn = 1;
  static __device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
  }
  static __device__ __forceinline__ float rcp(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
  }
  // 2^t for a pair on the FMA pipe: t clamped to [-125, 127], t = i + f with
  // i = rint(t) (1.5 * 2^23 trick), 2^f by a cubic (rel. err 7.5e-5, below
  // half an fp16 / bf16 ulp), 2^i added into the exponent field
  static __device__ __forceinline__ float2 ex2_fma(float2 t) {
    t.x = fminf(fmaxf(t.x, -125.f), 127.f);
    t.y = fminf(fmaxf(t.y, -125.f), 127.f);
    const float2 m = __fadd2_rn(t, make_float2(12582912.0f, 12582912.0f));
    const float2 r = __fadd2_rn(m, make_float2(-12582912.0f, -12582912.0f));
    const float2 f = __ffma2_rn(r, make_float2(-1.f, -1.f), t);
    float2 q = __ffma2_rn(f, make_float2(0.0551702793f, 0.0551702793f),
                          make_float2(0.242607975f, 0.242607975f));
    q = __ffma2_rn(q, f, make_float2(0.693260928f, 0.693260928f));
    q = __ffma2_rn(q, f, make_float2(0.999928276f, 0.999928276f));
    return make_float2(__uint_as_float(__float_as_uint(q.x) + (__float_as_uint(m.x) << 23)),
                       __uint_as_float(__float_as_uint(q.y) + (__float_as_uint(m.y) << 23)));
  }
  template <int n>
  __device__ __forceinline__ void apply(float (&x)[n], const float (&)[n]) const {
    static_assert(n % 2 == 0, "pairs");
    constexpr bool kLowp = n == 8;   // 8 values per 16-byte pack: a 16-bit type
#pragma unroll
    for (int e = 0; e < n; e += 2) {
      float d0, d1;
      if (kLowp && NTB_SILU_FMA_EVERY &&
          (e / 2) % (NTB_SILU_FMA_EVERY ? NTB_SILU_FMA_EVERY : 1) == NTB_SILU_FMA_EVERY - 1) {
        const float2 t = ex2_fma(__fmul2_rn(make_float2(x[e], x[e + 1]),
                                            make_float2(-1.4426950408889634f, -1.4426950408889634f)));
        d0 = 1.0f + t.x;
        d1 = 1.0f + t.y;
      } else {
        d0 = 1.0f + ex2(-x[e] * 1.4426950408889634f);
        d1 = 1.0f + ex2(-x[e + 1] * 1.4426950408889634f);
      }
      const float pr = d0 * d1;
      float s0, s1;
      if (pr < 0x1p126f) {
        const float r = rcp(pr);
        s0 = d1 * r;
        s1 = d0 * r;
      } else {
        s0 = rcp(d0);
        s1 = rcp(d1);
      }
      x[e] *= s0;
      x[e + 1] *= s1;
    }
  }
  // one element (generic strided path)
  __device__ __forceinline__ float one(float x) const {
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
      op.apply(fa, fb);
      P r;
      r.from_float(fa);
      st_stream(out + (i + u * stride) * P::N, r.raw);
    }
  }
}

// ---- TMA-bulk streaming path ------------------------------------------------
// Persistent CTAs (one per SM) of 16 warps.  The array is cut into chunks of
// 32 x VPL 16-byte packs per input; chunk c belongs to warp (c mod G) of the
// grid-interleaved warp order (G = grid x 16 warps), as rows are in the
// row-streaming kernel.  Each warp owns a ring of STAGES shared-memory slots
// (one buffer per input), each filled by one cp.async.bulk per input with
// completion on the slot's mbarrier; the warp moves a chunk to registers,
// requests the chunk STAGES ahead into the same slot right away, then
// computes and writes it with 128-bit streaming stores - no per-thread load
// queue.  The first chunks of every warp are requested into L2 before the
// PDL wait.  Measured (silu fp16 2^24, B200): 2 KB chunks, one slot, 16
// warps: 12.6 us; 8 KB chunks 14.4 us (the SFU work of a chunk then runs
// in one burst per warp); 2-4 slots or 32 warps 12.9-14.5 us.
#ifndef NTB_EW_WARPS
#define NTB_EW_WARPS 16
#endif
#ifndef NTB_EW_STAGES
#define NTB_EW_STAGES 1
#endif
#ifndef NTB_EW_VPL1
#define NTB_EW_VPL1 4
#endif
constexpr int kEwWarps = NTB_EW_WARPS;

template <typename T, typename Op, int VPL, int kEwStages>
__global__ void __launch_bounds__(kEwWarps * 32, 1)
    ew_stream_kernel(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ out,
                     int64_t n_vec) {
  using P = Pack<T>;
  constexpr int CH = 32 * VPL;                // packs per chunk
  constexpr uint32_t CH_BYTES = CH * 16;
  constexpr uint32_t SLOT = Op::kIn * CH_BYTES;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[kEwWarps][kEwStages];
  Op op;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem + (size_t)warp * kEwStages * SLOT;
  const int64_t n_chunks = (n_vec + CH - 1) / CH;
  const int64_t step = (int64_t)gridDim.x * kEwWarps;
  const int64_t first = (int64_t)blockIdx.x + (int64_t)gridDim.x * warp;
  auto chunk_bytes = [&](int64_t c) -> uint32_t {
    const int64_t v = n_vec - c * CH;
    return (uint32_t)((v < CH ? v : CH) * 16);
  };
  auto request = [&](int64_t c, int s) {
    const uint32_t nb = chunk_bytes(c);
    uint8_t* buf = ring + s * SLOT;
    bar_expect(&bars[warp][s], nb * Op::kIn);
    bulk_g2s(buf, a + c * CH * P::N, nb, &bars[warp][s]);
    if (Op::kIn == 2) bulk_g2s(buf + CH_BYTES, b + c * CH * P::N, nb, &bars[warp][s]);
  };
#if !NTB_EW_NO_PREFETCH
  if (lane < kEwStages * Op::kIn) {
    const int64_t c = first + (lane / Op::kIn) * step;
    if (c < n_chunks) prefetch_l2_bulk(((lane % Op::kIn) ? b : a) + c * CH * P::N, chunk_bytes(c));
  }
#endif
  pdl_wait();
  pdl_trigger();
  if (lane == 0) {
    for (int s = 0; s < kEwStages; ++s) bar_init(&bars[warp][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < kEwStages; ++s)
      if (first + s * step < n_chunks) request(first + s * step, s);
  }
  __syncwarp();
  int64_t k = 0;
  for (int64_t c = first; c < n_chunks; c += step, ++k) {
    const int s = (int)(k % kEwStages);
    bar_wait(&bars[warp][s], (uint32_t)((k / kEwStages) & 1));
    const uint4* sa = reinterpret_cast<const uint4*>(ring + s * SLOT);
    const uint4* sb = reinterpret_cast<const uint4*>(ring + s * SLOT + CH_BYTES);
    const int64_t v0 = c * CH;
    const int nv = (int)(n_vec - v0 < CH ? n_vec - v0 : CH);
    P va[VPL], vb[VPL];
#pragma unroll
    for (int u = 0; u < VPL; ++u) {
      const int i = lane + 32 * u;
      if (i < nv) {
        va[u].raw = sa[i];
        if (Op::kIn == 2) vb[u].raw = sb[i];
      }
    }
    // all lanes have read the buffer: refill it with the warp's chunk S ahead
    __syncwarp();
    if (lane == 0 && c + kEwStages * step < n_chunks) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      request(c + kEwStages * step, s);
    }
#pragma unroll
    for (int u = 0; u < VPL; ++u) {
      const int i = lane + 32 * u;
      if (i >= nv) break;
      float fa[P::N], fb[P::N];
      va[u].to_float(fa);
      if (Op::kIn == 2) vb[u].to_float(fb);
      op.apply(fa, fb);
      P r;
      r.from_float(fa);
      st_stream(out + (v0 + i) * P::N, r.raw);
    }
  }
}

// Launch the streaming path; false if its shared memory cannot be granted.
template <typename T, typename Op>
static bool try_ew_stream(const T* a, const T* b, T* out, int64_t n_vec, cudaStream_t s) {
  constexpr int VPL = Op::kIn == 1 ? NTB_EW_VPL1 : 8;
  constexpr int64_t CH = 32 * VPL;
  // ring depth: the configured one, capped at 192 KB of buffers per CTA
  constexpr int64_t kMaxStages = (192 * 1024) / (kEwWarps * Op::kIn * CH * 16);
  constexpr int STAGES = NTB_EW_STAGES < kMaxStages ? NTB_EW_STAGES : (kMaxStages > 0 ? kMaxStages : 1);
  const size_t smem = (size_t)kEwWarps * STAGES * Op::kIn * CH * 16;
  auto kern = ew_stream_kernel<T, Op, VPL, STAGES>;
  static size_t attr[kMaxDevices] = {};
  if (smem_attr_once(kern, smem, attr) != cudaSuccess) {
    cudaGetLastError();   // not sticky: the caller falls back to the register-queue kernel
    return false;
  }
  const int64_t n_chunks = cdiv64(n_vec, CH);
  int64_t blocks = cdiv64(n_chunks, kEwWarps);
  if (blocks > sm_count()) blocks = sm_count();
  return launch_pdl(kern, dim3((unsigned)blocks), dim3(kEwWarps * 32), smem, s, a, b, out,
                    n_vec) == cudaSuccess;
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
    float r;
    if constexpr (Op::kIn == 2) r = x + y;
    else r = op.one(x);
    out[i * so] = Elem<T>::from_f(r);
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
    // path choice (measured): the bulk-copy streaming
    // kernel once a launch moves >= 32 MB (silu fp16 2^24: 0.74-0.79 -> 0.81
    // of HBM, add fp32 2^24: 0.97 -> 1.01); below that the register-queue
    // kernel, whose first wave is one L2-prefetched round trip (add fp32
    // 2^20: 3.1-3.3 us vs 3.5-3.6 streaming).  NTB_EW_PATH=vec|stream forces one.
    static const int forced = [] {
      const char* e = getenv("NTB_EW_PATH");
      return !e ? 0 : (e[0] == 's' ? 2 : 1);
    }();
    const int64_t bytes = no * (int64_t)sizeof(T) * (nin + 1);
    const bool stream = forced ? forced == 2 : bytes >= (32ll << 20);
    if (stream && try_ew_stream<T, Op>(a, b, out, n_vec, A.stream))
      return check_launch("elementwise stream", NTB_PATH_EW_STREAM);
    // one wave of 8 resident 256-thread CTAs per SM, each thread U vectors
    // per input in flight per iteration; this kernel now serves launches
    // below 32 MB, where 4 is best (add fp32 2^20: 2.88-3.08 us vs 3.06-3.13
    // with 8, 3.51-3.66 with 2, 3.93-4.07 with 16)
    constexpr int U = NTB_EW_UNROLL ? NTB_EW_UNROLL : 4;
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
