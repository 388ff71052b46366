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

#include <type_traits>

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


// ---- TMA-bulk row streaming (the B200 fast path) --------------------------
// Persistent CTAs of 8 warps; every warp owns a private ring of S row
// buffers in shared memory filled by cp.async.bulk (global -> shared, one
// bulk copy per row, completion on a per-buffer mbarrier), so each SM keeps
// 8 x (S-1) rows (>= 100 KB) in flight - enough to cover HBM latency at full
// bandwidth.  The warp reduces its row out of shared memory (warp shuffles,
// fp32) and writes the result with 128-bit streaming stores.
constexpr int kStreamWarps = 16;
#ifndef NTB_ROWS_REG
#define NTB_ROWS_REG 1
#endif

constexpr int kStreamMaxStages = 8;

__device__ __forceinline__ float fast_exp(float x) { return exp2f(x * 1.4426950408889634f); }


// ---- 16-bit rows (fp16 / bf16): 16-bit I/O, fp32 arithmetic ----------------
// The reference simulates every kernel in f32 (catalog.py:155-
// 223).  Here every arithmetic operation is fp32: sm_100 has mixed-precision
// FHADD / FHFMA (f32 result from f16 or bf16 register halves, PTX
// add/sub/fma .f32.f16 / .f32.bf16), so a 16-bit element enters fp32 math
// without a separate conversion.
//   rms_norm: sum of x*x by FHFMA (each product exact in fp32, one rounding
//     per accumulate: no scaling and no underflow for any 16-bit input);
//     out = (x*w) * (1 / sqrt(ss / C + eps)): x*w is exact in fp32 (FHFMA
//     with a zero addend), so the output carries one fp32 rounding + the
//     store rounding.
//   softmax: row max on the 16-bit pairs (HMNMX2, exact); d = x - m by FHADD
//     (fp32), e = 2^(d log2 e) on the SFU (one ex2 per element), s = sum e
//     in fp32.  e is held in the row's 16-bit type between the sum and the
//     normalisation (the row stays register-resident: 64 registers a lane),
//     so the output e * (1/s), computed in fp32, has two 16-bit roundings:
//     <= 1 ulp of the output type (a single rounding would be 0.5 ulp).
//     Recomputing e instead costs a second ex2 per element and made the
//     kernel SFU-bound (14.4 vs 10.8 us at 4096 x 4096, B200).
template <typename T> struct Pair16;
template <> struct Pair16<__half> {
  static __device__ __forceinline__ float2 f2(uint32_t u) {
    return __half22float2(*reinterpret_cast<const __half2*>(&u));
  }
  static __device__ __forceinline__ uint32_t pk(float2 f) {
    const __half2 h = __float22half2_rn(f);
    return *reinterpret_cast<const uint32_t*>(&h);
  }
  static __device__ __forceinline__ uint32_t mx(uint32_t a, uint32_t b) {
    const __half2 r = __hmax2(*reinterpret_cast<const __half2*>(&a),
                              *reinterpret_cast<const __half2*>(&b));
    return *reinterpret_cast<const uint32_t*>(&r);
  }
  // a + c and a * b + c with 16-bit a, b and fp32 c, d
  static __device__ __forceinline__ float hadd(uint16_t a, float c) {
    float d;
    asm("add.f32.f16 %0, %1, %2;" : "=f"(d) : "h"(a), "f"(c));
    return d;
  }
  static __device__ __forceinline__ float hfma(uint16_t a, uint16_t b, float c) {
    float d;
    asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d) : "h"(a), "h"(b), "f"(c));
    return d;
  }
  static constexpr uint32_t kNegInf2 = 0xFC00FC00u;
};
template <> struct Pair16<__nv_bfloat16> {
  static __device__ __forceinline__ float2 f2(uint32_t u) {
    return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xFFFF0000u));
  }
  static __device__ __forceinline__ uint32_t pk(float2 f) {
    const __nv_bfloat162 h = __float22bfloat162_rn(f);
    return *reinterpret_cast<const uint32_t*>(&h);
  }
  static __device__ __forceinline__ uint32_t mx(uint32_t a, uint32_t b) {
    const __nv_bfloat162 r = __hmax2(*reinterpret_cast<const __nv_bfloat162*>(&a),
                                     *reinterpret_cast<const __nv_bfloat162*>(&b));
    return *reinterpret_cast<const uint32_t*>(&r);
  }
  static __device__ __forceinline__ float hadd(uint16_t a, float c) {
    float d;
    asm("add.f32.bf16 %0, %1, %2;" : "=f"(d) : "h"(a), "f"(c));
    return d;
  }
  static __device__ __forceinline__ float hfma(uint16_t a, uint16_t b, float c) {
    float d;
    asm("fma.rn.f32.bf16 %0, %1, %2, %3;" : "=f"(d) : "h"(a), "h"(b), "f"(c));
    return d;
  }
  static constexpr uint32_t kNegInf2 = 0xFF80FF80u;
};

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t w4(const uint4& v, int k) {
  return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w;
}
__device__ __forceinline__ uint16_t lo16(uint32_t u) { return (uint16_t)(u & 0xFFFFu); }
__device__ __forceinline__ uint16_t hi16(uint32_t u) { return (uint16_t)(u >> 16); }

constexpr float kLog2e = 1.4426950408889634f;

// Per-pack (8 elements) steps shared by the register-resident and the
// shared-memory variants.
template <typename T>
struct Row16 {
  using H = Pair16<T>;
  static __device__ __forceinline__ uint32_t pack_max(uint32_t acc, const uint4& v) {
    return H::mx(acc, H::mx(H::mx(v.x, v.y), H::mx(v.z, v.w)));
  }
  static __device__ __forceinline__ float pair_max(uint32_t p) {
    const float2 f = H::f2(p);
    return fmaxf(f.x, f.y);
  }
  // e = 2^((x - m) log2 e) of one pack, returned in T; acc += e (fp32)
  static __device__ __forceinline__ uint4 exp_pack(const uint4& v, float nm, float2& acc) {
    const float2 l2e = make_float2(kLog2e, kLog2e);
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t u = w4(v, k);
      const float2 t = __fmul2_rn(make_float2(H::hadd(lo16(u), nm), H::hadd(hi16(u), nm)), l2e);
      const float2 e = make_float2(ex2f(t.x), ex2f(t.y));
      acc = __fadd2_rn(acc, e);
      o[k] = H::pk(e);
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
  }
  static __device__ __forceinline__ uint4 scale_pack(const uint4& e, float inv) {
    const float2 i2 = make_float2(inv, inv);
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) o[k] = H::pk(__fmul2_rn(H::f2(w4(e, k)), i2));
    return make_uint4(o[0], o[1], o[2], o[3]);
  }
  static __device__ __forceinline__ void sq_pack(const uint4& v, float (&acc)[4]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t u = w4(v, k);
      acc[k] = H::hfma(hi16(u), hi16(u), H::hfma(lo16(u), lo16(u), acc[k]));
    }
  }
  static __device__ __forceinline__ uint4 rms_pack(const uint4& v, const uint4& g, float r) {
    const float2 r2 = make_float2(r, r);
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t u = w4(v, k), q = w4(g, k);
      const float2 xw = make_float2(H::hfma(lo16(u), lo16(q), 0.f), H::hfma(hi16(u), hi16(q), 0.f));
      o[k] = H::pk(__fmul2_rn(xw, r2));
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
  }
  static __device__ __forceinline__ float rinv(const float (&acc)[4], int cols) {
    const float ss = warp_sum((acc[0] + acc[1]) + (acc[2] + acc[3]));
    return 1.0f / sqrtf(ss / (float)cols + kRmsEps);
  }
};

template <typename T>
__device__ __forceinline__ void softmax_row16(const uint4* buf, T* dst, int n_vec, int lane) {
  using R = Row16<T>;
  uint32_t mx = Pair16<T>::kNegInf2;
  for (int c = lane; c < n_vec; c += 32) mx = R::pack_max(mx, buf[c]);
  const float nm = -warp_max(R::pair_max(mx));
  float2 s2 = make_float2(0.f, 0.f);
  uint4* ebuf = const_cast<uint4*>(buf);   // e overwrites the row in place
  for (int c = lane; c < n_vec; c += 32) ebuf[c] = R::exp_pack(buf[c], nm, s2);
  const float inv = 1.0f / warp_sum(s2.x + s2.y);
  for (int c = lane; c < n_vec; c += 32) st_stream(dst + (int64_t)c * 8, R::scale_pack(buf[c], inv));
}

template <typename T>
__device__ __forceinline__ void rms_row16(const uint4* buf, const uint4* wv, T* dst, int n_vec,
                                          int cols, int lane) {
  using R = Row16<T>;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int c = lane; c < n_vec; c += 32) R::sq_pack(buf[c], acc);
  const float r = R::rinv(acc, cols);
  for (int c = lane; c < n_vec; c += 32) st_stream(dst + (int64_t)c * 8, R::rms_pack(buf[c], wv[c], r));
}

// Register-resident variants for rows of exactly 32 * VPL packs (4096
// 16-bit columns = VPL 16): the row is read from shared memory ONCE into
// registers (64 per lane) and every pass runs there.
template <typename T, int VPL>
__device__ __forceinline__ void softmax_row16_reg(uint4 (&v)[VPL], T* dst, int lane) {
  using R = Row16<T>;
  uint32_t mx = Pair16<T>::kNegInf2;
#pragma unroll
  for (int u = 0; u < VPL; ++u) mx = R::pack_max(mx, v[u]);
  const float nm = -warp_max(R::pair_max(mx));
  float2 sa = make_float2(0.f, 0.f), sb = sa;
#pragma unroll
  for (int u = 0; u < VPL; ++u) v[u] = R::exp_pack(v[u], nm, (u & 1) ? sb : sa);
  const float inv = 1.0f / warp_sum((sa.x + sa.y) + (sb.x + sb.y));
#pragma unroll
  for (int u = 0; u < VPL; ++u) st_stream(dst + (int64_t)(lane + 32 * u) * 8, R::scale_pack(v[u], inv));
}

template <typename T, int VPL>
__device__ __forceinline__ void rms_row16_reg(const uint4 (&v)[VPL], const uint4* wv, T* dst,
                                              int cols, int lane) {
  using R = Row16<T>;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int u = 0; u < VPL; ++u) R::sq_pack(v[u], acc);
  const float r = R::rinv(acc, cols);
#pragma unroll
  for (int u = 0; u < VPL; ++u)
    st_stream(dst + (int64_t)(lane + 32 * u) * 8, R::rms_pack(v[u], wv[lane + 32 * u], r));
}

template <typename T, bool kSoftmax>
__global__ void __launch_bounds__(kStreamWarps * 32, 1)
    row_stream_kernel(const T* __restrict__ in, int64_t in_rs, const T* __restrict__ w,
                      T* __restrict__ out, int64_t out_rs, int64_t rows, int cols, int stages) {
  using P = Pack<T>;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[kStreamWarps][kStreamMaxStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t row_bytes = (uint32_t)cols * sizeof(T);
  const uint32_t row_pad = (row_bytes + 127u) & ~127u;
  uint8_t* wbase = smem + (size_t)warp * stages * row_pad;
  // row r goes to CTA r % grid: every SM gets floor or ceil(rows / grid) rows
  // (a block of 16 consecutive rows per CTA gives 4096 rows on 148 SMs as
  // 108 CTAs x 32 rows + 40 x 16 - a 16% longer critical path)
  const int64_t step = (int64_t)gridDim.x * kStreamWarps;
  const int64_t first = (int64_t)blockIdx.x + (int64_t)gridDim.x * warp;
#if !NTB_ROWS_NO_PREFETCH
  // the warp's first rows into L2 while the previous kernel drains
  if (lane < stages && first + lane * step < rows && (row_bytes & 15) == 0)
    prefetch_l2_bulk(in + (first + lane * step) * in_rs, row_bytes);
#endif
  pdl_wait();
  pdl_trigger();
  // each warp's first row copies are in flight before anything else
  if (lane == 0) {
    for (int s = 0; s < stages; ++s) bar_init(&bars[warp][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < stages; ++s) {
      const int64_t r = first + s * step;
      if (r < rows) {
        bar_expect(&bars[warp][s], row_bytes);
        bulk_g2s(wbase + (size_t)s * row_pad, in + r * in_rs, row_bytes, &bars[warp][s]);
      }
    }
  }
  const T* wsh = nullptr;
  if (!kSoftmax) {
    // weight row once per CTA, after the per-warp rings
    uint8_t* wdst = smem + (size_t)kStreamWarps * stages * row_pad;
    for (int c = threadIdx.x; c < cols / P::N; c += blockDim.x)
      reinterpret_cast<uint4*>(wdst)[c] = reinterpret_cast<const uint4*>(w)[c];
    wsh = reinterpret_cast<const T*>(wdst);
  }
  __syncthreads();
  const int n_vec = cols / P::N;
  int64_t k = 0;
  for (int64_t r = first; r < rows; r += step, ++k) {
    const int s = (int)(k % stages);
    bar_wait(&bars[warp][s], (uint32_t)((k / stages) & 1));
    const uint4* buf = reinterpret_cast<const uint4*>(wbase + (size_t)s * row_pad);
    T* dst = out + r * out_rs;
    // release the buffer (all lanes done reading) and refill it with the
    // warp's next row
    auto refill = [&]() {
      __syncwarp();
      if (lane == 0) {
        const int64_t nr = r + (int64_t)stages * step;
        if (nr < rows) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          bar_expect(&bars[warp][s], row_bytes);
          bulk_g2s(wbase + (size_t)s * row_pad, in + nr * in_rs, row_bytes, &bars[warp][s]);
        }
      }
    };
    if constexpr (sizeof(T) == 2) {
      if (n_vec == 32 * 16 && NTB_ROWS_REG) {
        // the row moves to registers and the next row's copy starts before
        // any of this row's math or stores
        uint4 v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = buf[lane + 32 * u];
        refill();
        if (kSoftmax) softmax_row16_reg<T, 16>(v, dst, lane);
        else rms_row16_reg<T, 16>(v, reinterpret_cast<const uint4*>(wsh), dst, cols, lane);
        continue;
      } else if (kSoftmax) {
        softmax_row16<T>(buf, dst, n_vec, lane);
      } else {
        rms_row16<T>(buf, reinterpret_cast<const uint4*>(wsh), dst, n_vec, cols, lane);
      }
    } else if (kSoftmax) {
      // fp32 rows. pass 1: row max; pass 2: e = exp(x - m) written back in
      // place (fp32, exact) + row sum; pass 3: e / sum.
      using E = float;
      float m = -INFINITY;
      for (int c = lane; c < n_vec; c += 32) {
        P v;
        v.raw = buf[c];
        float f[P::N];
        v.to_float(f);
#pragma unroll
        for (int e = 0; e < P::N; ++e) m = fmaxf(m, f[e]);
      }
      m = warp_max(m);
      float sum = 0.f;
      uint4* ebuf = const_cast<uint4*>(buf);
      for (int c = lane; c < n_vec; c += 32) {
        P v;
        v.raw = buf[c];
        float f[P::N];
        v.to_float(f);
#pragma unroll
        for (int e = 0; e < P::N; ++e) {
          f[e] = fast_exp(f[e] - m);
          sum += f[e];
        }
        Pack<E> o;
        o.from_float(f);
        ebuf[c] = o.raw;
      }
      const float inv = 1.0f / warp_sum(sum);
      for (int c = lane; c < n_vec; c += 32) {
        Pack<E> v;
        v.raw = buf[c];
        float f[P::N];
        v.to_float(f);
#pragma unroll
        for (int e = 0; e < P::N; ++e) f[e] *= inv;
        P o;
        o.from_float(f);
        st_stream(dst + (int64_t)c * P::N, o.raw);
      }
    } else {
      float ss = 0.f;
      for (int c = lane; c < n_vec; c += 32) {
        P v;
        v.raw = buf[c];
        float f[P::N];
        v.to_float(f);
#pragma unroll
        for (int e = 0; e < P::N; ++e) ss = fmaf(f[e], f[e], ss);
      }
      const float rinv = 1.0f / sqrtf(warp_sum(ss) / (float)cols + kRmsEps);
      const uint4* wv = reinterpret_cast<const uint4*>(wsh);
      for (int c = lane; c < n_vec; c += 32) {
        P v, g;
        v.raw = buf[c];
        g.raw = wv[c];
        float f[P::N], gf[P::N];
        v.to_float(f);
        g.to_float(gf);
#pragma unroll
        for (int e = 0; e < P::N; ++e) f[e] = f[e] * rinv * gf[e];
        P o;
        o.from_float(f);
        st_stream(dst + (int64_t)c * P::N, o.raw);
      }
    }
    refill();
  }
}

template <typename T, bool kSoftmax>
static bool try_stream(const T* in, int64_t in_rs, const T* w, T* out, int64_t out_rs,
                       int64_t rows, int64_t cols, cudaStream_t s) {
  constexpr int N = Pack<T>::N;
  const int64_t row_bytes = cols * (int64_t)sizeof(T);
  if (cols % N || (in_rs * (int64_t)sizeof(T)) % 16 || out_rs % N || !aligned16(in) ||
      !aligned16(out) || (w && !aligned16(w)) || rows < 1)
    return false;
  const int64_t row_pad = (row_bytes + 127) & ~int64_t(127);
  const int64_t budget = 200 * 1024 - (kSoftmax ? 0 : row_pad);
  int64_t stages = budget / (kStreamWarps * row_pad);
  if (stages > kStreamMaxStages) stages = kStreamMaxStages;
  if (stages < 1) return false;
  const size_t smem = (size_t)(kStreamWarps * stages * row_pad + (kSoftmax ? 0 : row_pad));
  auto kern = row_stream_kernel<T, kSoftmax>;
  static size_t attr[kMaxDevices] = {};
  if (smem_attr_once(kern, smem, attr) != cudaSuccess) return false;
  int64_t blocks = cdiv64(rows, kStreamWarps);
  if (blocks > sm_count()) blocks = sm_count();
  launch_pdl(kern, dim3((unsigned)blocks), dim3(kStreamWarps * 32), smem, s, in, in_rs, w, out,
             out_rs, rows, (int)cols, (int)stages);
  return true;
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
    bool ok = softmax ? try_stream<T, true>(in, irs, nullptr, out, ors, R, C, A.stream)
                      : try_stream<T, false>(in, irs, w, out, ors, R, C, A.stream);
    if (ok) return check_launch("rowwise stream", NTB_PATH_ROW_STREAM);
    ok = softmax ? try_vec<T, true>(in, irs, nullptr, out, ors, R, C, A.stream)
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
