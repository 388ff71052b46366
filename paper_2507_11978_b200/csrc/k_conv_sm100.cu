// conv2d (NCHW, stride 1, no padding) as an implicit GEMM on the sm_100a
// tensor cores (reference catalog.py:295-330, conv2d.py.golden; oracle.py:64-80).
//
// The reference lowers conv2d to the matmul arrangement over
//   M = N*P*Q pixels, K = C*R*S, N = K_out
// with the image addressed through mixed-radix // and % maps
// (conv2d.py.golden:56).  On B200 the same product is computed transposed,
//   D[k_out, pixel] = sum_{(r,s), c} W'[k_out, (r,s), c] * X[c, pixel + r*W + s]
// where "pixel" runs over a VIRTUAL output row width of W (not Q): for a
// fixed (r, s) the 256 pixels of a tile then read one contiguous run of
// image pixels starting at pixel + r*W + s, i.e. a plain 2-D TMA box of the
// image viewed as [N][H*W][C] (channels innermost, K-major operand) - no
// im2col buffer.  The W - Q "virtual" columns (2 of 56 at the BASELINE
// shape) are computed and discarded (96.4% useful work).
// TMA needs the innermost box coordinate 16-byte aligned, so the (r, s)
// shift must fall on the pixel dimension, not the innermost one: NCHW
// inputs are therefore transposed once per call to [N][H*W][C8] (C padded
// to a multiple of 8) by a tiled smem transpose (2 x image bytes of HBM
// traffic); channels_last inputs are consumed in place.  The filter is
// repacked to W'[k_out][(r,s)][C8] (K-major).
//
// Pipeline = the CTA-pair GEMM of k_gemm_sm100.cu: 2-SM clusters, tile
// 256 (k_out) x 256 (pixels), 6-stage TMA ring, tcgen05.mma.cta_group::2,
// double-buffered TMEM accumulators, and an epilogue that transposes each
// 32x32 accumulator block through shared memory so that a warp's stores run
// along the output rows (coalesced NCHW writes).
// Tensor roofline: 2*N*P*Q*K*C*R*S flop per launch.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <stdio.h>
#include <stdlib.h>

#include <type_traits>

#include "common.cuh"
#include "k_sm100.cuh"
#include "sm100_ptx.cuh"

namespace ntb {
namespace {

constexpr int BK = 64;
constexpr int STAGES = 6;          // unfused (NHWC / TMA image) kernel
#ifndef NTB_CONV_FSTAGES
#define NTB_CONV_FSTAGES 6
#endif
constexpr int FSTAGES = NTB_CONV_FSTAGES;   // fused kernel's filter ring (max)
constexpr int A_BYTES = 128 * BK * 2;
constexpr int B_BYTES = 128 * BK * 2;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int XPOSE_FLOATS = 32 * 33;                       // per epilogue warp
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024;  // + static xpose buffer
constexpr int TMEM_COLS = 512;

struct ConvMaps {
  CUtensorMap w;  // W' dims {C8, RS, K}
  CUtensorMap x;  // X' dims {C8, H*W, N} (channels innermost)
};

struct ConvParams {
  int N, C, H, W, K, R, S, P, Q;
  int cb;            // channel blocks of 64
  int pix_tiles;     // per image: cdiv(P*W, 256)
  int k_tiles;       // cdiv(K, 256)
  void* y;
  int64_t ys[4];
};

// W'[k][rs][c8] <- W[k][c][r][s] (zero for c >= C)
template <typename T>
__global__ void repack_filter(const T* __restrict__ w, int64_t s0, int64_t s1, int64_t s2,
                              int64_t s3, T* __restrict__ out, int K, int C, int C8, int R,
                              int S) {
  const int64_t total = (int64_t)K * R * S * C8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C8);
    const int64_t rest = i / C8;
    const int rs = (int)(rest % (R * S));
    const int k = (int)(rest / (R * S));
    const int r = rs / S, s = rs % S;
    out[i] = c < C ? w[k * s0 + c * s1 + r * s2 + s * s3] : T(0.f);
  }
}

// X'[n][pix][c8] <- X[n][c][pix]: 64 channels x 64 pixels per CTA.  Each
// thread loads 8 pixels of a channel PAIR (two 128-bit loads), packs the
// pair per pixel into 32-bit words and writes them to a [pixel][pair] tile
// (row pitch 36 words: bank-conflict-free both ways); the store phase reads
// 128-bit runs of 8 channels per pixel and writes 128 B per pixel.
template <typename T>
__global__ void __launch_bounds__(256) nchw_to_nhwc(const T* __restrict__ x, int64_t sn,
                                                    int64_t sc, T* __restrict__ out, int C,
                                                    int C8, int HW) {
  constexpr int TP = 64, PITCH = 36;          // pixels per tile, words per row
  __shared__ __align__(16) uint32_t tile[TP * PITCH];
  const int n = blockIdx.z;
  const int c0 = blockIdx.y * 64, p0 = blockIdx.x * TP;
  const uint16_t* src = reinterpret_cast<const uint16_t*>(x) + (int64_t)n * sn;
  const bool vec_ok = (sc % 8) == 0 && (HW % 8) == 0 && ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
  {
    const int cw = threadIdx.x & 31, pb = threadIdx.x >> 5;   // channel pair, 8-pixel block
    const int pix = p0 + pb * 8;
    uint16_t a[8], b[8];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint16_t* e = h ? b : a;
      const int c = c0 + 2 * cw + h;
      if (c < C && vec_ok && pix + 8 <= HW) {
        const uint4 v = *reinterpret_cast<const uint4*>(src + (int64_t)c * sc + pix);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          e[2 * k] = (uint16_t)(w[k] & 0xFFFF);
          e[2 * k + 1] = (uint16_t)(w[k] >> 16);
        }
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          e[k] = (c < C && pix + k < HW) ? src[(int64_t)c * sc + pix + k] : (uint16_t)0;
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) tile[(pb * 8 + k) * PITCH + cw] = a[k] | ((uint32_t)b[k] << 16);
  }
  __syncthreads();
  uint16_t* dst = reinterpret_cast<uint16_t*>(out) + (int64_t)n * HW * C8;
  for (int i = threadIdx.x; i < TP * 8; i += blockDim.x) {
    const int pp = i >> 3, q = i & 7;             // pixel, group of 8 channels
    const int c = c0 + q * 8, pix = p0 + pp;
    if (pix >= HW || c >= C8) continue;
    const uint4 v = *reinterpret_cast<const uint4*>(&tile[pp * PITCH + q * 4]);
    *reinterpret_cast<uint4*>(dst + (int64_t)pix * C8 + c) = v;
  }
}


// Epilogue store of one 32 (output channels) x 32 (virtual pixels) block that
// sits transposed in shared memory (xp[channel * 33 + pixel]): lane = pixel,
// so every store instruction writes 32 consecutive outputs of one channel
// (consecutive virtual pixels are consecutive in NCHW memory except across
// the discarded W - Q columns).  Branch-free: the per-lane validity is a
// predicate, the channel bound is warp-uniform.
template <bool BF16>
__device__ __forceinline__ void store_chunk_rows(const float* xp, int lane, char* ybase, int m,
                                                 int W, int PW, int Q, int k0, int K,
                                                 const int64_t* ys) {
  using T = typename std::conditional<BF16, __nv_bfloat16, __half>::type;
  const int pp = m / W, q = m - pp * W;
  const bool ok = m < PW && q < Q;
  T* yp = reinterpret_cast<T*>(ybase) + (int64_t)k0 * ys[1] + (int64_t)pp * ys[2] +
          (int64_t)q * ys[3];
  const int64_t kst = ys[1];
  const int kn = K - k0;
  if (kn >= 32) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float f = xp[j * 33 + lane];
      if (ok) yp[j * kst] = BF16 ? T(__float2bfloat16_rn(f)) : T(__float2half_rn(f));
    }
  } else {
    for (int j = 0; j < kn; ++j) {
      const float f = xp[j * 33 + lane];
      if (ok) yp[j * kst] = BF16 ? T(__float2bfloat16_rn(f)) : T(__float2half_rn(f));
    }
  }
}

template <bool BF16>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    conv_pair_kernel(const __grid_constant__ ConvMaps maps, const ConvParams p) {
  using namespace sm100;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  // static (not carved from the dynamic buffer) so the compiler keeps the
  // shared address space: LDS/STS instead of generic LD/ST + MEMBARs
  __shared__ float xpose[4 * XPOSE_FLOATS];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int RS = p.R * p.S;
  const int nk = RS * p.cb;
  const int tiles_img = p.pix_tiles * p.k_tiles;
  const int total = tiles_img * p.N;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 8);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&maps.w);
    tma_prefetch(&maps.x);
  }
  if (warp == 2) {
    tmem_alloc_pair(&tmem_slot, TMEM_COLS);
    tc_fence_before();
  }
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      int st = 0;
      uint32_t ph = 0;
      for (int t = cid; t < total; t += ncl) {
        const int n = t / tiles_img, rr = t % tiles_img;
        const int pt = rr / p.k_tiles, kt = rr % p.k_tiles;
        const int krow = kt * 256 + (int)rank * 128;
        const int pix = pt * 256 + (int)rank * 128;
        for (int kb = 0; kb < nk; ++kb) {
          const int rs = kb / p.cb, cbk = kb % p.cb;
          const int shift = (rs / p.S) * p.W + (rs % p.S);
          mbar_wait(&empty[st], ph ^ 1);
          if (rank == 0) mbar_expect_tx(&full[st], 2 * STAGE_BYTES);
          const uint32_t bar = leader_addr(&full[st]);
          tma_load_3d_pair(sA + st * A_BYTES, &maps.w, bar, cbk * BK, rs, krow);
          tma_load_3d_pair(sB + st * B_BYTES, &maps.x, bar, cbk * BK, pix + shift, n);
          if (++st == STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && elect_one()) {
      constexpr uint32_t idesc = idesc_f16(BF16, false, false, 256, 256);
      int st = 0;
      uint32_t ph = 0;
      int tl = 0;
      for (int t = cid; t < total; t += ncl, ++tl) {
        const int acc = tl & 1;
        const uint32_t aph = (tl >> 1) & 1;
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[st], ph);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + st * A_BYTES);
          const uint32_t b_addr = smem_u32(sB + st * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = umma_desc_sw128(a_addr + k * 32, 16, 1024);
            const uint64_t bd = umma_desc_sw128(b_addr + k * 32, 16, 1024);
            mma_f16_ss_pair(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          mma_commit_pair(&empty[st]);
          if (++st == STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
        mma_commit_pair(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    float* xp = xpose + ew * XPOSE_FLOATS;

    int tl = 0;
    for (int t = cid; t < total; t += ncl, ++tl) {
      const int n = t / tiles_img, rr = t % tiles_img;
      const int pt = rr / p.k_tiles, kt = rr % p.k_tiles;
      const int acc = tl & 1;
      const uint32_t aph = (tl >> 1) & 1;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const int k0 = kt * 256 + (int)rank * 128 + ew * 32;  // this warp's 32 output channels
      const uint32_t taddr = tmem_base + acc * 256 + ((uint32_t)(ew * 32) << 16);
      char* ybase = reinterpret_cast<char*>(p.y) + (int64_t)n * p.ys[0] * 2;
#pragma unroll 1
      for (int cc = 0; cc < 8; ++cc) {
        uint32_t v[32];
        __syncwarp();
        tmem_ld_32x32b_x32(taddr + cc * 32, v);
        tmem_ld_wait();
        // lane = output channel row; transpose so lanes run along pixels
#pragma unroll
        for (int i = 0; i < 32; ++i) xp[lane * 33 + i] = __uint_as_float(v[i]);
        __syncwarp();
        const int m = pt * 256 + cc * 32 + lane;
        store_chunk_rows<BF16>(xp, lane, ybase, m, p.W, p.P * p.W, p.Q, k0, p.K, p.ys);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_addr(&tempty[acc]));
    }
  }
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, TMEM_COLS);
  }
}

template <bool BF16>
int launch_conv(const ConvMaps& maps, const ConvParams& p, cudaStream_t s) {
  auto k = conv_pair_kernel<BF16>;
  static size_t attr[kMaxDevices] = {};
  cudaError_t e = smem_attr_once(k, SMEM_BYTES, attr);
  if (e != cudaSuccess) return cuda_fail(e, "conv smem attribute");
  const int total = p.N * p.pix_tiles * p.k_tiles;
  int clusters = sm_count() / 2;
  if (total < clusters) clusters = total;
  k<<<2 * clusters, 256, SMEM_BYTES, s>>>(maps, p);
  return check_launch("conv2d tcgen05 pair", NTB_PATH_CONV_TC);
}


// ---- fused NCHW implicit GEMM: no transpose pass --------------------------
// The image operand of a (pixel tile, 64-channel block) is staged ONCE per
// CTA as a K-major 128B-swizzled "window" of rows = pixels [q0, q0 + 128 +
// (R-1)W + (S-1)) x 64 channels, filled straight from the NCHW tensor by
// four producer warps (coalesced 16-pixel loads per channel pair, packed to
// channel pairs, conflict-free 32-bit stores at the swizzled position of the
// absolute smem address).  The R*S shifted operands are then just UMMA
// descriptors whose start address moves by (r*W + s) rows of 128 B: the
// hardware applies the 128B swizzle on absolute address bits (measured:
// tools/ubench/desc_offset.cu, base_offset = 0 is exact at every row offset),
// so no data is moved per (r, s).  The filter still streams through a TMA
// ring (W'[k_out][(r,s)][C8], one 16 KB stage per (r, s, channel block)).
constexpr int kFusedThreads = 384;
#ifndef NTB_CONV_TRACE
#define NTB_CONV_TRACE 0
#endif
#if NTB_CONV_TRACE
__device__ long long g_conv_trace[4096];
#endif   // w0 TMA(W') w1 MMA w2 TMEM w3 - w4-7 epilogue w8-11 window

struct FusedParams {
  int N, C, H, W, K, R, S, P, Q;
  int cb, pix_tiles, k_tiles;
  int win_rows, stages;
  int n_whole, n_split;   // whole tiles, then 2 x n_split half-width tail units
  const void* x;
  int64_t xs0, xs1;   // batch / channel strides (elements); planes are contiguous H*W runs
  int vec;            // 16-byte image loads allowed
  void* y;
  int64_t ys[4];
};

__device__ __forceinline__ void mbar_arrive_cluster_rel(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n}" ::"r"(sm100::smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <bool BF16, int TN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kFusedThreads, 1)
    conv_fused_kernel(const __grid_constant__ CUtensorMap wmap, const FusedParams p) {
  using namespace sm100;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int WIN_BYTES = p.win_rows * 128;
  uint8_t* sA = smem;
  uint8_t* sWin = smem + p.stages * A_BYTES;
  __shared__ float xpose[4 * XPOSE_FLOATS];
  __shared__ __align__(8) uint64_t full[FSTAGES], empty[FSTAGES], tfull[2], tempty[2], wfull[2],
      wempty[2];
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int RS = p.R * p.S;
  const int tiles_img = p.pix_tiles * p.k_tiles;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  // work units: whole tiles (TN pixels), then the two TN/2-pixel halves of
  // each tail tile (N = TN/2 MMAs) so the last wave keeps every pair busy
  const int total = p.n_whole + 2 * p.n_split;
  struct Unit { int n, pt, kt, pix0, npix; };
  auto decode = [&](int u) {
    Unit w;
    int t = u, off = 0, np = TN;
    if (u >= p.n_whole) {
      const int s2 = u - p.n_whole;
      t = p.n_whole + (s2 >> 1);
      off = (s2 & 1) * (TN / 2);
      np = TN / 2;
    }
    w.n = t / tiles_img;
    const int rr = t % tiles_img;
    w.pt = rr / p.k_tiles;
    w.kt = rr % p.k_tiles;
    w.pix0 = w.pt * TN + off;
    w.npix = np;
    return w;
  };
  const int stages = p.stages;

  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 8);
      mbar_init(&wfull[i], 2);   // one publisher arrival per CTA (on CTA 0)
      mbar_init(&wempty[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) tma_prefetch(&wmap);
  if (warp == 2) {
    tmem_alloc_pair(&tmem_slot, TMEM_COLS);
    tc_fence_before();
  }
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = tmem_slot;
#if !NTB_CONV_NO_PDL
  // programmatic launch (as in the GEMM): the first filter stages go to L2
  // before waiting for the previous kernel
  if (warp == 0 && lane == 0 && cid < total) {
    const int krow = decode(cid).kt * 256 + (int)rank * 128;
    int n = 0;
    for (int cbk = 0; cbk < p.cb && n < stages; ++cbk)
      for (int rs = 0; rs < RS && n < stages; ++rs, ++n) tma_prefetch_3d(&wmap, cbk * BK, rs, krow);
  }
  pdl_wait();
  pdl_trigger();
#endif

  if (warp == 0) {
    if (elect_one()) {
      int st = 0;
      uint32_t ph = 0;
      for (int t = cid; t < total; t += ncl) {
        const int kt = decode(t).kt;
        const int krow = kt * 256 + (int)rank * 128;
        for (int cbk = 0; cbk < p.cb; ++cbk)
          for (int rs = 0; rs < RS; ++rs) {
            mbar_wait(&empty[st], ph ^ 1);
            if (rank == 0) mbar_expect_tx(&full[st], 2 * A_BYTES);
            tma_load_3d_pair(sA + st * A_BYTES, &wmap, leader_addr(&full[st]), cbk * BK, rs, krow);
            if (++st == stages) {
              st = 0;
              ph ^= 1;
            }
          }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && elect_one()) {
      constexpr uint32_t idesc_w = idesc_f16(BF16, false, false, 256, TN);
      constexpr uint32_t idesc_h = idesc_f16(BF16, false, false, 256, TN / 2);
      int st = 0;
      uint32_t ph = 0;
      int tl = 0, wc = 0;
      for (int t = cid; t < total; t += ncl, ++tl) {
        const uint32_t idesc = decode(t).npix == TN ? idesc_w : idesc_h;
        const int acc = tl & 1;
        mbar_wait(&tempty[acc], ((tl >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * TN;
        for (int cbk = 0; cbk < p.cb; ++cbk, ++wc) {
          const int wb = wc & 1;
#if NTB_CONV_TRACE
          const bool tr = blockIdx.x == 0 && tl < 3;
          if (tr) g_conv_trace[(tl * 8 + cbk) * 64 + 0] = clock64();
#endif
          mbar_wait_cluster(&wfull[wb], (wc >> 1) & 1);
          tc_fence_after();
#if NTB_CONV_TRACE
          if (tr) g_conv_trace[(tl * 8 + cbk) * 64 + 1] = clock64();
#endif
          const uint32_t win = smem_u32(sWin + wb * WIN_BYTES);
          for (int rs = 0; rs < RS; ++rs) {
#if NTB_CONV_TRACE
            if (tr) g_conv_trace[(tl * 8 + cbk) * 64 + 2 + 2 * rs] = clock64();
#endif
            mbar_wait(&full[st], ph);
            tc_fence_after();
#if NTB_CONV_TRACE
            if (tr) g_conv_trace[(tl * 8 + cbk) * 64 + 3 + 2 * rs] = clock64();
#endif
            const uint32_t a_addr = smem_u32(sA + st * A_BYTES);
            const uint32_t b_addr = win + (uint32_t)((rs / p.S) * p.W + (rs % p.S)) * 128u;
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              mma_f16_ss_pair(d_tmem, umma_desc_sw128(a_addr + k * 32, 16, 1024),
                              umma_desc_sw128(b_addr + k * 32, 16, 1024), idesc,
                              (cbk | rs | k) != 0);
            mma_commit_pair(&empty[st]);
            if (++st == stages) {
              st = 0;
              ph ^= 1;
            }
          }
          mma_commit_pair(&wempty[wb]);
        }
        mma_commit_pair(&tfull[acc]);
      }
    }
  } else if (warp == 3) {
    // window publisher: waits for the 4 producer warps of this CTA, then one
    // cluster-scope release-arrive on CTA 0's window barrier
    int wc = 0;
    for (int t = cid; t < total; t += ncl)
      for (int cbk = 0; cbk < p.cb; ++cbk, ++wc) {
        asm volatile("bar.sync %0, 160;" ::"r"(1 + (wc & 1)) : "memory");
        if (lane == 0) mbar_arrive_cluster_rel(leader_addr(&wfull[wc & 1]));
      }
  } else if (warp >= 8) {
    // window producers: lane = channel pair, warp = 16-pixel groups.  The
    // first chunk (<= 4 groups per warp) of the NEXT window is loaded into
    // registers while the MMA still consumes the current one, so the global
    // latency is off the critical path; only the stores wait for the buffer.
    const int pw = warp - 8;
    const int HW = p.H * p.W;
    const int halo = (p.R - 1) * p.W + (p.S - 1);
    const uint16_t* xb = reinterpret_cast<const uint16_t*>(p.x);
    uint4 v[4][4];
    auto load_chunk = [&](int t, int cbk, int g0) {
      const Unit w = decode(t);
      const int n = w.n;
      const int q0 = w.pix0 + (int)rank * (w.npix / 2);
      const int groups = (w.npix / 2 + halo + 15) / 16;
      const int c = cbk * BK + 2 * lane;
      const bool c0ok = c < p.C, c1ok = c + 1 < p.C;
      const uint16_t* src0 = xb + (int64_t)n * p.xs0 + (int64_t)c * p.xs1;
      const uint16_t* src1 = src0 + p.xs1;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int g = g0 + 4 * u;
        const int pix = q0 + g * 16;
        if (g < groups && p.vec && pix + 16 <= HW) {
          const uint4 z = make_uint4(0, 0, 0, 0);
          v[u][0] = c0ok ? ld_keep(src0 + pix) : z;
          v[u][1] = c0ok ? ld_keep(src0 + pix + 8) : z;
          v[u][2] = c1ok ? ld_keep(src1 + pix) : z;
          v[u][3] = c1ok ? ld_keep(src1 + pix + 8) : z;
        } else {
          uint32_t w0[8], w1[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const bool in0 = g < groups && pix + 2 * i < HW, in1 = g < groups && pix + 2 * i + 1 < HW;
            w0[i] = (in0 && c0ok ? src0[pix + 2 * i] : 0u) |
                    ((uint32_t)(in1 && c0ok ? src0[pix + 2 * i + 1] : 0u) << 16);
            w1[i] = (in0 && c1ok ? src1[pix + 2 * i] : 0u) |
                    ((uint32_t)(in1 && c1ok ? src1[pix + 2 * i + 1] : 0u) << 16);
          }
          v[u][0] = make_uint4(w0[0], w0[1], w0[2], w0[3]);
          v[u][1] = make_uint4(w0[4], w0[5], w0[6], w0[7]);
          v[u][2] = make_uint4(w1[0], w1[1], w1[2], w1[3]);
          v[u][3] = make_uint4(w1[4], w1[5], w1[6], w1[7]);
        }
      }
    };
    auto store_chunk = [&](uint32_t win_a, int g0, int groups) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int g = g0 + 4 * u;
        if (g >= groups) break;
        const uint32_t w0[8] = {v[u][0].x, v[u][0].y, v[u][0].z, v[u][0].w,
                                v[u][1].x, v[u][1].y, v[u][1].z, v[u][1].w};
        const uint32_t w1[8] = {v[u][2].x, v[u][2].y, v[u][2].z, v[u][2].w,
                                v[u][3].x, v[u][3].y, v[u][3].z, v[u][3].w};
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          // (channel c, channel c+1) of pixel i as one 32-bit word
          const uint32_t word = (i & 1) ? __byte_perm(w0[i >> 1], w1[i >> 1], 0x7632)
                                        : __byte_perm(w0[i >> 1], w1[i >> 1], 0x5410);
          const int row = g * 16 + i;
          const uint32_t addr = win_a + row * 128 + (((lane >> 2) ^ (row & 7)) << 4) +
                                ((lane & 3) << 2);
          asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(word) : "memory");
        }
      }
    };
    int wc = 0;
    if (cid < total) load_chunk(cid, 0, pw);
    for (int t = cid; t < total; t += ncl) {
      for (int cbk = 0; cbk < p.cb; ++cbk, ++wc) {
        const int wb = wc & 1;
#if NTB_CONV_TRACE
        const bool trp = blockIdx.x == 0 && pw == 0 && lane == 0 && wc < 12;
        if (trp) g_conv_trace[3200 + wc * 8 + 0] = clock64();
#endif
        mbar_wait(&wempty[wb], ((wc >> 1) & 1) ^ 1);
#if NTB_CONV_TRACE
        if (trp) g_conv_trace[3200 + wc * 8 + 1] = clock64();
#endif
        const uint32_t win_a = smem_u32(sWin + wb * WIN_BYTES);
        const int groups = (decode(t).npix / 2 + halo + 15) / 16;
        for (int g0 = pw; g0 < groups; g0 += 16) {
          if (g0 != pw) load_chunk(t, cbk, g0);
          store_chunk(win_a, g0, groups);
        }
#if NTB_CONV_TRACE
        if (trp) g_conv_trace[3200 + wc * 8 + 2] = clock64();
#endif
        // hand the window to the publisher warp (named barrier 1 / 2 by
        // window parity): the cluster-scope release it needs costs ~1k
        // cycles and must not stall the next window's loads
        fence_proxy_async();
        asm volatile("bar.arrive %0, 160;" ::"r"(1 + (wc & 1)) : "memory");
#if NTB_CONV_TRACE
        if (trp) g_conv_trace[3200 + wc * 8 + 3] = clock64();
#endif
        // prefetch the first chunk of the next window
        if (cbk + 1 < p.cb) load_chunk(t, cbk + 1, pw);
        else if (t + ncl < total) load_chunk(t + ncl, 0, pw);
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    float* xp = xpose + ew * XPOSE_FLOATS;

    int tl = 0;
    for (int t = cid; t < total; t += ncl, ++tl) {
      const Unit w = decode(t);
      const int n = w.n, kt = w.kt;
      const int acc = tl & 1;
#if NTB_CONV_TRACE
      const bool tr = blockIdx.x == 0 && tl < 3 && ew == 0 && lane == 0;
      if (tr) g_conv_trace[3000 + tl * 4] = clock64();
#endif
      mbar_wait(&tfull[acc], (tl >> 1) & 1);
      tc_fence_after();
#if NTB_CONV_TRACE
      if (tr) g_conv_trace[3000 + tl * 4 + 1] = clock64();
#endif
      const int k0 = kt * 256 + (int)rank * 128 + ew * 32;
      const uint32_t taddr = tmem_base + acc * TN + ((uint32_t)(ew * 32) << 16);
      char* ybase = reinterpret_cast<char*>(p.y) + (int64_t)n * p.ys[0] * 2;
#pragma unroll 1
      for (int cc = 0; cc < w.npix / 32; ++cc) {
        uint32_t v[32];
        __syncwarp();
        tmem_ld_32x32b_x32(taddr + cc * 32, v);
        tmem_ld_wait();
#if NTB_CONV_TRACE
        if (tr && tl == 1) g_conv_trace[3100 + cc * 4] = clock64();
#endif
#pragma unroll
        for (int i = 0; i < 32; ++i) xp[lane * 33 + i] = __uint_as_float(v[i]);
        __syncwarp();
#if NTB_CONV_TRACE
        if (tr && tl == 1) g_conv_trace[3100 + cc * 4 + 1] = clock64();
#endif
        const int m = w.pix0 + cc * 32 + lane;
        store_chunk_rows<BF16>(xp, lane, ybase, m, p.W, p.P * p.W, p.Q, k0, p.K, p.ys);
#if NTB_CONV_TRACE
        if (tr && tl == 1) g_conv_trace[3100 + cc * 4 + 2] = clock64();
#endif
      }
      tc_fence_before();
      __syncwarp();
#if NTB_CONV_TRACE
      if (tr) g_conv_trace[3000 + tl * 4 + 2] = clock64();
#endif
      if (lane == 0) mbar_arrive_cluster(leader_addr(&tempty[acc]));
    }
  }
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, TMEM_COLS);
  }
}

template <bool BF16, int TN>
int launch_conv_fused(const CUtensorMap& wmap, const FusedParams& p, size_t smem, cudaStream_t s) {
  auto k = conv_fused_kernel<BF16, TN>;
  static size_t attr[kMaxDevices] = {};
  cudaError_t e = smem_attr_once(k, smem, attr);
  if (e != cudaSuccess) return cuda_fail(e, "conv fused smem attribute");
  const int total = p.N * p.pix_tiles * p.k_tiles;
  int clusters = sm_count() / 2;
  if (total < clusters) clusters = total;
#if NTB_CONV_NO_PDL
  k<<<2 * clusters, kFusedThreads, smem, s>>>(wmap, p);
#else
  launch_pdl(k, dim3(2 * clusters), dim3(kFusedThreads), smem, s, wmap, p);
#endif
#if NTB_CONV_TRACE
  {
    static long long h[4096];
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(h, g_conv_trace, sizeof(h));
    const long long t0 = h[0];
    for (int tl = 0; tl < 3; ++tl)
      for (int cb = 0; cb < p.cb; ++cb) {
        const long long* r = h + (tl * 8 + cb) * 64;
        fprintf(stderr, "tile %d cb %d: @%7lld win-wait %5lld |", tl, cb, r[0] - t0, r[1] - r[0]);
        for (int rs = 0; rs < p.R * p.S; ++rs)
          fprintf(stderr, " %4lld/%4lld", r[3 + 2 * rs] - r[2 + 2 * rs],
                  (rs + 1 < p.R * p.S ? r[4 + 2 * rs] : r[3 + 2 * rs]) - r[3 + 2 * rs]);
        fprintf(stderr, "\n");
      }
    for (int tl = 0; tl < 3; ++tl)
      fprintf(stderr, "epilogue tile %d: wait@%lld got@%lld done@%lld\n", tl, h[3000 + tl * 4] - t0,
              h[3000 + tl * 4 + 1] - t0, h[3000 + tl * 4 + 2] - t0);
    for (int w = 0; w < 12; ++w) {
      const long long* r = h + 3200 + w * 8;
      fprintf(stderr, "producer window %2d: start@%6lld wempty-wait %5lld stores %5lld arrive %5lld\n", w,
              r[0] - t0, r[1] - r[0], r[2] - r[1], r[3] - r[2]);
    }
    for (int cc = 0; cc < 8; ++cc)
      fprintf(stderr, "  tile1 chunk %d: ld@%lld xpose %lld stores %lld\n", cc, h[3100 + cc * 4] - t0,
              h[3100 + cc * 4 + 1] - h[3100 + cc * 4], h[3100 + cc * 4 + 2] - h[3100 + cc * 4 + 1]);
  }
#endif
  return check_launch("conv2d tcgen05 fused", NTB_PATH_CONV_TC);
}
}  // namespace

int conv_sm100(const ConvDesc& c, int dtype, cudaStream_t s) {
  if (c.N >= 65536 || c.K >= (1 << 30) || (int64_t)c.H * c.W >= (1ll << 31) || c.C >= (1 << 30))
    return NTB_ERR_UNSUPPORTED;
  const bool bf16 = dtype == NTB_BF16;
  const CUtensorMapDataType dt = bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  const int64_t HW = c.H * c.W;
  // channels_last input already is [N][H][W][C]: use it in place
  const bool nhwc = c.xs[1] == 1 && c.xs[3] == c.C && c.xs[2] == c.W * c.C &&
                    (c.N == 1 || c.xs[0] == HW * c.C) && c.C % 8 == 0 && aligned16(c.x);
  const int64_t C8 = nhwc ? c.C : (c.C + 7) / 8 * 8;
  const int64_t RS = c.R * c.S;
  const size_t wbytes = ((size_t)c.K * RS * C8 * 2 + 255) / 256 * 256;
  const size_t xbytes = nhwc ? 0 : (size_t)c.N * HW * C8 * 2;
  char* ws = (char*)workspace(wbytes + xbytes, s);
  if (!ws) return fail(NTB_ERR_CUDA, "conv2d: workspace allocation failed");
  void* wp = ws;
  const void* xp = nhwc ? c.x : (const void*)(ws + wbytes);
  const int sms = sm_count();
  {
    int64_t total = c.K * RS * C8;
    int blocks = (int)cdiv64(total, 256);
    if (blocks > sms * 8) blocks = sms * 8;
    if (bf16)
      repack_filter<__nv_bfloat16><<<blocks, 256, 0, s>>>(
          (const __nv_bfloat16*)c.w, c.ws[0], c.ws[1], c.ws[2], c.ws[3], (__nv_bfloat16*)wp,
          (int)c.K, (int)c.C, (int)C8, (int)c.R, (int)c.S);
    else
      repack_filter<__half><<<blocks, 256, 0, s>>>((const __half*)c.w, c.ws[0], c.ws[1], c.ws[2],
                                                   c.ws[3], (__half*)wp, (int)c.K, (int)c.C,
                                                   (int)C8, (int)c.R, (int)c.S);
    int rc = check_launch("conv2d filter repack", NTB_PATH_REPACK);
    if (rc) return rc;
  }
  if (!nhwc && c.xs[3] == 1 && c.xs[2] == c.W) {
    // fused path: the image window is staged from NCHW inside the kernel.
    // Pixel tile per CTA pair: 256.  (192 fits the BASELINE shape's waves
    // better - 13.8 instead of 10.4 waves over 74 CTA pairs - but measured
    // 197 us vs 182 us: the per-tile window fill and epilogue dominate;
    // NTB_CONV_TN=192 selects it for experiments.)
    static const char* tn_env = getenv("NTB_CONV_TN");
    const int TN = tn_env && atoi(tn_env) == 192 ? 192 : 256;
    const int64_t win_rows = ((TN / 2 + (c.R - 1) * c.W + (c.S - 1)) + 15) / 16 * 16;
    const size_t budget = 227 * 1024 - sizeof(float) * 4 * XPOSE_FLOATS - 512 - 1024;
    const size_t win_bytes = (size_t)win_rows * 128;
    int stages = FSTAGES;
    while (stages >= 3 && (size_t)stages * A_BYTES + 2 * win_bytes > budget) --stages;
    if (stages >= 3 && !getenv("NTB_CONV_UNFUSED")) {
      CUtensorMap wmap;
      uint64_t dims[3] = {(uint64_t)C8, (uint64_t)RS, (uint64_t)c.K};
      uint64_t str[2] = {(uint64_t)C8 * 2, (uint64_t)(RS * C8 * 2)};
      uint32_t box[3] = {64, 1, 128};
      if (!encode_tmap(&wmap, dt, 3, wp, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B))
        return fail(NTB_ERR_UNSUPPORTED, "conv2d: filter tensor map");
      FusedParams f;
      f.N = (int)c.N; f.C = (int)c.C; f.H = (int)c.H; f.W = (int)c.W; f.K = (int)c.K;
      f.R = (int)c.R; f.S = (int)c.S; f.P = (int)c.P; f.Q = (int)c.Q;
      f.cb = (int)cdiv64(c.C, BK);
      f.pix_tiles = (int)cdiv64((int64_t)c.P * c.W, TN);
      f.k_tiles = (int)cdiv64(c.K, 256);
      f.win_rows = (int)win_rows;
      {
        // narrow tail (as in the GEMM): last-wave tiles split into two
        // half-width units when more than half the CTA pairs would idle
        const int64_t total = (int64_t)c.N * f.pix_tiles * f.k_tiles;
        const int64_t pairs = sm_count() / 2;
        const int64_t rem = total % pairs;
        static const bool split = !getenv("NTB_CONV_NO_SPLIT");
        f.n_split = (split && total > pairs && rem > 0 && 2 * rem <= pairs) ? (int)rem : 0;
        f.n_whole = (int)(total - f.n_split);
      }
      f.stages = stages;
      f.x = c.x;
      f.xs0 = c.xs[0];
      f.xs1 = c.xs[1];
      f.vec = aligned16(c.x) && c.xs[0] % 8 == 0 && c.xs[1] % 8 == 0 && HW % 8 == 0;
      f.y = c.y;
      for (int d = 0; d < 4; ++d) f.ys[d] = c.ys[d];
      const size_t smem = (size_t)stages * A_BYTES + 2 * win_bytes + 1024;
      if (TN == 192)
        return bf16 ? launch_conv_fused<true, 192>(wmap, f, smem, s)
                    : launch_conv_fused<false, 192>(wmap, f, smem, s);
      return bf16 ? launch_conv_fused<true, 256>(wmap, f, smem, s)
                  : launch_conv_fused<false, 256>(wmap, f, smem, s);
    }
  }
  if (!nhwc) {
    // NCHW planes must be contiguous H*W runs for the transpose
    if (c.xs[3] != 1 || c.xs[2] != c.W) return NTB_ERR_UNSUPPORTED;
    dim3 grid((unsigned)cdiv64(HW, 64), (unsigned)cdiv64(C8, 64), (unsigned)c.N);
    if (bf16)
      nchw_to_nhwc<__nv_bfloat16><<<grid, 256, 0, s>>>((const __nv_bfloat16*)c.x, c.xs[0], c.xs[1],
                                                      (__nv_bfloat16*)xp, (int)c.C, (int)C8,
                                                      (int)HW);
    else
      nchw_to_nhwc<__half><<<grid, 256, 0, s>>>((const __half*)c.x, c.xs[0], c.xs[1], (__half*)xp,
                                               (int)c.C, (int)C8, (int)HW);
    int rc = check_launch("conv2d NCHW->NHWC", NTB_PATH_REPACK);
    if (rc) return rc;
  }
  ConvMaps maps;
  {
    uint64_t dims[3] = {(uint64_t)C8, (uint64_t)RS, (uint64_t)c.K};
    uint64_t str[2] = {(uint64_t)C8 * 2, (uint64_t)(RS * C8 * 2)};
    uint32_t box[3] = {64, 1, 128};
    if (!encode_tmap(&maps.w, dt, 3, wp, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return fail(NTB_ERR_UNSUPPORTED, "conv2d: filter tensor map");
  }
  {
    uint64_t dims[3] = {(uint64_t)C8, (uint64_t)HW, (uint64_t)c.N};
    uint64_t str[2] = {(uint64_t)C8 * 2, (uint64_t)(HW * C8 * 2)};
    uint32_t box[3] = {64, 128, 1};
    if (!encode_tmap(&maps.x, dt, 3, xp, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return fail(NTB_ERR_UNSUPPORTED, "conv2d: image tensor map");
  }
  ConvParams p;
  p.N = (int)c.N; p.C = (int)c.C; p.H = (int)c.H; p.W = (int)c.W; p.K = (int)c.K;
  p.R = (int)c.R; p.S = (int)c.S; p.P = (int)c.P; p.Q = (int)c.Q;
  p.cb = (int)cdiv64(c.C, BK);
  p.pix_tiles = (int)cdiv64((int64_t)c.P * c.W, 256);
  p.k_tiles = (int)cdiv64(c.K, 256);
  p.y = c.y;
  for (int d = 0; d < 4; ++d) p.ys[d] = c.ys[d];
  return bf16 ? launch_conv<true>(maps, p, s) : launch_conv<false>(maps, p, s);
}

}  // namespace ntb
