// fp32 mm / bmm / addmm on the sm_100a tensor cores (reference catalog.py:
// 82-118, 226-292: every catalog parameter is f32; the reference computes Dot
// in f64 and rounds to f32, sim.py:317-320).
//
// 3xTF32: tcgen05.mma kind::tf32 reads 32-bit operands from shared memory and
// TRUNCATES them to tf32 (10 explicit mantissa bits; measured,
// tools/ubench/tf32_round.cu, profiles/r2_tf32_round_ubench.txt).  With
// lo = a - trunc(a) (exact in fp32) the product a*b is recovered to ~2^-21
// relative by three MMAs into one fp32 accumulator:
//     acc += A*B + A*B_lo + A_lo*B        (A, B as loaded: the hardware sees hi)
// (the dropped A_lo*B_lo term is below 2^-20 of |a*b|).
//
// Layout (CTA pair, cta_group::2, 256 x 256 output tiles as in the fp16 pair
// kernel, k_gemm_sm100.cu), 384 threads:
//   * warp 0: TMA producer, this CTA's 128 rows of A and 128 rows of B per
//     32-wide K block (128-byte fp32 rows; K-major SWIZZLE_128B, MN-major
//     SWIZZLE_128B_ATOM_32B, the only MN-major layout tf32 UMMA reads) into a
//     3-stage ring; each CTA's bytes complete on its OWN barrier;
//   * warps 2-3: lo converters - read the stage's raw A and B tiles and write
//     lo = a - trunc(a) into the stage's A_lo / B_lo tiles (same swizzled
//     offsets: the split is element-wise, so the layout is copied as is).
//     CTA 0's converters arrive on CTA 0's "stage ready" barrier directly;
//     CTA 1's hand over to warp 1 of CTA 1 (named barrier per stage), which
//     does the one cluster-scope release-arrive (~1k cycles, off their path);
//   * warp 1 of CTA 0: issues 12 tcgen05.mma.cta_group::2.kind::tf32
//     (M = 256, N = 256, K = 8) per K block; K runs in chunks of
//     NTB_TF32_CHUNK blocks, each accumulated from zero in one of the two
//     256-column TMEM buffers (alternating);
//   * warps 4-11: epilogue - each thread drains its row's 128 columns of every
//     chunk into fp32 registers (round-to-nearest adds: the tensor core's own
//     accumulation rounds toward zero and drifts over long K), then
//     alpha * acc + beta * addend, 128B-swizzled staging, TMA store.
// Tensor roofline: 2*M*N*K useful flop per launch (3 MMAs issued per product).
#include <stdlib.h>

#include "common.cuh"
#include "k_sm100.cuh"
#include "sm100_ptx.cuh"

namespace ntb {
namespace {

constexpr int TBK = 32;                              // fp32 K elements per 128-byte row
constexpr int T_TILE = 128 * TBK * 4;                // 16 KB: 128 rows x 32 K
constexpr int T_STAGE = 4 * T_TILE;                  // A | B | A_lo | B_lo
constexpr int T_STAGES = 3;
constexpr int T_STAGE_C = 8 * 32 * 128;              // 8 epilogue warps x (32 rows x 32 fp32)
constexpr int T_SMEM = T_STAGES * T_STAGE + T_STAGE_C + 1024;
constexpr int T_THREADS = 384;
#ifndef NTB_TF32_REGSPLIT
#define NTB_TF32_REGSPLIT 1  // 0: no setmaxnreg (A/B: the epilogue then spills; ~2% slower)
#endif
// registers to the epilogue warps (128 fp32 partial sums per thread):
// 72 x 128 + 216 x 256 = the launch pool of 168 x 384
#if NTB_TF32_REGSPLIT
#ifndef NTB_TF32_REG_LO
#define NTB_TF32_REG_LO 72
#endif
#define NTB_TF32_REG_HI ((168 * 384 - NTB_TF32_REG_LO * 128) / 256 / 8 * 8)
#define TF32_REG_DEC asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(NTB_TF32_REG_LO));
#define TF32_REG_INC asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(NTB_TF32_REG_HI));
#else
#define TF32_REG_DEC
#define TF32_REG_INC
#endif
#ifndef NTB_TF32_CHUNK
#define NTB_TF32_CHUNK 4   // K blocks (x 32) accumulated in TMEM before the epilogue drains them
#endif
constexpr int T_CHUNK = NTB_TF32_CHUNK;
constexpr int T_TMEM_COLS = 512;

struct TMaps {
  CUtensorMap a, b, c;
};

struct TParams {
  int M, N, K, batch, num_m, num_n;   // num_m / num_n: 256-row / 256-column tiles
  const float* d;
  int64_t d_m, d_n, d_sm, d_sn;
  float alpha, beta;
  int has_d;
  int passes;   // 3 (default); 1 = plain TF32 (NTB_TF32_PASSES=1, A/B only)
  // conv2d (implicit GEMM, CONV = true): A = filter W'[k][(r,s)][c4],
  // B = image X'[n][pixel][c4]; `batch` = N images, tiles of 256 output
  // channels x 256 virtual pixels (row width W, the W - Q tail discarded)
  int cb, pix_tiles, k_tiles, S, W, PW, Q, RS;
  float* y;
  int64_t ys[4];
  // narrow tail (as the fp16 pair GEMM): units [n_whole, n_whole + 2 n_split)
  // are the two 128-column halves of the last n_split tiles (N = 128 MMAs)
  int n_whole, n_split;
};

__host__ __device__ constexpr uint32_t idesc_tf32(bool a_mn, bool b_mn, int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void arrive_cluster_release(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
__device__ __forceinline__ void wait_cluster_acquire(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITT_%=;\n}" ::"r"(sm100::smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// lo = a - trunc_tf32(a), exact; 0 for inf / nan (the hi term carries them)
__device__ __forceinline__ uint32_t tf32_lo(uint32_t u) {
  const float a = __uint_as_float(u);
  const float lo = a - __uint_as_float(u & 0xFFFFE000u);
  return (u & 0x7F800000u) == 0x7F800000u ? 0u : __float_as_uint(lo);
}

// UMMA descriptor of the K-step k (8 fp32) of a 128-row x 32-K tile.
//   K-major : SWIZZLE_128B, 128-byte rows, the step is 32 bytes along the
//             swizzled row (16-byte units XOR row % 8).
//   MN-major: tf32 needs SWIZZLE_128B_BASE32B (descriptor layout type 1; TMA
//             CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B: 32-byte units XOR row % 4,
//             4-row atoms of 512 B = SBO); 32-element MN chunks 4 KB apart
//             (LBO); the step is 8 K rows (1 KB).  The plain 128B swizzle
//             reads garbage for MN-major tf32 (measured).
__device__ __forceinline__ uint64_t desc_mn_base32b(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  d |= (uint64_t)1 << 61;  // SWIZZLE_128B_BASE32B
  return d;
}
template <bool MN>
__device__ __forceinline__ uint64_t tdesc(uint32_t addr, int k) {
  return MN ? desc_mn_base32b(addr + k * 1024, TBK * 128, 512)
            : sm100::umma_desc_sw128(addr + k * 32, 16, 1024);
}

template <bool A_MN, bool B_MN, bool CONV>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(T_THREADS, 1)
    gemm_tf32_kernel(const __grid_constant__ TMaps maps, const TParams p) {
  using namespace sm100;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sC = smem + T_STAGES * T_STAGE;
  __shared__ __align__(8) uint64_t full[T_STAGES], empty[T_STAGES], ready[T_STAGES], tfull[2],
      tempty[2];
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  // GEMM tile t = (batch, n tile, m tile); conv tile t = (image, pixel tile, channel tile)
  const int tiles_per_batch = CONV ? p.pix_tiles * p.k_tiles : p.num_m * p.num_n;
  const int nk = CONV ? p.RS * p.cb : (p.K + TBK - 1) / TBK;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int units = p.n_whole + 2 * p.n_split;
  // unit -> tile t and column half hu (-1: the whole 256-column tile)
  auto decode = [&](int u, int& t, int& hu) {
    if (u < p.n_whole) {
      t = u;
      hu = -1;
    } else {
      t = p.n_whole + ((u - p.n_whole) >> 1);
      hu = (u - p.n_whole) & 1;
    }
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < T_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
      mbar_init(&ready[i], 3);   // CTA 0: its 2 converter warps + CTA 1's publisher
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 16);   // 8 epilogue warps x 2 CTAs
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&maps.a);
    tma_prefetch(&maps.b);
    if (!CONV) tma_prefetch(&maps.c);
  }
  if (warp == 2) {
    tmem_alloc_pair(&tmem_slot, T_TMEM_COLS);
    tc_fence_before();
  }
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = tmem_slot;
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    TF32_REG_DEC
    if (elect_one()) {
      int st = 0;
      uint32_t ph = 0;
      for (int u = cid; u < units; u += ncl) {
        int t, hu;
        decode(u, t, hu);
        const int b = t / tiles_per_batch, r = t % tiles_per_batch;
        // conv: pixel tile = r / k_tiles ("n" role), channel tile = r % k_tiles ("m" role)
        const int nt = CONV ? r / p.k_tiles : r / p.num_m, mt = CONV ? r % p.k_tiles : r % p.num_m;
        // narrow units: each CTA supplies 64 of the 128 columns (the box still
        // brings 128 rows; the N = 128 MMA reads the first 64)
        const int row = mt * 256 + (int)rank * 128;
        const int col = hu < 0 ? nt * 256 + (int)rank * 128 : nt * 256 + hu * 128 + (int)rank * 64;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty[st], ph ^ 1);
          mbar_expect_tx(&full[st], 2 * T_TILE);
          uint8_t* a_dst = smem + st * T_STAGE;
          uint8_t* b_dst = a_dst + T_TILE;
          if constexpr (CONV) {
            // K order (r, s) outer, 32-channel blocks inner; the image rows of
            // tap (r, s) are the tile's virtual pixels shifted by r * W + s
            const int rs = kb / p.cb, cbk = kb % p.cb;
            const int shift = (rs / p.S) * p.W + (rs % p.S);
            tma_load_3d(a_dst, &maps.a, &full[st], cbk * TBK, rs, row);
            tma_load_3d(b_dst, &maps.b, &full[st], cbk * TBK, col + shift, b);
          } else {
          if (!A_MN) {
            tma_load_3d(a_dst, &maps.a, &full[st], kb * TBK, row, b);
          } else {
#pragma unroll
            for (int c = 0; c < 4; ++c)
              tma_load_3d(a_dst + c * (TBK * 128), &maps.a, &full[st], row + c * 32, kb * TBK, b);
          }
          if (!B_MN) {
            tma_load_3d(b_dst, &maps.b, &full[st], kb * TBK, col, b);
          } else {
#pragma unroll
            for (int c = 0; c < 4; ++c)
              tma_load_3d(b_dst + c * (TBK * 128), &maps.b, &full[st], col + c * 32, kb * TBK, b);
          }
          }
          if (++st == T_STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1 && rank == 1) {
    TF32_REG_DEC
    // CTA 1's publisher: after its 2 converter warps (named barrier 1 + stage),
    // one cluster-scope release-arrive on CTA 0's "stage ready" barrier (the
    // release costs ~1k cycles, kept off the converters' path)
    int st = 0;
    for (int u = cid; u < units; u += ncl)
      for (int kb = 0; kb < nk; ++kb) {
        asm volatile("bar.sync %0, 96;" ::"r"(1 + st) : "memory");
        if (lane == 0) arrive_cluster_release(leader_addr(&ready[st]));
        if (++st == T_STAGES) st = 0;
      }
  } else if (warp == 1) {
    TF32_REG_DEC
    if (elect_one()) {
      // K chunks of T_CHUNK blocks alternate between the two TMEM buffers,
      // each starting from zero; the epilogue adds them in fp32 registers
      constexpr uint32_t idesc_w = idesc_tf32(A_MN, B_MN, 256, 256);
      constexpr uint32_t idesc_n = idesc_tf32(A_MN, B_MN, 256, 128);
      int st = 0;
      uint32_t ph = 0;
      int g = 0;   // chunk sequence number (buffer g & 1)
      for (int u = cid; u < units; u += ncl) {
        const uint32_t idesc = u < p.n_whole ? idesc_w : idesc_n;
        for (int kb = 0; kb < nk; ++kb) {
          if (kb % T_CHUNK == 0) {
            mbar_wait(&tempty[g & 1], ((g >> 1) & 1) ^ 1);
            tc_fence_after();
          }
          const uint32_t d_tmem = tmem_base + (g & 1) * 256;
          wait_cluster_acquire(&ready[st], ph);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + st * T_STAGE);
          const uint32_t b_addr = a_addr + T_TILE;
          const uint32_t alo = a_addr + 2 * T_TILE, blo = a_addr + 3 * T_TILE;
#pragma unroll
          for (int k = 0; k < TBK / 8; ++k) {
            const uint64_t ad = tdesc<A_MN>(a_addr, k), bd = tdesc<B_MN>(b_addr, k);
            mma_tf32_pair(d_tmem, ad, bd, idesc, ((kb % T_CHUNK) | k) != 0);
            if (p.passes == 3) {
              mma_tf32_pair(d_tmem, ad, tdesc<B_MN>(blo, k), idesc, 1);
              mma_tf32_pair(d_tmem, tdesc<A_MN>(alo, k), bd, idesc, 1);
            }
          }
          mma_commit_pair(&empty[st]);
          if (++st == T_STAGES) {
            st = 0;
            ph ^= 1;
          }
          if (kb % T_CHUNK == T_CHUNK - 1 || kb == nk - 1) {
            mma_commit_pair(&tfull[g & 1]);
            ++g;
          }
        }
      }
    }
  } else if (warp == 2 || warp == 3) {
    TF32_REG_DEC
    // lo converters: 2 x 16 KB of raw tiles -> 2 x 16 KB of lo tiles per stage
    const int ct = threadIdx.x - 64;
    int st = 0;
    uint32_t ph = 0;
    for (int u = cid; u < units; u += ncl)
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&full[st], ph);
        const uint32_t raw = smem_u32(smem + st * T_STAGE);
        const uint32_t lo = raw + 2 * T_TILE;
        constexpr int UNITS = 2 * T_TILE / 16;   // 16-byte units
        constexpr int PER = UNITS / 64;
#pragma unroll
        for (int h = 0; h < PER; h += 8) {
          uint4 v[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t off = (uint32_t)((h + i) * 64 + ct) * 16u;
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v[i].x), "=r"(v[i].y), "=r"(v[i].z), "=r"(v[i].w)
                         : "r"(raw + off));
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t off = (uint32_t)((h + i) * 64 + ct) * 16u;
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(lo + off),
                         "r"(tf32_lo(v[i].x)), "r"(tf32_lo(v[i].y)), "r"(tf32_lo(v[i].z)),
                         "r"(tf32_lo(v[i].w))
                         : "memory");
          }
        }
        fence_proxy_async();
        if (rank == 0) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&ready[st]);
        } else {
          asm volatile("bar.arrive %0, 96;" ::"r"(1 + st) : "memory");
        }
        if (++st == T_STAGES) {
          st = 0;
          ph ^= 1;
        }
      }
  } else if (warp >= 4) {
    TF32_REG_INC
    // 8 epilogue warps: TMEM lane quadrant = warp % 4, column half = (warp - 4) / 4.
    // Each thread keeps its row's 128 columns as fp32 partial sums across the
    // K chunks (the tensor core's own accumulation is not round-to-nearest:
    // a single 4096-long TMEM accumulation drifts ~10x further from the f64
    // product than fp32 SGEMM; 128-K chunks summed here in fp32 do not).
    const int quad = warp & 3, half = (warp - 4) >> 2;
    uint8_t* stage = sC + (warp - 4) * (32 * 128);
    const int nchunks = (nk + T_CHUNK - 1) / T_CHUNK;
    int g = 0;
    for (int u = cid; u < units; u += ncl) {
      int t, hu;
      decode(u, t, hu);
      const int b = t / tiles_per_batch, r = t % tiles_per_batch;
      const int nt = CONV ? r / p.k_tiles : r / p.num_m, mt = CONV ? r % p.k_tiles : r % p.num_m;
      // this thread's columns: 128 of a whole tile, 64 of a narrow unit
      const int nq = hu < 0 ? 4 : 2;   // 32-column chunks
      const int cbase = hu < 0 ? nt * 256 + half * 128 : nt * 256 + hu * 128 + half * 64;
      float acc[128];
      for (int c = 0; c < nchunks; ++c, ++g) {
        mbar_wait(&tfull[g & 1], (g >> 1) & 1);
        tc_fence_after();
        const uint32_t taddr = tmem_base + (g & 1) * 256 + half * (hu < 0 ? 128 : 64) +
                               ((uint32_t)(quad * 32) << 16);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (q >= 2 * nq) break;
          uint32_t v[16];
          tmem_ld_32x32b_x16(taddr + q * 16, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i)
            acc[q * 16 + i] = c == 0 ? __uint_as_float(v[i]) : acc[q * 16 + i] + __uint_as_float(v[i]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(leader_addr(&tempty[g & 1]));
      }
      if constexpr (CONV) {
        // this thread: output channel k0 + lane, virtual pixels pix0 + [0, 128).
        // Each 32 x 32 block goes through shared memory (element (row, col)
        // at col * 32 + (row + col) % 32: conflict-free both ways) so that a
        // warp's stores run along the output row of one channel
        const int k0 = mt * 256 + (int)rank * 128 + quad * 32;
        const int pix0 = cbase;
        float* xp = reinterpret_cast<float*>(stage);
        const int kn = p.K - k0;
        float* ybase = p.y + (int64_t)b * p.ys[0] + (int64_t)k0 * p.ys[1];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (q >= nq) break;
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 32; ++i) xp[i * 32 + ((lane + i) & 31)] = acc[q * 32 + i];
          __syncwarp();
          const int m = pix0 + q * 32 + lane;
          const int pp = m / p.W, qq = m - pp * p.W;
          const bool ok = m < p.PW && qq < p.Q;
          float* yp = ybase + (int64_t)pp * p.ys[2] + (int64_t)qq * p.ys[3];
          if (kn >= 32) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float f = xp[lane * 32 + ((j + lane) & 31)];
              if (ok) yp[(int64_t)j * p.ys[1]] = f;
            }
          } else {
            for (int j = 0; j < kn; ++j) {
              const float f = xp[lane * 32 + ((j + lane) & 31)];
              if (ok) yp[(int64_t)j * p.ys[1]] = f;
            }
          }
        }
        continue;
      }
      const int row0 = mt * 256 + (int)rank * 128 + quad * 32;
      const int row = row0 + lane;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (q >= nq) break;
        const int col0 = cbase + q * 32;
        float* f = acc + q * 32;
#pragma unroll
        for (int i = 0; i < 32; ++i) f[i] *= p.alpha;
        if (p.has_d && row < p.d_m) {
          const float* drow = p.d + (int64_t)row * p.d_sm;
          if (p.d_sn == 1 && col0 + 32 <= p.d_n && (p.d_sm % 4) == 0 &&
              (reinterpret_cast<uintptr_t>(p.d) & 15) == 0) {
            const float4* dp = reinterpret_cast<const float4*>(drow + col0);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const float4 w = dp[u];
              f[u * 4] += p.beta * w.x;
              f[u * 4 + 1] += p.beta * w.y;
              f[u * 4 + 2] += p.beta * w.z;
              f[u * 4 + 3] += p.beta * w.w;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (col0 + i < p.d_n) f[i] += p.beta * drow[(int64_t)(col0 + i) * p.d_sn];
          }
        }
        // staging: row = lane, 8 16-byte units, unit u at u ^ (lane & 7)
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
        const uint32_t base = smem_u32(stage) + lane * 128;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(base + ((u ^ (lane & 7)) << 4)),
                       "r"(__float_as_uint(f[u * 4])), "r"(__float_as_uint(f[u * 4 + 1])),
                       "r"(__float_as_uint(f[u * 4 + 2])), "r"(__float_as_uint(f[u * 4 + 3]))
                       : "memory");
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          tma_store_3d(&maps.c, stage, col0, row0, b);
          bulk_commit();
        }
      }
    }
    if (lane == 0) bulk_wait<0>();
  }
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, T_TMEM_COLS);
  }
}

template <bool A_MN, bool B_MN, bool CONV = false>
int launch_tf32(const TMaps& maps, const TParams& p, cudaStream_t s) {
  auto k = gemm_tf32_kernel<A_MN, B_MN, CONV>;
  static size_t attr[kMaxDevices] = {};
  cudaError_t e = smem_attr_once(k, T_SMEM, attr);
  if (e != cudaSuccess) return cuda_fail(e, "gemm tf32 smem attribute");
  const int total = p.n_whole + p.n_split;
  int clusters = sm_count() / 2;
  if (total < clusters) clusters = total;
  e = launch_pdl(k, dim3(2 * clusters), dim3(T_THREADS), T_SMEM, s, maps, p);
  if (e != cudaSuccess) return cuda_fail(e, "gemm tf32 launch");
  return check_launch(CONV ? "conv2d 3xtf32 tcgen05 pair" : "gemm 3xtf32 tcgen05 pair",
                      CONV ? NTB_PATH_CONV_TF32 : NTB_PATH_GEMM_TF32);
}

bool ok_stride4(int64_t elems) { return elems > 0 && (elems * 4) % 16 == 0; }

// narrow tail: if the last wave would leave more than half of the CTA pairs
// idle, its tiles run as two 256 x 128 units each (NTB_GEMM_NO_SPLIT=1: off)
void set_tail(TParams& p, int64_t total) {
  const int64_t pairs = sm_count() / 2;
  const int64_t rem = total % pairs;
  static const bool split = !getenv("NTB_GEMM_NO_SPLIT");
  p.n_split = (split && total > pairs && rem > 0 && 2 * rem <= pairs) ? (int)rem : 0;
  p.n_whole = (int)(total - p.n_split);
}

}  // namespace

int gemm_tf32_sm100(const GemmDesc& g, cudaStream_t s) {
  if (g.k < 1 || g.c_m < 1 || g.c_n < 1 || g.batch < 1) return NTB_ERR_UNSUPPORTED;
  if (g.c_m >= (1ll << 31) || g.c_n >= (1ll << 31) || g.k >= (1ll << 31) || g.batch >= 65536)
    return NTB_ERR_UNSUPPORTED;
  if (!aligned16(g.a) || !aligned16(g.b) || !aligned16(g.c)) return NTB_ERR_UNSUPPORTED;
  bool a_mn, b_mn;
  if (g.a_sk == 1 && (g.a_m == 1 || ok_stride4(g.a_sm))) a_mn = false;
  else if (g.a_sm == 1 && ok_stride4(g.a_sk)) a_mn = true;
  else return NTB_ERR_UNSUPPORTED;
  if (g.b_sk == 1 && (g.b_n == 1 || ok_stride4(g.b_sn))) b_mn = false;
  else if (g.b_sn == 1 && ok_stride4(g.b_sk)) b_mn = true;
  else return NTB_ERR_UNSUPPORTED;
  if (g.batch > 1 && (!ok_stride4(g.a_sb) || !ok_stride4(g.b_sb))) return NTB_ERR_UNSUPPORTED;
  // output through TMA stores: unit column stride, 16-byte rows
  if (g.c_sn != 1 || !(g.c_m == 1 || ok_stride4(g.c_sm)) || (g.batch > 1 && !ok_stride4(g.c_sb)))
    return NTB_ERR_UNSUPPORTED;
  const CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  TMaps maps;
  auto operand = [&](CUtensorMap* m, const void* ptr, bool mn, int64_t rows, int64_t s_row,
                     int64_t s_k, int64_t s_b) {
    uint64_t dims[3], str[2];
    uint32_t box[3];
    const int64_t rstride = mn ? s_k : (rows == 1 ? g.k : s_row);
    if (!mn) {
      dims[0] = g.k; dims[1] = rows; box[0] = TBK; box[1] = 128;
    } else {
      dims[0] = rows; dims[1] = g.k; box[0] = 32; box[1] = TBK;
    }
    dims[2] = g.batch;
    box[2] = 1;
    str[0] = (uint64_t)rstride * 4;
    str[1] = g.batch > 1 ? (uint64_t)s_b * 4 : (uint64_t)dims[1] * str[0];
    return encode_tmap(m, dt, 3, ptr, dims, str, box,
                       mn ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B);
  };
  if (!operand(&maps.a, g.a, a_mn, g.a_m, g.a_sm, g.a_sk, g.a_sb) ||
      !operand(&maps.b, g.b, b_mn, g.b_n, g.b_sn, g.b_sk, g.b_sb))
    return NTB_ERR_UNSUPPORTED;
  {
    const int64_t cs = g.c_m == 1 ? g.c_n : g.c_sm;
    if (!ok_stride4(cs)) return NTB_ERR_UNSUPPORTED;
    uint64_t dims[3] = {(uint64_t)g.c_n, (uint64_t)g.c_m, (uint64_t)g.batch};
    uint64_t str[2] = {(uint64_t)cs * 4, g.batch > 1 ? (uint64_t)g.c_sb * 4 : (uint64_t)g.c_m * cs * 4};
    uint32_t box[3] = {32, 32, 1};
    if (!encode_tmap(&maps.c, dt, 3, g.c, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return NTB_ERR_UNSUPPORTED;
  }
  TParams p;
  p.M = (int)g.c_m;
  p.N = (int)g.c_n;
  p.K = (int)g.k;
  p.batch = (int)g.batch;
  p.num_m = (int)cdiv64(g.c_m, 256);
  p.num_n = (int)cdiv64(g.c_n, 256);
  p.d = static_cast<const float*>(g.d);
  p.d_m = g.d_m;
  p.d_n = g.d_n;
  p.d_sm = g.d_sm;
  p.d_sn = g.d_sn;
  p.alpha = g.alpha;
  p.beta = g.beta;
  p.has_d = g.d != nullptr;
  set_tail(p, (int64_t)p.num_m * p.num_n * p.batch);
  static const int passes = [] {
    const char* e = getenv("NTB_TF32_PASSES");
    return e && e[0] == '1' ? 1 : 3;
  }();
  p.passes = passes;
  if (a_mn) return b_mn ? launch_tf32<true, true>(maps, p, s) : launch_tf32<true, false>(maps, p, s);
  return b_mn ? launch_tf32<false, true>(maps, p, s) : launch_tf32<false, false>(maps, p, s);
}

// ---- conv2d fp32: filter repack + NCHW -> pixel-major transpose, then the
// same 3xTF32 pair kernel in implicit-GEMM mode ------------------------------

namespace {

// W'[k][rs][c4] <- W[k][c][r][s] (0 for c >= C)
__global__ void repack_filter_f32(const float* __restrict__ w, int64_t s0, int64_t s1, int64_t s2,
                                  int64_t s3, float* __restrict__ out, int K, int C, int C4, int R,
                                  int S) {
  const int64_t total = (int64_t)K * R * S * C4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C4);
    const int64_t rest = i / C4;
    const int rs = (int)(rest % (R * S));
    const int k = (int)(rest / (R * S));
    const int r = rs / S, s = rs % S;
    out[i] = c < C ? w[k * s0 + c * s1 + r * s2 + s * s3] : 0.f;
  }
}

// X'[n][pix][c4] <- X[n][c][pix]: 32 channels x 32 pixels per 32 x 8 block
// through a padded shared tile (coalesced along pixels in, channels out).
__global__ void __launch_bounds__(256) nchw_to_pixel_major_f32(const float* __restrict__ x,
                                                               int64_t sn, int64_t sc,
                                                               float* __restrict__ out, int C,
                                                               int C4, int HW) {
  __shared__ float tile[32][33];
  const int n = blockIdx.z, c0 = blockIdx.y * 32, p0 = blockIdx.x * 32;
  const float* src = x + (int64_t)n * sn;
  for (int cy = threadIdx.y; cy < 32; cy += 8) {
    const int c = c0 + cy, pix = p0 + threadIdx.x;
    tile[cy][threadIdx.x] = (c < C && pix < HW) ? src[(int64_t)c * sc + pix] : 0.f;
  }
  __syncthreads();
  float* dst = out + (int64_t)n * HW * C4;
  for (int py = threadIdx.y; py < 32; py += 8) {
    const int pix = p0 + py, c = c0 + threadIdx.x;
    if (pix < HW && c < C4) dst[(int64_t)pix * C4 + c] = tile[threadIdx.x][py];
  }
}

}  // namespace

int conv_tf32_sm100(const ConvDesc& c, cudaStream_t s) {
  if (c.N >= 65536 || c.K >= (1 << 30) || (int64_t)c.H * c.W >= (1ll << 31) || c.C >= (1 << 30))
    return NTB_ERR_UNSUPPORTED;
  const int64_t HW = c.H * c.W, RS = c.R * c.S;
  // channels_last fp32 input ([N][H][W][C], C % 4 == 0) is read in place
  const bool nhwc = c.xs[1] == 1 && c.xs[3] == c.C && c.xs[2] == c.W * c.C &&
                    (c.N == 1 || c.xs[0] == HW * c.C) && c.C % 4 == 0 && aligned16(c.x);
  const bool nchw = c.xs[3] == 1 && c.xs[2] == c.W;
  if (!nhwc && !nchw) return NTB_ERR_UNSUPPORTED;
  const int64_t C4 = nhwc ? c.C : (c.C + 3) / 4 * 4;
  const size_t wbytes = ((size_t)c.K * RS * C4 * 4 + 255) / 256 * 256;
  const size_t xbytes = nhwc ? 0 : (size_t)c.N * HW * C4 * 4;
  char* ws = (char*)workspace(wbytes + xbytes, s);
  if (!ws) return fail(NTB_ERR_CUDA, "conv2d: workspace allocation failed");
  float* wp = reinterpret_cast<float*>(ws);
  const float* xp = nhwc ? static_cast<const float*>(c.x) : reinterpret_cast<const float*>(ws + wbytes);
  const int sms = sm_count();
  {
    const int64_t total = c.K * RS * C4;
    int blocks = (int)cdiv64(total, 256);
    if (blocks > sms * 8) blocks = sms * 8;
    repack_filter_f32<<<blocks, 256, 0, s>>>(static_cast<const float*>(c.w), c.ws[0], c.ws[1],
                                             c.ws[2], c.ws[3], wp, (int)c.K, (int)c.C, (int)C4,
                                             (int)c.R, (int)c.S);
    int rc = check_launch("conv2d fp32 filter repack", NTB_PATH_REPACK);
    if (rc) return rc;
  }
  if (!nhwc) {
    dim3 grid((unsigned)cdiv64(HW, 32), (unsigned)cdiv64(C4, 32), (unsigned)c.N);
    nchw_to_pixel_major_f32<<<grid, dim3(32, 8), 0, s>>>(static_cast<const float*>(c.x), c.xs[0],
                                                        c.xs[1], const_cast<float*>(xp), (int)c.C,
                                                        (int)C4, (int)HW);
    int rc = check_launch("conv2d fp32 NCHW -> pixel-major", NTB_PATH_REPACK);
    if (rc) return rc;
  }
  TMaps maps;
  const CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  {
    uint64_t dims[3] = {(uint64_t)C4, (uint64_t)RS, (uint64_t)c.K};
    uint64_t str[2] = {(uint64_t)C4 * 4, (uint64_t)(RS * C4 * 4)};
    uint32_t box[3] = {TBK, 1, 128};
    if (!encode_tmap(&maps.a, dt, 3, wp, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return fail(NTB_ERR_UNSUPPORTED, "conv2d fp32: filter tensor map");
  }
  {
    uint64_t dims[3] = {(uint64_t)C4, (uint64_t)HW, (uint64_t)c.N};
    uint64_t str[2] = {(uint64_t)C4 * 4, (uint64_t)(HW * C4 * 4)};
    uint32_t box[3] = {TBK, 128, 1};
    if (!encode_tmap(&maps.b, dt, 3, xp, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return fail(NTB_ERR_UNSUPPORTED, "conv2d fp32: image tensor map");
  }
  maps.c = maps.a;   // unused in conv mode
  TParams p = {};
  p.batch = (int)c.N;
  p.K = (int)c.K;
  p.cb = (int)cdiv64(c.C, TBK);
  p.RS = (int)RS;
  p.S = (int)c.S;
  p.W = (int)c.W;
  p.PW = (int)(c.P * c.W);
  p.Q = (int)c.Q;
  p.pix_tiles = (int)cdiv64((int64_t)c.P * c.W, 256);
  p.k_tiles = (int)cdiv64(c.K, 256);
  p.alpha = 1.f;
  p.y = static_cast<float*>(c.y);
  for (int d = 0; d < 4; ++d) p.ys[d] = c.ys[d];
  set_tail(p, (int64_t)p.pix_tiles * p.k_tiles * p.batch);
  static const int passes = [] {
    const char* e = getenv("NTB_TF32_PASSES");
    return e && e[0] == '1' ? 1 : 3;
  }();
  p.passes = passes;
  return launch_tf32<false, false, true>(maps, p, s);
}

}  // namespace ntb
