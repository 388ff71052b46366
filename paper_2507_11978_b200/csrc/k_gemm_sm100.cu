// mm / bmm / addmm on the sm_100a tensor cores (reference catalog.py:82-118,
// 226-292; mm.py.golden / bmm.py.golden / addmm.py.golden).
//
// Logical program (pid_0, pid_1) of the reference computes the
// (BLOCK_SIZE_M x BLOCK_SIZE_N) output block with a K loop of BLOCK_SIZE_K
// steps (mm.py.golden:34-45).  Physically this kernel computes 128 x 256
// output tiles (the meta block sizes only define the logical grid; the
// output is identical up to fp32 summation order, covered by the stated
// tolerance):
//
//   * persistent CTAs (one per SM, 1 CTA/SM), static round-robin tile order;
//   * warp 0: TMA producer into a 4-stage shared-memory ring (A 128x64,
//     B 256x64 per stage, 128B-swizzled, K-major or MN-major per operand);
//   * warp 1: one elected thread issues tcgen05.mma (M=128, N=256, K=16)
//     into a double-buffered TMEM accumulator (2 x 256 columns);
//   * warp 2: TMEM allocation owner;
//   * warps 4-7: epilogue - tcgen05.ld TMEM -> registers, fp32 epilogue
//     (addmm: beta*input + alpha*acc, addmm.py.golden:52-53), convert, store;
//     runs concurrently with the next tile's MMAs.
//
// Masks: TMA zero-fills every out-of-range A row / B column / K element, so
// partial tiles need no special casing; the epilogue masks the store to the
// output extent and the addend load to the addend's own extent.
// Tensor roofline: 2*M*N*K flop per launch (x batch).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdlib.h>

#include "common.cuh"
#include "k_sm100.cuh"
#include "sm100_ptx.cuh"

namespace ntb {

bool encode_tmap(CUtensorMap* map, CUtensorMapDataType dt, int rank, const void* base,
                 const uint64_t* dims, const uint64_t* strides_bytes, const uint32_t* box,
                 CUtensorMapSwizzle swizzle) {
  using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                          CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                          CUtensorMapFloatOOBfill);
  static Fn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        !p)
      return false;
    fn = (Fn)p;
  }
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(map, dt, (cuuint32_t)rank, const_cast<void*>(base), (const cuuint64_t*)dims,
                  (const cuuint64_t*)strides_bytes, (const cuuint32_t*)box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

namespace {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;   // 16 KB
constexpr int B_BYTES = BN * BK * 2;   // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024;
constexpr int TMEM_COLS = 512;         // 2 accumulators x 256 fp32 columns

struct GemmMaps {
  CUtensorMap a, b, c;   // c: output, box {64 cols, 32 rows, 1}, 128B swizzle (TMA-store epilogue)
};

struct GemmParams {
  int M, N, K, batch, num_m, num_n;
  void* c;
  int64_t c_sm, c_sn, c_sb;
  const void* d;
  int64_t d_m, d_n, d_sm, d_sn;
  float alpha, beta;
  int has_d;
  int tma_c;   // output written by TMA stores from a swizzled smem staging tile
  // narrow tail: units [n_whole, n_whole + 2 * n_split) are the two 128-
  // column halves of the last n_split tiles (M = 256, N = 128 MMAs)
  int n_whole, n_split;
};

template <bool BF16>
__device__ __forceinline__ float load_el(const void* p, int64_t i) {
  if constexpr (BF16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
  else return __half2float(reinterpret_cast<const __half*>(p)[i]);
}

template <bool BF16>
__device__ __forceinline__ void store_el(void* p, int64_t i, float v) {
  if constexpr (BF16) reinterpret_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
  else reinterpret_cast<__half*>(p)[i] = __float2half_rn(v);
}


// One accumulator row (this thread's TMEM lane) of a 256-column tile:
// tcgen05.ld 32 columns at a time, fp32 epilogue (alpha*acc + beta*addend),
// convert, 128-bit stores when the row segment is aligned.
template <bool BF16>
__device__ __forceinline__ void epilogue_row(const GemmParams& p, uint32_t taddr, int b, int row,
                                             int col_base) {
  using namespace sm100;
  char* cbase = reinterpret_cast<char*>(p.c) + (int64_t)b * p.c_sb * 2;
#pragma unroll 1
  for (int cc = 0; cc < 256 / 32; ++cc) {
    uint32_t v[32];
    __syncwarp();
    tmem_ld_32x32b_x32(taddr + cc * 32, v);
    tmem_ld_wait();
    const int col0 = col_base + cc * 32;
    if (row < p.M && col0 < p.N) {
      float f[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]) * p.alpha;
      if (p.has_d) {
        const bool dvec = p.d_sn == 1 && row < p.d_m && col0 + 32 <= p.d_n && (p.d_sm % 8) == 0 &&
                          ((reinterpret_cast<uintptr_t>(p.d) & 15) == 0);
        if (dvec) {
          const uint4* dp = reinterpret_cast<const uint4*>(
              reinterpret_cast<const char*>(p.d) + ((int64_t)row * p.d_sm + col0) * 2);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 u = dp[q];
            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float lo, hi;
              if constexpr (BF16) {
                __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&w[e]);
                lo = __low2float(h);
                hi = __high2float(h);
              } else {
                __half2 h = *reinterpret_cast<const __half2*>(&w[e]);
                lo = __low2float(h);
                hi = __high2float(h);
              }
              f[q * 8 + e * 2] += p.beta * lo;
              f[q * 8 + e * 2 + 1] += p.beta * hi;
            }
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int col = col0 + i;
            const float dv = (row < p.d_m && col < p.d_n)
                                 ? load_el<BF16>(p.d, (int64_t)row * p.d_sm + (int64_t)col * p.d_sn)
                                 : 0.f;
            f[i] += p.beta * dv;
          }
        }
      }
      const bool cvec = p.c_sn == 1 && col0 + 32 <= p.N && (p.c_sm % 8) == 0 &&
                        ((reinterpret_cast<uintptr_t>(cbase) & 15) == 0);
      if (cvec) {
        uint4* cp = reinterpret_cast<uint4*>(cbase + ((int64_t)row * p.c_sm + col0) * 2);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            w[e] = BF16 ? pack_bf16(f[q * 8 + e * 2], f[q * 8 + e * 2 + 1])
                        : pack_f16(f[q * 8 + e * 2], f[q * 8 + e * 2 + 1]);
          cp[q] = make_uint4(w[0], w[1], w[2], w[3]);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (col0 + i < p.N)
            store_el<BF16>(cbase, (int64_t)row * p.c_sm + (int64_t)(col0 + i) * p.c_sn, f[i]);
      }
    }
  }
  __syncwarp();
}

template <bool A_MN, bool B_MN, bool BF16>
__global__ void __launch_bounds__(256, 1)
    gemm_tc_kernel(const __grid_constant__ GemmMaps maps, const GemmParams p) {
  using namespace sm100;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_per_batch = p.num_m * p.num_n;
  const int total = tiles_per_batch * p.batch;
  const int nk = (p.K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 128);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&maps.a);
    tma_prefetch(&maps.b);
  }
  if (warp == 2) {
    tmem_alloc(&tmem_slot, TMEM_COLS);
    tc_fence_before();
  }
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      int st = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int b = t / tiles_per_batch, r = t % tiles_per_batch;
        const int nt = r / p.num_m, mt = r % p.num_m;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty[st], ph ^ 1);
          mbar_expect_tx(&full[st], STAGE_BYTES);
          uint8_t* a_dst = sA + st * A_BYTES;
          uint8_t* b_dst = sB + st * B_BYTES;
          if (!A_MN) {
            tma_load_3d(a_dst, &maps.a, &full[st], kb * BK, mt * BM, b);
          } else {
#pragma unroll
            for (int c = 0; c < BM / 64; ++c)
              tma_load_3d(a_dst + c * (BK * 128), &maps.a, &full[st], mt * BM + c * 64, kb * BK, b);
          }
          if (!B_MN) {
            tma_load_3d(b_dst, &maps.b, &full[st], kb * BK, nt * BN, b);
          } else {
#pragma unroll
            for (int c = 0; c < BN / 64; ++c)
              tma_load_3d(b_dst + c * (BK * 128), &maps.b, &full[st], nt * BN + c * 64, kb * BK, b);
          }
          if (++st == STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_f16(BF16, A_MN, B_MN, BM, BN);
      int st = 0;
      uint32_t ph = 0;
      int tl = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++tl) {
        const int acc = tl & 1;
        const uint32_t aph = (tl >> 1) & 1;
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[st], ph);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + st * A_BYTES);
          const uint32_t b_addr = smem_u32(sB + st * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? umma_desc_sw128(a_addr + k * 2048, BK * 128, 1024)
                                     : umma_desc_sw128(a_addr + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? umma_desc_sw128(b_addr + k * 2048, BK * 128, 1024)
                                     : umma_desc_sw128(b_addr + k * 32, 16, 1024);
            mma_f16_ss(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          mma_commit(&empty[st]);
          if (++st == STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
        mma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    int tl = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++tl) {
      const int b = t / tiles_per_batch, r = t % tiles_per_batch;
      const int nt = r / p.num_m, mt = r % p.num_m;
      const int acc = tl & 1;
      const uint32_t aph = (tl >> 1) & 1;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const int row = mt * BM + ew * 32 + lane;
      epilogue_row<BF16>(p, tmem_base + acc * BN + ((uint32_t)(ew * 32) << 16), b, row, nt * BN);
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

template <bool A_MN, bool B_MN, bool BF16>
int launch_tc(const GemmMaps& maps, const GemmParams& p, cudaStream_t s) {
  auto k = gemm_tc_kernel<A_MN, B_MN, BF16>;
  static size_t attr[kMaxDevices] = {};
  cudaError_t e = smem_attr_once(k, SMEM_BYTES, attr);
  if (e != cudaSuccess) return cuda_fail(e, "gemm smem attribute");
  const int total = p.num_m * p.num_n * p.batch;
  int grid = sm_count();
  if (total < grid) grid = total;
  k<<<grid, 256, SMEM_BYTES, s>>>(maps, p);
  return check_launch("gemm tcgen05", NTB_PATH_GEMM_TC);
}


// ---- CTA-pair variant (cta_group::2): 256 x 256 tiles per 2-SM cluster ----
// Each CTA of the pair TMA-loads half of A (128 rows) and half of B (128
// rows of N) per 64-wide K step; CTA 0 issues tcgen05.mma.cta_group::2
// (M = 256, N = 256) reading both CTAs' shared memory, so each SM streams
// 32 KB per K step instead of 48 KB (the 1-CTA kernel sits at the L2->SM
// bandwidth ceiling); both CTAs' TMA bytes complete on CTA 0's barrier, the
// MMA commit multicasts stage-free / accumulator-ready to both CTAs, and the
// epilogue warps of both CTAs release the accumulator on CTA 0's barrier.
constexpr int PSTAGES = 6;
constexpr int PA_BYTES = 128 * BK * 2;
constexpr int PB_BYTES = 128 * BK * 2;
constexpr int PSTAGE_BYTES = PA_BYTES + PB_BYTES;
constexpr int PSTAGE_C_BYTES = 4 * 2 * 32 * 128;   // 4 epilogue warps x 2 buffers x 32 rows x 128 B
constexpr int PSMEM_BYTES = PSTAGES * PSTAGE_BYTES + PSTAGE_C_BYTES + 1024;

// TMA-store epilogue for one warp's 32 accumulator rows of a 256-column
// tile: 64 columns at a time, fp32 alpha/beta epilogue, packed to 16-bit and
// written row-per-lane into a 128B-swizzled 32 x 64 staging tile (conflict-
// free: lanes 8 apart hit the same 16-byte chunk column only after the XOR),
// then one lane issues a TMA store that clips at the output extent.  Two
// staging buffers per warp: a buffer is rewritten only after the store that
// read it has finished reading (bulk wait_group.read).
// f[64] = alpha * acc (+ beta * addend) for 64 columns of one row.
template <bool BF16>
__device__ __forceinline__ void add_addend(const GemmParams& p, float* f, int row, int col0) {
  if (!(p.has_d && row < p.d_m)) return;
  const bool dvec = p.d_sn == 1 && col0 + 64 <= p.d_n && (p.d_sm % 8) == 0 &&
                    ((reinterpret_cast<uintptr_t>(p.d) & 15) == 0);
  if (dvec) {
    const uint4* dp = reinterpret_cast<const uint4*>(
        reinterpret_cast<const char*>(p.d) + ((int64_t)row * p.d_sm + col0) * 2);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint4 u = dp[q];
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float lo, hi;
        if constexpr (BF16) {
          __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&w[e]);
          lo = __low2float(h);
          hi = __high2float(h);
        } else {
          __half2 h = *reinterpret_cast<const __half2*>(&w[e]);
          lo = __low2float(h);
          hi = __high2float(h);
        }
        f[q * 8 + e * 2] += p.beta * lo;
        f[q * 8 + e * 2 + 1] += p.beta * hi;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      const int col = col0 + i;
      const float dv = col < p.d_n
                           ? load_el<BF16>(p.d, (int64_t)row * p.d_sm + (int64_t)col * p.d_sn)
                           : 0.f;
      f[i] += p.beta * dv;
    }
  }
}

// One warp's 32 rows x 64 columns (row per lane, values in f) to global via
// a 128B-swizzled staging tile and one TMA store (clipped at the output
// extent).  `chunk` alternates the warp's two staging buffers; a buffer is
// rewritten only after the store that read it has finished reading.
template <bool BF16>
__device__ __forceinline__ void store_chunk_tma(const CUtensorMap* cmap, const float* f,
                                                uint8_t* stage, int chunk, int b, int row0,
                                                int col0, int lane) {
  using namespace sm100;
  uint8_t* buf = stage + (chunk & 1) * (32 * 128);
  if (lane == 0) bulk_wait_read<1>();
  __syncwarp();
  const uint32_t base = smem_u32(buf) + lane * 128;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
      w[e] = BF16 ? pack_bf16(f[q * 8 + e * 2], f[q * 8 + e * 2 + 1])
                  : pack_f16(f[q * 8 + e * 2], f[q * 8 + e * 2 + 1]);
    const uint32_t addr = base + ((q ^ (lane & 7)) << 4);
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(w[0]), "r"(w[1]),
                 "r"(w[2]), "r"(w[3])
                 : "memory");
  }
  fence_proxy_async();
  __syncwarp();
  if (lane == 0) {
    tma_store_3d(cmap, buf, col0, row0, b);
    bulk_commit();
  }
}

// TMA-store epilogue for one warp's 32 accumulator rows of a 256-column
// tile: 64 columns at a time, fp32 alpha/beta epilogue, packed to 16-bit and
// written row-per-lane into a 128B-swizzled 32 x 64 staging tile (conflict-
// free: lanes 8 apart hit the same 16-byte chunk column only after the XOR),
// then one lane issues a TMA store that clips at the output extent.  Two
// staging buffers per warp.  TMEM is released as soon as the last chunk is
// in registers.
template <bool BF16>
__device__ __forceinline__ void epilogue_tma(const GemmParams& p, const CUtensorMap* cmap,
                                             uint32_t taddr, uint8_t* stage, int b, int row0,
                                             int row, int col_base, uint64_t* tempty_leader_bar,
                                             int lane, int nchunks = 4) {
  using namespace sm100;
#pragma unroll 1
  for (int cc = 0; cc < nchunks; ++cc) {
    uint32_t v[64];
    __syncwarp();
    tmem_ld_32x32b_x32(taddr + cc * 64, v);
    tmem_ld_32x32b_x32(taddr + cc * 64 + 32, v + 32);
    tmem_ld_wait();
    if (cc == nchunks - 1) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_addr(tempty_leader_bar));
    }
    const int col0 = col_base + cc * 64;
    float f[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) f[i] = __uint_as_float(v[i]) * p.alpha;
    add_addend<BF16>(p, f, row, col0);
    store_chunk_tma<BF16>(cmap, f, stage, cc, b, row0, col0, lane);
  }
}

template <bool A_MN, bool B_MN, bool BF16>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    gemm_pair_kernel(const __grid_constant__ GemmMaps maps, const GemmParams p) {
  using namespace sm100;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + PSTAGES * PA_BYTES;
  uint8_t* sC = smem + PSTAGES * PSTAGE_BYTES;   // epilogue staging (TMA-store path)
  __shared__ __align__(8) uint64_t full[PSTAGES], empty[PSTAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int tiles_per_batch = p.num_m * p.num_n;
  const int nk = (p.K + BK - 1) / BK;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  // work units: whole 256 x 256 tiles, then the two 256 x 128 column halves
  // of each tail tile (so the last wave keeps every CTA pair busy)
  const int units = p.n_whole + 2 * p.n_split;
  auto decode = [&](int u, int& t, int& half) {
    if (u < p.n_whole) {
      t = u; half = -1;
    } else {
      const int s2 = u - p.n_whole;
      t = p.n_whole + (s2 >> 1); half = s2 & 1;
    }
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < PSTAGES; ++i) {
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
    tma_prefetch(&maps.a);
    tma_prefetch(&maps.b);
    if (p.tma_c) tma_prefetch(&maps.c);
  }
  if (warp == 2) {
    tmem_alloc_pair(&tmem_slot, TMEM_COLS);
    tc_fence_before();
  }
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = tmem_slot;
#if !NTB_GEMM_NO_PDL
  // launched with programmatic stream serialization: everything above ran
  // while the previous kernel drained; the first unit's first K blocks are
  // requested into L2 before the wait (L2 is coherent with the previous
  // kernel's writes), then every thread waits for it to complete
  if (warp == 0 && lane == 0 && cid < units) {
    int t, half;
    decode(cid, t, half);
    const int b = t / tiles_per_batch, r = t % tiles_per_batch;
    const int nt = r / p.num_m, mt = r % p.num_m;
    const int row = mt * 256 + (int)rank * 128;
    const int col = half < 0 ? nt * 256 + (int)rank * 128 : nt * 256 + half * 128 + (int)rank * 64;
    for (int kb = 0; kb < nk && kb < PSTAGES; ++kb) {
      if (!A_MN) {
        tma_prefetch_3d(&maps.a, kb * BK, row, b);
      } else {
        tma_prefetch_3d(&maps.a, row, kb * BK, b);
        tma_prefetch_3d(&maps.a, row + 64, kb * BK, b);
      }
      if (!B_MN) {
        tma_prefetch_3d(&maps.b, kb * BK, col, b);
      } else {
        tma_prefetch_3d(&maps.b, col, kb * BK, b);
        tma_prefetch_3d(&maps.b, col + 64, kb * BK, b);
      }
    }
  }
  pdl_wait();
  pdl_trigger();
#endif

  if (warp == 0) {
    if (elect_one()) {
      int st = 0;
      uint32_t ph = 0;
      for (int u = cid; u < units; u += ncl) {
        int t, half;
        decode(u, t, half);
        const int b = t / tiles_per_batch, r = t % tiles_per_batch;
        const int nt = r / p.num_m, mt = r % p.num_m;
        // narrow units: each CTA supplies 64 of the 128 columns (the TMA box
        // still brings 128 rows / 2 chunks; the MMA reads the first 64)
        const int row = mt * 256 + (int)rank * 128;
        const int col = half < 0 ? nt * 256 + (int)rank * 128 : nt * 256 + half * 128 + (int)rank * 64;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty[st], ph ^ 1);
          if (rank == 0) mbar_expect_tx(&full[st], 2 * PSTAGE_BYTES);
          const uint32_t bar = leader_addr(&full[st]);
          uint8_t* a_dst = sA + st * PA_BYTES;
          uint8_t* b_dst = sB + st * PB_BYTES;
          if (!A_MN) {
            tma_load_3d_pair(a_dst, &maps.a, bar, kb * BK, row, b);
          } else {
            tma_load_3d_pair(a_dst, &maps.a, bar, row, kb * BK, b);
            tma_load_3d_pair(a_dst + BK * 128, &maps.a, bar, row + 64, kb * BK, b);
          }
          if (!B_MN) {
            tma_load_3d_pair(b_dst, &maps.b, bar, kb * BK, col, b);
          } else {
            tma_load_3d_pair(b_dst, &maps.b, bar, col, kb * BK, b);
            tma_load_3d_pair(b_dst + BK * 128, &maps.b, bar, col + 64, kb * BK, b);
          }
          if (++st == PSTAGES) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && elect_one()) {
      constexpr uint32_t idesc = idesc_f16(BF16, A_MN, B_MN, 256, 256);
      int st = 0;
      uint32_t ph = 0;
      int tl = 0;
      constexpr uint32_t idesc_n = idesc_f16(BF16, A_MN, B_MN, 256, 128);
      for (int u = cid; u < units; u += ncl, ++tl) {
        int t, half;
        decode(u, t, half);
        const uint32_t id = half < 0 ? idesc : idesc_n;
        const int acc = tl & 1;
        const uint32_t aph = (tl >> 1) & 1;
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[st], ph);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + st * PA_BYTES);
          const uint32_t b_addr = smem_u32(sB + st * PB_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? umma_desc_sw128(a_addr + k * 2048, BK * 128, 1024)
                                     : umma_desc_sw128(a_addr + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? umma_desc_sw128(b_addr + k * 2048, BK * 128, 1024)
                                     : umma_desc_sw128(b_addr + k * 32, 16, 1024);
            mma_f16_ss_pair(d_tmem, ad, bd, id, (kb | k) != 0);
          }
          mma_commit_pair(&empty[st]);
          if (++st == PSTAGES) {
            st = 0;
            ph ^= 1;
          }
        }
        mma_commit_pair(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    int tl = 0;
    for (int u = cid; u < units; u += ncl, ++tl) {
      int t, half;
      decode(u, t, half);
      const int b = t / tiles_per_batch, r = t % tiles_per_batch;
      const int nt = r / p.num_m, mt = r % p.num_m;
      const int acc = tl & 1;
      const uint32_t aph = (tl >> 1) & 1;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const int row0 = mt * 256 + (int)rank * 128 + ew * 32;
      const int row = row0 + lane;
      if (half >= 0) {
        epilogue_tma<BF16>(p, &maps.c, tmem_base + acc * 256 + ((uint32_t)(ew * 32) << 16),
                           sC + ew * (2 * 32 * 128), b, row0, row, nt * 256 + half * 128,
                           &tempty[acc], lane, 2);
      } else if (p.tma_c) {
        epilogue_tma<BF16>(p, &maps.c, tmem_base + acc * 256 + ((uint32_t)(ew * 32) << 16),
                           sC + ew * (2 * 32 * 128), b, row0, row, nt * 256, &tempty[acc], lane);
      } else {
        epilogue_row<BF16>(p, tmem_base + acc * 256 + ((uint32_t)(ew * 32) << 16), b, row,
                           nt * 256);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(leader_addr(&tempty[acc]));
      }
    }
    if (p.tma_c && lane == 0) bulk_wait<0>();   // all output stores complete before exit
  }
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, TMEM_COLS);
  }
}

template <bool A_MN, bool B_MN, bool BF16>
int launch_pair(const GemmMaps& maps, const GemmParams& p, cudaStream_t s) {
  auto k = gemm_pair_kernel<A_MN, B_MN, BF16>;
  static size_t attr[kMaxDevices] = {};
  cudaError_t e = smem_attr_once(k, PSMEM_BYTES, attr);
  if (e != cudaSuccess) return cuda_fail(e, "gemm pair smem attribute");
  const int total = p.num_m * p.num_n * p.batch;
  int clusters = sm_count() / 2;
  if (total < clusters) clusters = total;
#if NTB_GEMM_NO_PDL
  k<<<2 * clusters, 256, PSMEM_BYTES, s>>>(maps, p);
#else
  launch_pdl(k, dim3(2 * clusters), dim3(256), PSMEM_BYTES, s, maps, p);
#endif
  return check_launch("gemm tcgen05 pair", NTB_PATH_GEMM_TC);
}

bool ok_stride(int64_t elems) { return elems > 0 && (elems * 2) % 16 == 0; }



}  // namespace

int gemm_sm100(const GemmDesc& g, int dtype, cudaStream_t s) {
  if (g.k < 1 || g.c_m < 1 || g.c_n < 1 || g.batch < 1) return NTB_ERR_UNSUPPORTED;
  if (g.c_m >= (1ll << 31) || g.c_n >= (1ll << 31) || g.k >= (1ll << 31) || g.batch >= 65536)
    return NTB_ERR_UNSUPPORTED;
  if (!aligned16(g.a) || !aligned16(g.b)) return NTB_ERR_UNSUPPORTED;
  const bool bf16 = dtype == NTB_BF16;
  const CUtensorMapDataType dt = bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  bool a_mn, b_mn;
  if (g.a_sk == 1 && (g.a_m == 1 || ok_stride(g.a_sm))) a_mn = false;
  else if (g.a_sm == 1 && ok_stride(g.a_sk)) a_mn = true;
  else return NTB_ERR_UNSUPPORTED;
  if (g.b_sk == 1 && (g.b_n == 1 || ok_stride(g.b_sn))) b_mn = false;
  else if (g.b_sn == 1 && ok_stride(g.b_sk)) b_mn = true;
  else return NTB_ERR_UNSUPPORTED;
  if (g.batch > 1 && (!ok_stride(g.a_sb) || !ok_stride(g.b_sb))) return NTB_ERR_UNSUPPORTED;
  static const bool pair_enabled = [] {
    const char* e = getenv("NTB_GEMM_PAIR");
    return !(e && e[0] == '0');
  }();
  const bool pair = pair_enabled && g.c_m > 128;

  GemmMaps maps;
  {
    uint64_t dims[3], str[2];
    uint32_t box[3];
    const int64_t a_rows_stride = a_mn ? g.a_sk : (g.a_m == 1 ? g.k : g.a_sm);
    if (!a_mn) {
      dims[0] = g.k; dims[1] = g.a_m; box[0] = 64; box[1] = BM;
    } else {
      dims[0] = g.a_m; dims[1] = g.k; box[0] = 64; box[1] = BK;
    }
    dims[2] = g.batch;
    box[2] = 1;
    str[0] = (uint64_t)a_rows_stride * 2;
    str[1] = g.batch > 1 ? (uint64_t)g.a_sb * 2 : (uint64_t)dims[1] * str[0];
    if (!encode_tmap(&maps.a, dt, 3, g.a, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return NTB_ERR_UNSUPPORTED;
  }
  {
    uint64_t dims[3], str[2];
    uint32_t box[3];
    const int64_t b_rows_stride = b_mn ? g.b_sk : (g.b_n == 1 ? g.k : g.b_sn);
    if (!b_mn) {
      dims[0] = g.k; dims[1] = g.b_n; box[0] = 64; box[1] = pair ? 128 : BN;
    } else {
      dims[0] = g.b_n; dims[1] = g.k; box[0] = 64; box[1] = BK;
    }
    dims[2] = g.batch;
    box[2] = 1;
    str[0] = (uint64_t)b_rows_stride * 2;
    str[1] = g.batch > 1 ? (uint64_t)g.b_sb * 2 : (uint64_t)dims[1] * str[0];
    if (!encode_tmap(&maps.b, dt, 3, g.b, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return NTB_ERR_UNSUPPORTED;
  }
  GemmParams p;
  p.M = (int)g.c_m;
  p.N = (int)g.c_n;
  p.K = (int)g.k;
  p.batch = (int)g.batch;
  p.num_m = (int)cdiv64(g.c_m, BM);
  p.num_n = (int)cdiv64(g.c_n, BN);
  p.c = g.c;
  p.c_sm = g.c_sm;
  p.c_sn = g.c_sn;
  p.c_sb = g.c_sb;
  p.d = g.d;
  p.d_m = g.d_m;
  p.d_n = g.d_n;
  p.d_sm = g.d_sm;
  p.d_sn = g.d_sn;
  p.alpha = g.alpha;
  p.beta = g.beta;
  p.has_d = g.d != nullptr;
  p.tma_c = 0;
  if (pair && g.c_sn == 1 && aligned16(g.c) && ok_stride(g.c_sm) &&
      (g.batch == 1 || ok_stride(g.c_sb)) && !getenv("NTB_GEMM_NO_TMA_STORE")) {
    uint64_t dims[3] = {(uint64_t)g.c_n, (uint64_t)g.c_m, (uint64_t)g.batch};
    uint64_t str[2] = {(uint64_t)g.c_sm * 2,
                       g.batch > 1 ? (uint64_t)g.c_sb * 2 : (uint64_t)g.c_m * g.c_sm * 2};
    uint32_t box[3] = {64, 32, 1};
    p.tma_c = encode_tmap(&maps.c, dt, 3, g.c, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
  }
  p.n_split = 0;
  if (pair) {
    p.num_m = (int)cdiv64(g.c_m, 256);
    p.num_n = (int)cdiv64(g.c_n, 256);
    // narrow tail: if the last wave would leave more than half of the CTA
    // pairs idle, its tiles run as two 256 x 128 halves each
    const int64_t total = (int64_t)p.num_m * p.num_n * p.batch;
    const int64_t pairs = sm_count() / 2;
    const int64_t rem = total % pairs;
    static const bool split_enabled = !getenv("NTB_GEMM_NO_SPLIT");
    if (split_enabled && p.tma_c && total > pairs && rem > 0 && 2 * rem <= pairs) p.n_split = (int)rem;
    p.n_whole = (int)(total - p.n_split);
    if (bf16) {
      if (a_mn) return b_mn ? launch_pair<true, true, true>(maps, p, s) : launch_pair<true, false, true>(maps, p, s);
      return b_mn ? launch_pair<false, true, true>(maps, p, s) : launch_pair<false, false, true>(maps, p, s);
    }
    if (a_mn) return b_mn ? launch_pair<true, true, false>(maps, p, s) : launch_pair<true, false, false>(maps, p, s);
    return b_mn ? launch_pair<false, true, false>(maps, p, s) : launch_pair<false, false, false>(maps, p, s);
  }
  if (bf16) {
    if (a_mn) return b_mn ? launch_tc<true, true, true>(maps, p, s) : launch_tc<true, false, true>(maps, p, s);
    return b_mn ? launch_tc<false, true, true>(maps, p, s) : launch_tc<false, false, true>(maps, p, s);
  }
  if (a_mn) return b_mn ? launch_tc<true, true, false>(maps, p, s) : launch_tc<true, false, false>(maps, p, s);
  return b_mn ? launch_tc<false, true, false>(maps, p, s) : launch_tc<false, false, false>(maps, p, s);
}

}  // namespace ntb
