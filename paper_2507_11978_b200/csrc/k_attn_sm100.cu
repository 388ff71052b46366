// scaled_dot_product_attention on the sm_100a tensor cores (builder-defined
// spec: the reference declares sdpa out of scope, catalog.py:36; the paper's
// sdpa is FlashAttention-2).
//
// One CTA per (batch, head, 256 query rows) = two 128-row query tiles that
// share every K/V tile (ping-pong, as in FlashAttention-4):
//   * warp 0: TMA producer - Q0/Q1 once, then K_j / V_j (112 keys per tile)
//     into a 2-stage ring (128B-swizzled; K K-major, V MN-major);
//   * warp 1: one thread issues tcgen05.mma in the order
//       S0_0, S1_0, { PV0_j, S0_{j+1}, PV1_j, S1_{j+1} }_j
//     so the tensor core has the other query tile's work while a softmax
//     warpgroup is busy;
//   * warps 4-7 / 8-11: softmax warpgroups for Q0 / Q1, ONE THREAD PER QUERY
//     ROW (32x32b TMEM loads give each thread its own row: no shuffles);
//     P = exp2(S*scale*log2e - m) is written back as packed 16-bit INTO THE
//     S COLUMNS OF TMEM and consumed from there (tcgen05.mma, A in TMEM);
//   * the ROW SUM IS COMPUTED BY THE TENSOR CORE: the P.V MMA multiplies by
//     [V | 1] (N = D + 16; a constant chunk of ones sits after V in every
//     ring stage), so the accumulator carries l next to O, rescaled with it
//     - the softmax threads only do FFMA + EX2 + pack per score, which keeps
//     the SFU and FMA pipes under the tensor-core time per tile;
//   * lazy rescaling: the running max only moves when a row max grows by
//     more than 2^8; only then is the [O | l] row (TMEM) rescaled.  S_{g,j}
//     is issued after PV_{g,j-1}, so waiting for S_{g,j} already means the
//     accumulator is current.
// TMEM (512 cols): S0/P0 [0,112) S1/P1 [112,224) then [O|l]0, [O|l]1.
// Keys beyond S_k are masked to -inf; query rows beyond S_q are not stored.
// Tensor roofline: 4*B*H*S_q*S_k*D flop per launch.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "k_sm100.cuh"
#include "sm100_ptx.cuh"

namespace ntb {
namespace {

constexpr int BM = 128, BN = 112;  // query rows per tile, keys per KV tile
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

struct AttnMaps {
  CUtensorMap q, k, v;
};

struct AttnParams {
  int B, H, Sq, Sk;
  float scale_log2;
  void* o;
  int64_t os[4];
};

template <int D>
struct Layout {
  static constexpr int DCH = D / 64;               // 128B chunks along D
  static constexpr int NO = D + 16;                // [O | l] accumulator width
  static constexpr int Q_BYTES = BM * D * 2;       // one query tile
  static constexpr int KCH = BN * 128;             // one 64-wide chunk of a K/V tile
  static constexpr int K_BYTES = DCH * KCH;
  static constexpr int V_BYTES = (DCH + 1) * KCH;  // V chunks + the ones chunk
  static constexpr int ST_BYTES = K_BYTES + V_BYTES;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_KV = 2 * Q_BYTES;
  static constexpr int SMEM = OFF_KV + 2 * ST_BYTES + 1024;
  static constexpr uint32_t T_S0 = 0, T_S1 = BN, T_O0 = 2 * BN, T_O1 = 2 * BN + NO;
  static_assert(2 * BN + 2 * NO <= 512, "TMEM budget");
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA/ALU pipes (Cody-Waite split + cubic, rel. err 7.5e-5 <
// half an fp16 ulp): takes a quarter of the exponentials off the SFU, which
// otherwise needs ~94% of the tensor-core time per KV tile (FA4's trick).
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -125.f);
  const float t = x + 12582912.0f;                    // 1.5 * 2^23: round to int
  const int i = __float_as_int(t) - 0x4B400000;
  const float f = x - (t - 12582912.0f);             // f in [-0.5, 0.5]
  const float q = fmaf(fmaf(fmaf(0.0551702793f, f, 0.242607975f), f, 0.693260928f), f, 0.999928276f);
  return __int_as_float(__float_as_int(q) + (i << 23));
}

#ifndef NTB_ATTN_POLY
#define NTB_ATTN_POLY 0  // measured: no gain on B200 (8.05-8.30 ms either way, within noise)
#endif

template <bool BF16>
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  return BF16 ? sm100::pack_bf16(a, b) : sm100::pack_f16(a, b);
}

template <int D, bool BF16>
__global__ void __launch_bounds__(384, 1)
    attn_fwd_kernel(const __grid_constant__ AttnMaps maps, const AttnParams p) {
  using namespace sm100;
  using L = Layout<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t q_full, kv_full[2], kv_empty[2], s_full[2], p_full[2],
      o_full[2];
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int n_kv = (p.Sk + BN - 1) / BN;

  // constant "ones" chunk after V in both ring stages (row-sum operand)
  {
    const uint16_t one = BF16 ? 0x3F80 : 0x3C00;
    const uint32_t w = one | ((uint32_t)one << 16);
    for (int st = 0; st < 2; ++st) {
      uint4* dst = reinterpret_cast<uint4*>(smem + L::OFF_KV + st * L::ST_BYTES + L::K_BYTES +
                                            L::DCH * L::KCH);
      for (int i = threadIdx.x; i < L::KCH / 16; i += blockDim.x) dst[i] = make_uint4(w, w, w, w);
    }
    fence_proxy_async();
  }
  if (threadIdx.x == 0) {
    mbar_init(&q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&o_full[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(&tmem_slot, 512);
    tc_fence_before();
  }
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch(&maps.q);
      tma_prefetch(&maps.k);
      tma_prefetch(&maps.v);
      mbar_expect_tx(&q_full, 2 * L::Q_BYTES);
#pragma unroll
      for (int g = 0; g < 2; ++g)
#pragma unroll
        for (int c = 0; c < L::DCH; ++c)
          tma_load_4d(smem + L::OFF_Q + g * L::Q_BYTES + c * (BM * 128), &maps.q, &q_full,
                      c * 64, qt * 2 * BM + g * BM, h, b);
      for (int j = 0; j < n_kv; ++j) {
        const int st = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(&kv_empty[st], ph ^ 1);
        mbar_expect_tx(&kv_full[st], L::K_BYTES + L::DCH * L::KCH);
        uint8_t* kdst = smem + L::OFF_KV + st * L::ST_BYTES;
        uint8_t* vdst = kdst + L::K_BYTES;
#pragma unroll
        for (int c = 0; c < L::DCH; ++c) {
          tma_load_4d(kdst + c * L::KCH, &maps.k, &kv_full[st], c * 64, j * BN, h, b);
          tma_load_4d(vdst + c * L::KCH, &maps.v, &kv_full[st], c * 64, j * BN, h, b);
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc_s = idesc_f16(BF16, false, false, BM, BN);
      constexpr uint32_t idesc_o = idesc_f16(BF16, false, true, BM, L::NO);
      mbar_wait(&q_full, 0);
      auto issue_s = [&](int g, int j) {
        const int st = j & 1;
        const uint32_t q_addr = smem_u32(smem + L::OFF_Q + g * L::Q_BYTES);
        const uint32_t k_addr = smem_u32(smem + L::OFF_KV + st * L::ST_BYTES);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * (BM * 128) + (kk & 3) * 32;
          const uint32_t koff = (kk >> 2) * L::KCH + (kk & 3) * 32;
          mma_f16_ss(tmem + (g ? L::T_S1 : L::T_S0), umma_desc_sw128(q_addr + off, 16, 1024),
                     umma_desc_sw128(k_addr + koff, 16, 1024), idesc_s, kk != 0);
        }
        mma_commit(&s_full[g]);
      };
      auto issue_pv = [&](int g, int j) {
        const int st = j & 1;
        const uint32_t v_addr = smem_u32(smem + L::OFF_KV + st * L::ST_BYTES + L::K_BYTES);
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk)
          mma_f16_ts(tmem + (g ? L::T_O1 : L::T_O0), tmem + (g ? L::T_S1 : L::T_S0) + kk * 8,
                     umma_desc_sw128(v_addr + kk * 2048, L::KCH, 1024), idesc_o, (j | kk) != 0);
      };
      mbar_wait(&kv_full[0], 0);
      tc_fence_after();
      issue_s(0, 0);
      issue_s(1, 0);
      for (int j = 0; j < n_kv; ++j) {
        const int st = j & 1;
        const bool more = j + 1 < n_kv;
        mbar_wait(&p_full[0], j & 1);
        tc_fence_after();
        issue_pv(0, j);
        if (more) {
          mbar_wait(&kv_full[st ^ 1], ((j + 1) >> 1) & 1);   // K/V_{j+1} landed
          tc_fence_after();
          issue_s(0, j + 1);
        } else {
          mma_commit(&o_full[0]);
        }
        mbar_wait(&p_full[1], j & 1);
        tc_fence_after();
        issue_pv(1, j);
        mma_commit(&kv_empty[st]);
        if (more) issue_s(1, j + 1);
        else mma_commit(&o_full[1]);
      }
    }
  } else if (warp >= 4) {
    const int g = (warp - 4) >> 2;          // query tile of this warpgroup
    const int quad = warp & 3;              // TMEM lane quadrant
    const int row = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const uint32_t t_s = tmem + (g ? L::T_S1 : L::T_S0) + lane_off;
    const uint32_t t_o = tmem + (g ? L::T_O1 : L::T_O0) + lane_off;
    float m_used = -INFINITY;
    for (int j = 0; j < n_kv; ++j) {
      mbar_wait(&s_full[g], j & 1);
      tc_fence_after();
      const int kvalid = p.Sk - j * BN;
      // pass 1: row max (S row in registers: 3 x 32 + 16 columns)
      uint32_t v[BN];
      tmem_ld_32x32b_x32(t_s, v);
      tmem_ld_32x32b_x32(t_s + 32, v + 32);
      tmem_ld_32x32b_x32(t_s + 64, v + 64);
      tmem_ld_32x32b_x16(t_s + 96, v + 96);
      tmem_ld_wait();
      float mx = -INFINITY;
      if (kvalid >= BN) {
#pragma unroll
        for (int i = 0; i < BN; ++i) mx = fmaxf(mx, __uint_as_float(v[i]));
      } else {
#pragma unroll
        for (int i = 0; i < BN; ++i)
          if (i < kvalid) mx = fmaxf(mx, __uint_as_float(v[i]));
      }
      const float cand = mx * p.scale_log2;
      const bool warp_grow = __any_sync(0xffffffffu, cand > m_used + kRescaleThreshold);
      float alpha = 1.f, m_new = m_used;
      if (warp_grow) {
        m_new = fmaxf(m_used, cand);
        alpha = ex2(m_used - m_new);
      }
      // pass 2: P = exp2(s*scale - m), packed into the S columns (in order)
#pragma unroll
      for (int c = 0; c < BN / 16; ++c) {
        uint32_t pk[8];
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          const float x0 = fmaf(__uint_as_float(v[c * 16 + i]), p.scale_log2, -m_new);
          const float x1 = fmaf(__uint_as_float(v[c * 16 + i + 1]), p.scale_log2, -m_new);
          float e0, e1;
          if (NTB_ATTN_POLY && (i & 6) == 0) {   // 4 of every 16 scores on the FMA pipe
            e0 = ex2_poly(x0);
            e1 = ex2_poly(x1);
          } else {
            e0 = ex2(x0);
            e1 = ex2(x1);
          }
          if (kvalid < BN) {
            if (c * 16 + i >= kvalid) e0 = 0.f;
            if (c * 16 + i + 1 >= kvalid) e1 = 0.f;
          }
          pk[i / 2] = pack2<BF16>(e0, e1);
        }
        tmem_st_32x32b_x8(t_s + c * 8, pk);
      }
      if (warp_grow && j > 0) {
        // rescale the [O | l] row (current: S_{g,j} was issued after PV_{g,j-1})
#pragma unroll
        for (int c = 0; c < L::NO / 16; ++c) {
          uint32_t w[16];
          tmem_ld_32x32b_x16(t_o + c * 16, w);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) w[i] = __float_as_uint(__uint_as_float(w[i]) * alpha);
          tmem_st_32x32b_x16(t_o + c * 16, w);
        }
      }
      m_used = m_new;
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[g]);
    }
    // epilogue: O / l -> global (l = accumulator column D)
    mbar_wait(&o_full[g], 0);
    tc_fence_after();
    uint32_t lw[1];
    tmem_ld_32x32b_x1(t_o + D, lw);
    tmem_ld_wait();
    const float inv = 1.f / __uint_as_float(lw[0]);
    const int qrow = qt * 2 * BM + g * BM + row;
    char* obase = reinterpret_cast<char*>(p.o) +
                  ((int64_t)b * p.os[0] + (int64_t)h * p.os[1] + (int64_t)qrow * p.os[2]) * 2;
    const bool vec = p.os[3] == 1 && ((reinterpret_cast<uintptr_t>(obase) & 15) == 0);
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t w[32];
      tmem_ld_32x32b_x32(t_o + c * 32, w);
      tmem_ld_wait();
      if (qrow < p.Sq) {
        if (vec) {
          uint4* dst = reinterpret_cast<uint4*>(obase + c * 64);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            uint32_t q4[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
              q4[e] = pack2<BF16>(__uint_as_float(w[u * 8 + e * 2]) * inv,
                                  __uint_as_float(w[u * 8 + e * 2 + 1]) * inv);
            dst[u] = make_uint4(q4[0], q4[1], q4[2], q4[3]);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float f = __uint_as_float(w[i]) * inv;
            const int64_t off = (int64_t)(c * 32 + i) * p.os[3] * 2;
            if constexpr (BF16)
              *reinterpret_cast<__nv_bfloat16*>(obase + off) = __float2bfloat16_rn(f);
            else
              *reinterpret_cast<__half*>(obase + off) = __float2half_rn(f);
          }
        }
      }
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D, bool BF16>
int launch_attn(const AttnMaps& maps, const AttnParams& p, cudaStream_t s) {
  using L = Layout<D>;
  auto k = attn_fwd_kernel<D, BF16>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
    if (e != cudaSuccess) return cuda_fail(e, "attention smem attribute");
    attr_set = true;
  }
  dim3 grid((unsigned)((p.Sq + 2 * BM - 1) / (2 * BM)), (unsigned)p.H, (unsigned)p.B);
  k<<<grid, 384, L::SMEM, s>>>(maps, p);
  return check_launch("sdpa tcgen05", NTB_PATH_ATTN_TC);
}

bool map4(CUtensorMap* m, CUtensorMapDataType dt, const void* base, int64_t D, int64_t S, int64_t H,
          int64_t B, const int64_t* st, uint32_t rows) {
  if (st[3] != 1) return false;
  for (int i = 0; i < 3; ++i)
    if ((st[i] * 2) % 16 || st[i] <= 0) return false;
  uint64_t dims[4] = {(uint64_t)D, (uint64_t)S, (uint64_t)H, (uint64_t)B};
  uint64_t str[3] = {(uint64_t)st[2] * 2, (uint64_t)st[1] * 2, (uint64_t)st[0] * 2};
  uint32_t box[4] = {64, rows, 1, 1};
  return encode_tmap(m, dt, 4, base, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

}  // namespace

int attn_sm100(const AttnDesc& a, int dtype, cudaStream_t s) {
  if (a.D != 64 && a.D != 128) return NTB_ERR_UNSUPPORTED;
  if (a.Sk < 1 || a.Sq < 1 || a.B >= 65536 || a.H >= 65536 || a.Sq >= (1 << 30) ||
      a.Sk >= (1 << 30))
    return NTB_ERR_UNSUPPORTED;
  if (!aligned16(a.q) || !aligned16(a.k) || !aligned16(a.v)) return NTB_ERR_UNSUPPORTED;
  const bool bf16 = dtype == NTB_BF16;
  const CUtensorMapDataType dt = bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  int64_t qs[4], ks[4], vs[4];
  for (int i = 0; i < 4; ++i) {
    qs[i] = a.qs[i];
    ks[i] = a.ks[i];
    vs[i] = a.vs[i];
  }
  // size-1 dims: any stride is fine for TMA but must still be a 16B multiple
  auto fix = [](int64_t* st, int64_t B, int64_t H, int64_t S, int64_t D) {
    if (B == 1) st[0] = H * S * D;
    if (H == 1) st[1] = S * D;
    if (S == 1) st[2] = D;
  };
  fix(qs, a.B, a.H, a.Sq, a.D);
  fix(ks, a.B, a.H, a.Sk, a.D);
  fix(vs, a.B, a.H, a.Sk, a.D);
  AttnMaps maps;
  if (!map4(&maps.q, dt, a.q, a.D, a.Sq, a.H, a.B, qs, BM) ||
      !map4(&maps.k, dt, a.k, a.D, a.Sk, a.H, a.B, ks, BN) ||
      !map4(&maps.v, dt, a.v, a.D, a.Sk, a.H, a.B, vs, BN))
    return NTB_ERR_UNSUPPORTED;
  AttnParams p;
  p.B = (int)a.B;
  p.H = (int)a.H;
  p.Sq = (int)a.Sq;
  p.Sk = (int)a.Sk;
  p.scale_log2 = a.scale * kLog2e;
  p.o = a.o;
  for (int i = 0; i < 4; ++i) p.os[i] = a.os[i];
  if (a.D == 128) return bf16 ? launch_attn<128, true>(maps, p, s) : launch_attn<128, false>(maps, p, s);
  return bf16 ? launch_attn<64, true>(maps, p, s) : launch_attn<64, false>(maps, p, s);
}

}  // namespace ntb
