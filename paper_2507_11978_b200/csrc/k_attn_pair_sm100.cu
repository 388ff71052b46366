// scaled_dot_product_attention on CTA pairs (tcgen05.mma.cta_group::2),
// D = 128.  Same math as k_attn_sm100.cu (v4); different schedule:
//
//   * a CLUSTER of two CTAs (two SMs) owns a work item of 256 query rows;
//     each CTA holds its own 128-row Q tile, and the pair's MMAs are M = 256:
//     S = Q K^T with each CTA supplying 64 of the 128 keys of a K tile (the
//     B operand is split along N across the pair), O += P V with each CTA
//     supplying 64 of the 128 head dims of a V tile.  Per SM that is half
//     the K/V shared-memory traffic of the single-CTA kernel;
//   * TMEM per CTA: NB = 3 S buffers (S_j in buffer j % 3, P_j written in
//     place into its first 64 columns) + O.  S_{j+1} and S_{j+2} are issued
//     long before softmax_j ends, so the softmax runs tile after tile
//     without waiting for P.V + S; S_{j+3} reuses buffer j % 3 after P.V_j
//     (in-order tensor pipe).  Two softmax warpgroups per CTA split each row
//     (keys 0-63 / 64-127, O dims 0-63 / 64-127) and exchange the row max
//     through shared memory once per tile;
//   * warp 0: TMA producer (its CTA's Q tile and K / V halves; the bytes of
//     both CTAs complete on CTA 0's barriers), warp 1 of CTA 0: the MMA
//     issuer, warp 2: TMEM allocation, warps 4-11: softmax + epilogue.
// Measured (B32 H32 S4096 D128): 7.5-7.8 ms vs 7.0-7.25 ms for the
// single-CTA v4 kernel (at higher clocks: 1570-1600 vs 1485-1500 MHz); two
// or three S buffers measure the same, so the wait for S is not what bounds
// it.  NOT the default; NTB_ATTN_PAIR=1 selects it for A/B runs.
//   * ring order K_0, K_1, {V_j, K_{j+2}}: exactly the order the MMAs
//     release the slots in.
// Softmax / lazy rescale / exp split as in v4.  P chunks, s_full and the
// P.V completions are tracked per S buffer so the softmax (which may run a
// tile ahead of the MMA issuer) never gets two phases ahead of a barrier.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "k_sm100.cuh"
#include "sm100_ptx.cuh"

namespace ntb {
namespace {

constexpr int D = 128, BM = 128, BN = 128, PCH = 4;
constexpr int NS = 10;                         // K / V ring slots (16 KB per CTA each)
constexpr int Q_BYTES = BM * D * 2;            // 32 KB: this CTA's query tile
constexpr int SLOT = 16384;                    // K half (64 keys x 128 d) or V half (128 keys x 64 d)
constexpr int OFF_KV = Q_BYTES;
constexpr int SMEM = OFF_KV + NS * SLOT + 1024;
#ifndef NTB_PAIR_NB
#define NTB_PAIR_NB 3
#endif
constexpr int NB = NTB_PAIR_NB;                // S buffers per CTA
constexpr uint32_t T_S = 0, T_O = NB * BN;     // S buffers, then O
static_assert(NB * BN + D <= 512, "TMEM budget");
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kThr = 8.0f;
#ifndef NTB_ATTN_POLY_PAIRS
#define NTB_ATTN_POLY_PAIRS 4
#endif

struct PairMaps {
  CUtensorMap q, k, v;   // boxes: q {64, 128}, k {64, 64}, v {64, 128}
};
struct PairParams {
  int B, H, Sq, Sk, n_qt, n_items;
  float scale_log2;
  void* o;
  int64_t os[4];
};

__device__ __forceinline__ void tma_load_4d_pair(void* dst, const CUtensorMap* m, uint32_t bar_leader,
                                                 int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(sm100::smem_u32(dst)),
      "l"(m), "r"(bar_leader), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void mma_f16_ts_pair(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                                uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 t = __fadd2_rn(x, make_float2(12582912.0f, 12582912.0f));
  const float2 r = __fadd2_rn(t, make_float2(-12582912.0f, -12582912.0f));
  const float2 f = __ffma2_rn(r, make_float2(-1.f, -1.f), x);
  float2 q = __ffma2_rn(f, make_float2(0.0551702793f, 0.0551702793f),
                        make_float2(0.242607975f, 0.242607975f));
  q = __ffma2_rn(q, f, make_float2(0.693260928f, 0.693260928f));
  q = __ffma2_rn(q, f, make_float2(0.999928276f, 0.999928276f));
  return make_float2(__uint_as_float(__float_as_uint(q.x) + (__float_as_uint(t.x) << 23)),
                     __uint_as_float(__float_as_uint(q.y) + (__float_as_uint(t.y) << 23)));
}
template <bool BF16>
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  return BF16 ? sm100::pack_bf16(a, b) : sm100::pack_f16(a, b);
}

// ring sequence (within an item of n tiles) of V_j and K_j
// ring order K_0 .. K_{NB-1}, then {V_j, K_{j+NB}}
__device__ __forceinline__ uint32_t seq_v(int j, int n) { return min(NB + 2 * j, n + j); }
__device__ __forceinline__ uint32_t seq_k(int j) { return j < NB ? j : 2 * j - NB + 1; }

constexpr int THREADS = 384;   // warps 0-3 roles, 4-7 / 8-11 softmax halves

template <bool BF16>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    attn_pair_kernel(const __grid_constant__ PairMaps maps, const PairParams p) {
  using namespace sm100;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t q_full, q_empty, kv_full[NS], kv_empty[NS], s_full[NB],
      p_full[NB][PCH], pv_done[NB], o_full, o_empty;
  __shared__ uint32_t tmem_slot;
  __shared__ float xmax[2][2][BM];   // [tile parity][half] row maxima
  __shared__ float xsum[2][BM];      // [half] row sums (epilogue)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int n_kv = (p.Sk + BN - 1) / BN;

  if (threadIdx.x == 0) {
    mbar_init(&q_full, 1);
    mbar_init(&q_empty, 1);
    for (int i = 0; i < NS; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int b = 0; b < NB; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&pv_done[b], 1);
      for (int c = 0; c < PCH; ++c) mbar_init(&p_full[b][c], 8);   // 4 warps x 2 CTAs
    }
    mbar_init(&o_full, 1);
    mbar_init(&o_empty, 16);   // 8 softmax warps x 2 CTAs
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc_pair(&tmem_slot, 512);
    tc_fence_before();
  }
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch(&maps.q);
      tma_prefetch(&maps.k);
      tma_prefetch(&maps.v);
      uint32_t c = 0;
      int it = 0;
      for (int item = cid; item < p.n_items; item += ncl, ++it) {
        const int qt = item % p.n_qt, bh = item / p.n_qt, h = bh % p.H, b = bh / p.H;
        mbar_wait(&q_empty, (it & 1) ^ 1);
        if (rank == 0) mbar_expect_tx(&q_full, 2 * Q_BYTES);
#pragma unroll
        for (int ch = 0; ch < 2; ++ch)
          tma_load_4d_pair(smem + ch * (BM * 128), &maps.q, leader_addr(&q_full), ch * 64,
                           qt * 256 + (int)rank * BM, h, b);
        // ring order K_0, K_1, then V_j, K_{j+2}
        auto load = [&](uint32_t seq, bool is_v, int j) {
          const uint32_t slot = seq % NS;
          mbar_wait(&kv_empty[slot], ((seq / NS) & 1) ^ 1);
          if (rank == 0) mbar_expect_tx(&kv_full[slot], 2 * SLOT);
          uint8_t* dst = smem + OFF_KV + slot * SLOT;
          const uint32_t bar = leader_addr(&kv_full[slot]);
          if (is_v) {
            // this CTA's 64 head dims of V_j (128 keys), one 128B-swizzled chunk
            tma_load_4d_pair(dst, &maps.v, bar, (int)rank * 64, j * BN, h, b);
          } else {
            // this CTA's 64 keys of K_j, both 64-dim chunks
#pragma unroll
            for (int ch = 0; ch < 2; ++ch)
              tma_load_4d_pair(dst + ch * 8192, &maps.k, bar, ch * 64, j * BN + (int)rank * 64,
                               h, b);
          }
        };
        for (int j = 0; j < NB && j < n_kv; ++j) load(c + j, false, j);
        for (int j = 0; j < n_kv; ++j) {
          load(c + seq_v(j, n_kv), true, j);
          if (j + NB < n_kv) load(c + seq_k(j + NB), false, j + NB);
        }
        c += 2 * n_kv;
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && elect_one()) {
      constexpr uint32_t idesc_s = idesc_f16(BF16, false, false, 256, BN);
      constexpr uint32_t idesc_o = idesc_f16(BF16, false, true, 256, D);
      auto slot_addr = [&](uint32_t seq) { return smem_u32(smem + OFF_KV + (seq % NS) * SLOT); };
      auto wait_kv = [&](uint32_t seq) {
        mbar_wait(&kv_full[seq % NS], (seq / NS) & 1);
        tc_fence_after();
      };
      auto issue_s = [&](uint32_t buf, uint32_t kseq) {
        const uint32_t q_addr = smem_u32(smem);
        const uint32_t k_addr = slot_addr(kseq);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t qoff = (kk >> 2) * (BM * 128) + (kk & 3) * 32;
          const uint32_t koff = (kk >> 2) * 8192 + (kk & 3) * 32;
          mma_f16_ss_pair(tmem + T_S + buf * BN, umma_desc_sw128(q_addr + qoff, 16, 1024),
                          umma_desc_sw128(k_addr + koff, 16, 1024), idesc_s, kk != 0);
        }
        mma_commit_pair(&s_full[buf]);
        mma_commit_pair(&kv_empty[kseq % NS]);
      };
      uint32_t c = 0, t = 0;
      int it = 0;
      for (int item = cid; item < p.n_items; item += ncl, ++it) {
        mbar_wait(&q_full, it & 1);
        tc_fence_after();
        for (int j = 0; j < NB && j < n_kv; ++j) {
          wait_kv(c + j);
          issue_s((t + j) % NB, c + j);
        }
        if (n_kv <= NB) mma_commit_pair(&q_empty);
        for (int j = 0; j < n_kv; ++j, ++t) {
          const uint32_t buf = t % NB, ph = (t / NB) & 1;
          const uint32_t vseq = c + seq_v(j, n_kv);
#pragma unroll
          for (int q = 0; q < PCH; ++q) {
            mbar_wait(&p_full[buf][q], ph);
            tc_fence_after();
            if (q == 0) {
              if (j == 0 && it > 0) {
                mbar_wait(&o_empty, (it - 1) & 1);
                tc_fence_after();
              }
              wait_kv(vseq);
            }
            const uint32_t v_addr = slot_addr(vseq);
#pragma unroll
            for (int k2 = 0; k2 < BN / 16 / PCH; ++k2) {
              const int kk = q * (BN / 16 / PCH) + k2;
              mma_f16_ts_pair(tmem + T_O, tmem + T_S + buf * BN + kk * 8,
                              umma_desc_sw128(v_addr + kk * 2048, 16384, 1024), idesc_o,
                              !(j == 0 && kk == 0));
            }
          }
          mma_commit_pair(&kv_empty[vseq % NS]);
          mma_commit_pair(&pv_done[buf]);
          if (j + NB < n_kv) {
            const uint32_t kseq = c + seq_k(j + NB);
            wait_kv(kseq);
            issue_s(buf, kseq);          // same buffer: after P.V_j in the pipe
            if (j + NB + 1 == n_kv) mma_commit_pair(&q_empty);
          }
          if (j + 1 == n_kv) mma_commit_pair(&o_full);
        }
        c += 2 * n_kv;
      }
    }
  } else if (warp >= 4) {
    // two warpgroups per CTA share each query row: half hf takes keys
    // [64 hf, 64 hf + 64) of every tile and head dims [64 hf, 64 hf + 64) of
    // O; the row maximum is exchanged through shared memory once per tile
    constexpr int HB = BN / 2;
    const int hf = (warp - 4) >> 2;
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const uint32_t t_o = tmem + T_O + hf * (D / 2) + lane_off;
    const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
    uint32_t t = 0;
    int it = 0;
    for (int item = cid; item < p.n_items; item += ncl, ++it) {
      const int qt = item % p.n_qt, bh = item / p.n_qt, h = bh % p.H, b = bh / p.H;
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < n_kv; ++j, ++t) {
        const uint32_t buf = t % NB, par = t & 1;
        const uint32_t t_s = tmem + T_S + buf * BN + lane_off;
        mbar_wait(&s_full[buf], (t / NB) & 1);
        tc_fence_after();
        const int kvalid = p.Sk - j * BN - hf * HB;
        uint32_t v[HB];
#pragma unroll
        for (int ch = 0; ch < HB / 32; ++ch)
          tmem_ld_32x32b_x32(t_s + hf * HB + ch * 32, v + ch * 32);
        tmem_ld_wait();
        if (kvalid < HB) {
#pragma unroll
          for (int i = 0; i < HB; ++i)
            if (i >= kvalid) v[i] = 0xFF800000u;
        }
        float mx8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) mx8[u] = __uint_as_float(v[u]);
#pragma unroll
        for (int i = 8; i < HB; i += 8)
#pragma unroll
          for (int u = 0; u < 8; ++u) mx8[u] = fmaxf(mx8[u], __uint_as_float(v[i + u]));
        const float pmx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        xmax[par][hf][row] = pmx;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        const float mx = fmaxf(pmx, xmax[par][hf ^ 1][row]);
        const float cand = mx * p.scale_log2;
        const bool warp_grow = __any_sync(0xffffffffu, cand > m_used + kThr);
        float alpha = 1.f, m_new = m_used;
        if (warp_grow) {
          m_new = fmaxf(m_used, cand);
          alpha = ex2(m_used - m_new);
          if (j > 0) {
            // S_j ran ahead of P.V_{j-1}: wait for it before touching O
            mbar_wait(&pv_done[(t - 1) % NB], ((t - 1) / NB) & 1);
            tc_fence_after();
#pragma unroll
            for (int ch = 0; ch < D / 64; ++ch) {
              uint32_t w[32];
              tmem_ld_32x32b_x32(t_o + ch * 32, w);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) w[i] = __float_as_uint(__uint_as_float(w[i]) * alpha);
              tmem_st_32x32b_x32(t_o + ch * 32, w);
            }
          }
        }
        const float2 nm2 = make_float2(-m_new, -m_new);
        float2 sum2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int c = 0; c < HB / 32; ++c) {
          uint32_t pk[16];
          float2 xs[16], es[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int i = c * 32 + 2 * q;
            xs[q] = __ffma2_rn(make_float2(__uint_as_float(v[i]), __uint_as_float(v[i + 1])), sc2,
                               nm2);
          }
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            if (((q * NTB_ATTN_POLY_PAIRS) % 16) < NTB_ATTN_POLY_PAIRS) {
              es[q] = ex2_poly2(xs[q]);
            } else {
              es[q].x = ex2(xs[q].x);
              es[q].y = ex2(xs[q].y);
            }
          }
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            sum2[q & 1] = __fadd2_rn(sum2[q & 1], es[q]);
            pk[q] = pack2<BF16>(es[q].x, es[q].y);
          }
          const int chunk = hf * (HB / 32) + c;
          tmem_st_32x32b_x16(t_s + chunk * 16, pk);
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(leader_addr(&p_full[buf][chunk]));
        }
        l = fmaf(l, alpha, (sum2[0].x + sum2[0].y) + (sum2[1].x + sum2[1].y));
        m_used = m_new;
      }
      // epilogue: O half-row -> registers, release O, then O / l -> global
      xsum[hf][row] = l;
      mbar_wait(&o_full, it & 1);
      tc_fence_after();
      uint32_t o[D / 2];
#pragma unroll
      for (int ch = 0; ch < D / 64; ++ch) tmem_ld_32x32b_x32(t_o + ch * 32, o + ch * 32);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_addr(&o_empty));
      asm volatile("bar.sync 1, 256;" ::: "memory");
      const float inv = 1.f / (l + xsum[hf ^ 1][row]);
      asm volatile("bar.sync 1, 256;" ::: "memory");   // xsum reused next item
      const int qrow = qt * 256 + (int)rank * BM + row;
      if (qrow < p.Sq) {
        char* obase = reinterpret_cast<char*>(p.o) +
                      ((int64_t)b * p.os[0] + (int64_t)h * p.os[1] + (int64_t)qrow * p.os[2] +
                       (int64_t)hf * (D / 2) * p.os[3]) * 2;
        if (p.os[3] == 1 && ((reinterpret_cast<uintptr_t>(obase) & 15) == 0)) {
          uint4* dst = reinterpret_cast<uint4*>(obase);
#pragma unroll
          for (int u = 0; u < D / 16; ++u) {
            uint32_t q4[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
              q4[e] = pack2<BF16>(__uint_as_float(o[u * 8 + e * 2]) * inv,
                                  __uint_as_float(o[u * 8 + e * 2 + 1]) * inv);
            dst[u] = make_uint4(q4[0], q4[1], q4[2], q4[3]);
          }
        } else {
#pragma unroll
          for (int i = 0; i < D / 2; ++i) {
            const float f = __uint_as_float(o[i]) * inv;
            const int64_t off = (int64_t)i * p.os[3] * 2;
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
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

bool map4(CUtensorMap* m, CUtensorMapDataType dt, const void* base, int64_t D_, int64_t S, int64_t H,
          int64_t B, const int64_t* st, uint32_t rows) {
  if (st[3] != 1) return false;
  for (int i = 0; i < 3; ++i)
    if ((st[i] * 2) % 16 || st[i] <= 0) return false;
  uint64_t dims[4] = {(uint64_t)D_, (uint64_t)S, (uint64_t)H, (uint64_t)B};
  uint64_t str[3] = {(uint64_t)st[2] * 2, (uint64_t)st[1] * 2, (uint64_t)st[0] * 2};
  uint32_t box[4] = {64, rows, 1, 1};
  return encode_tmap(m, dt, 4, base, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

template <bool BF16>
int launch_pair_attn(const PairMaps& maps, const PairParams& p, cudaStream_t s) {
  auto k = attn_pair_kernel<BF16>;
  static size_t attr[kMaxDevices] = {};
  cudaError_t e = smem_attr_once(k, SMEM, attr);
  if (e != cudaSuccess) return cuda_fail(e, "attention pair smem attribute");
  int clusters = sm_count() / 2;
  if (p.n_items < clusters) clusters = p.n_items;
  k<<<2 * clusters, THREADS, SMEM, s>>>(maps, p);
  return check_launch("sdpa tcgen05 pair", NTB_PATH_ATTN_TC);
}

}  // namespace

int attn_pair_sm100(const AttnDesc& a, int dtype, cudaStream_t s) {
  if (a.D != D) return NTB_ERR_UNSUPPORTED;
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
  auto fix = [](int64_t* st, int64_t B, int64_t H, int64_t S, int64_t D_) {
    if (B == 1) st[0] = H * S * D_;
    if (H == 1) st[1] = S * D_;
    if (S == 1) st[2] = D_;
  };
  fix(qs, a.B, a.H, a.Sq, a.D);
  fix(ks, a.B, a.H, a.Sk, a.D);
  fix(vs, a.B, a.H, a.Sk, a.D);
  PairMaps maps;
  if (!map4(&maps.q, dt, a.q, a.D, a.Sq, a.H, a.B, qs, BM) ||
      !map4(&maps.k, dt, a.k, a.D, a.Sk, a.H, a.B, ks, 64) ||
      !map4(&maps.v, dt, a.v, a.D, a.Sk, a.H, a.B, vs, BN))
    return NTB_ERR_UNSUPPORTED;
  PairParams p;
  p.B = (int)a.B;
  p.H = (int)a.H;
  p.Sq = (int)a.Sq;
  p.Sk = (int)a.Sk;
  p.n_qt = (int)((a.Sq + 255) / 256);
  if ((int64_t)p.n_qt * a.H * a.B >= (1LL << 31)) return NTB_ERR_UNSUPPORTED;
  p.n_items = p.n_qt * p.H * p.B;
  p.scale_log2 = a.scale * kLog2e;
  p.o = a.o;
  for (int i = 0; i < 4; ++i) p.os[i] = a.os[i];
  return bf16 ? launch_pair_attn<true>(maps, p, s) : launch_pair_attn<false>(maps, p, s);
}

}  // namespace ntb
