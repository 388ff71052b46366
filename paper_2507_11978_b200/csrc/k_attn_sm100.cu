// scaled_dot_product_attention on the sm_100a tensor cores (builder-defined
// spec: the reference declares sdpa out of scope, catalog.py:36; the paper's
// sdpa is FlashAttention-2).  Version 4.
//
// Persistent CTAs (one per SM) walk work items (b, h, 256 query rows); each
// item is two 128-row query tiles that share every K/V tile (ping-pong, as
// in FlashAttention-4):
//   * warp 0: TMA producer - Q0/Q1 per item, then K_j and V_j as SEPARATE
//     ring entries (128 keys each, 128B-swizzled; K K-major, V MN-major) in
//     a 5-slot ring (D = 128), so K_{j+1} can land while V_j is still in use;
//   * warp 1: one thread issues tcgen05.mma in the order
//       S0_0, S1_0, { PV0_j, S0_{j+1}, PV1_j, S1_{j+1} }_j
//     so the tensor core has the other query tile's work while a softmax
//     warpgroup is busy; commits free K_j after S1_j and V_j after PV1_j;
//   * warps 4-7 / 8-11: softmax warpgroups for Q0 / Q1, ONE THREAD PER QUERY
//     ROW (32x32b TMEM loads give each thread its own row: no shuffles).
//     x = s*scale*log2e - m with packed FFMA2; 2^x on the SFU for most score
//     pairs and as a Cody-Waite + cubic polynomial on the FMA pipe (FFMA2)
//     for NTB_ATTN_POLY_PAIRS of every 16 pairs - the SFU alone would need
//     the whole tensor-core time per tile; row sums in fp32 by FADD2.  P is
//     written back as packed 16-bit INTO THE S COLUMNS OF TMEM and consumed
//     from there (tcgen05.mma, A operand in TMEM);
//   * lazy rescaling: the running max only moves when a row max grows by
//     more than 2^8; only then is the O row (TMEM) rescaled.  S_{g,j} is
//     issued after PV_{g,j-1}, so waiting for S_{g,j} means O is current;
//   * epilogue per item: O row -> registers, O released to the MMA warp
//     (o_empty) before the normalise-and-store, so the next item's PV can
//     start while the rows are written.
// TMEM (512 cols): S0/P0 [0,128) S1/P1 [128,256) O0 [256,256+D) O1 after.
// Keys beyond S_k are masked to -inf; query rows beyond S_q are not stored.
// Tensor roofline: 4*B*H*S_q*S_k*D flop per launch.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "k_sm100.cuh"
#include "sm100_ptx.cuh"

namespace ntb {
namespace {

constexpr int BM = 128, BN = 128;  // query rows per tile, keys per KV tile
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

#ifndef NTB_ATTN_POLY_PAIRS
#define NTB_ATTN_POLY_PAIRS 4  // of every 16 score pairs, 2^x on the FMA pipe
#endif

#ifndef NTB_ATTN_PCH
#define NTB_ATTN_PCH 4  // P_j released to the MMA warp in this many key chunks (4: ~2% over 2)
#endif
#ifndef NTB_ATTN_PCH64
#define NTB_ATTN_PCH64 2  // the same at D = 64 (2: 78.1-78.3 vs 79.2-79.5 us at the paper shape)
#endif
static_assert((NTB_ATTN_PCH == 2 || NTB_ATTN_PCH == 4) && (NTB_ATTN_PCH64 == 2 || NTB_ATTN_PCH64 == 4),
              "P chunks");

#ifndef NTB_ATTN_PBUF
#define NTB_ATTN_PBUF 1  // D = 64: P in its own TMEM columns, S_{j+1} issued during softmax_j
#endif

#ifndef NTB_ATTN_REG_LO
#define NTB_ATTN_REG_LO 72   // producer / MMA (/ rope) warps
#endif
#ifndef NTB_ATTN_REG_HI
#define NTB_ATTN_REG_HI 216  // softmax warpgroups (72/216: no spills; 96/200 spilled, 2-4% slower)
#endif
// setmaxnreg.inc blocks until the CTA's pool (168 registers x 384 threads at
// launch) can serve it: a larger split deadlocks
static_assert(NTB_ATTN_REG_LO * 128 + NTB_ATTN_REG_HI * 256 <= 168 * 384, "register split");
#ifndef NTB_ATTN_PDL
#define NTB_ATTN_PDL 1  // programmatic dependent launch (prologue under the previous kernel's tail)
#endif
#ifndef NTB_ATTN_TRACE
#define NTB_ATTN_TRACE 0  // debug builds: per-phase clock64 stamps of CTA 0's first item
#endif
#if NTB_ATTN_TRACE
__device__ long long g_attn_trace[2 * 64 * 8 + 64 * 8];
#define TRACE_SM(g, j, k)                                                          \
  if (blockIdx.x == 0 && it == 0 && lane == 0 && quad == 0 && (j) < 64)            \
    g_attn_trace[((g) * 64 + (j)) * 8 + (k)] = clock64();
#define TRACE_MMA(j, k) \
  if (blockIdx.x == 0 && it == 0 && (j) < 64) g_attn_trace[128 * 8 + (j) * 8 + (k)] = clock64();
#else
#define TRACE_SM(g, j, k)
#define TRACE_MMA(j, k)
#endif

#ifndef NTB_ATTN_ITRACE
#define NTB_ATTN_ITRACE 0  // debug builds: item-boundary clock64 stamps of CTA 0 (first 16 units)
#endif
#if NTB_ATTN_ITRACE
__device__ long long g_attn_items[3][16][4];
#define ITR(g, it, k)                                                              \
  if (blockIdx.x == 0 && lane == 0 && quad == 0 && (it) < 16) g_attn_items[g][it][k] = clock64();
#define ITRM(it, k) \
  if (blockIdx.x == 0 && (it) < 16) g_attn_items[2][it][k] = clock64();
#else
#define ITR(g, it, k)
#define ITRM(it, k)
#endif

struct AttnMaps {
  CUtensorMap q, k, v;
  CUtensorMap o;   // box {64, 32, 1, 1}, 128B swizzle (TMA-store epilogue), when o_tma
};

struct AttnParams {
  int B, H, Sq, Sk, n_qt, n_items;
  // work units: items [0, n_full) round-robin over the grid, then (when the
  // last round would leave more than half of the CTAs idle) the remaining
  // items as 2 * (n_items - n_full) = n_half SINGLE-TILE units, unit
  // n_full + u on CTA u: query tile u % 2 of item n_full + u / 2
  int n_full, n_half;
  // epilogue: O rows staged in the unit's (then free) Q buffer and written by
  // TMA stores (asynchronous to the softmax warps); else direct vector stores
  int o_tma;
  float scale_log2;
  void* o;
  int64_t os[4];
  // rope fusion (sdpa_rope): half-split rotary tables (S, D/2) of the query
  // rows, row strides in elements
  const void *sin_q, *cos_q;
  int64_t sq_rs, cq_rs;
};

// a * b + c with 16-bit a, b and an fp32 accumulate (FHFMA)
template <bool BF16>
__device__ __forceinline__ float hfma(uint16_t a, uint16_t b, float c) {
  float d;
  if constexpr (BF16) asm("fma.rn.f32.bf16 %0, %1, %2, %3;" : "=f"(d) : "h"(a), "h"(b), "f"(c));
  else asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d) : "h"(a), "h"(b), "f"(c));
  return d;
}

// Rotate `rows` rows of a 128B-swizzled K-major tile in place (half-split
// rotary embedding, x0 = columns [0, D/2), x1 = [D/2, D)):
//   x0' = x0*c - x1*s,  x1' = x0*s + x1*c   (fp32, rounded to 16 bit)
// with c/s = the table rows of positions pos0 + row.  Thread t of `nthr`
// takes 16-byte units round-robin; the pair of units (x0, x1) sits at the
// same swizzled offset of the two 64-column chunks (D = 128) or 64 bytes
// apart in one chunk (D = 64).  Conflict-free: 8 consecutive rows put the
// same unit at 8 different 16-byte columns.
template <int D, bool BF16>
__device__ __forceinline__ void rope_tile(uint8_t* tile, int chunk_bytes, int rows, int pos0,
                                          int pos_limit, const void* sn, int64_t sn_rs,
                                          const void* cs, int64_t cs_rs, int t, int nthr) {
  constexpr int UPR = D / 16;           // 16-byte units per half row (8 elements each)
  const uint16_t* sb = reinterpret_cast<const uint16_t*>(sn);
  const uint16_t* cb = reinterpret_cast<const uint16_t*>(cs);
  constexpr int BATCH = 4;   // units in flight per thread: table loads come from L2
  for (int i0 = t; i0 < rows * UPR; i0 += nthr * BATCH) {
    uint4 x0[BATCH], x1[BATCH], c4[BATCH], s4[BATCH];
    uint4* p0[BATCH];
    uint4* p1[BATCH];
    bool ok[BATCH];
#pragma unroll
    for (int k = 0; k < BATCH; ++k) {
      const int i = i0 + k * nthr;
      const int r = i / UPR, u = i % UPR;
      const int pos = pos0 + r;
      // rows past the sequence are zero (TMA fill) and never stored
      ok[k] = i < rows * UPR && pos < pos_limit;
      uint8_t* rowp = tile + r * 128;
      p0[k] = reinterpret_cast<uint4*>(rowp + ((u ^ (r & 7)) << 4));
      p1[k] = D == 128 ? reinterpret_cast<uint4*>(rowp + chunk_bytes + ((u ^ (r & 7)) << 4))
                       : reinterpret_cast<uint4*>(rowp + (((u + 4) ^ (r & 7)) << 4));
      if (ok[k]) {
        x0[k] = *p0[k];
        x1[k] = *p1[k];
        c4[k] = ld_keep(cb + (int64_t)pos * cs_rs + u * 8);
        s4[k] = ld_keep(sb + (int64_t)pos * sn_rs + u * 8);
      }
    }
#pragma unroll
    for (int k = 0; k < BATCH; ++k) {
      if (!ok[k]) continue;
      const uint32_t a[4] = {x0[k].x, x0[k].y, x0[k].z, x0[k].w};
      const uint32_t b[4] = {x1[k].x, x1[k].y, x1[k].z, x1[k].w};
      const uint32_t cc[4] = {c4[k].x, c4[k].y, c4[k].z, c4[k].w};
      const uint32_t ss[4] = {s4[k].x, s4[k].y, s4[k].z, s4[k].w};
      uint32_t o0[4], o1[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        // x0' = x0 c - x1 s, x1' = x0 s + x1 c with mixed-precision FMAs
        // (16-bit operands, fp32 accumulate: the 16 x 16-bit products are
        // exact in fp32, so this is bit-identical to converting first and
        // computing in fp32 as the standalone rope kernel does, with no
        // conversion instructions)
        float r0[2], r1[2];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const uint16_t x0 = (uint16_t)(a[e] >> (16 * hh)), x1 = (uint16_t)(b[e] >> (16 * hh));
          const uint16_t c = (uint16_t)(cc[e] >> (16 * hh)), sn = (uint16_t)(ss[e] >> (16 * hh));
          r0[hh] = hfma<BF16>(x0, c, -hfma<BF16>(x1, sn, 0.f));
          r1[hh] = hfma<BF16>(x1, c, hfma<BF16>(x0, sn, 0.f));
        }
        o0[e] = BF16 ? sm100::pack_bf16(r0[0], r0[1]) : sm100::pack_f16(r0[0], r0[1]);
        o1[e] = BF16 ? sm100::pack_bf16(r1[0], r1[1]) : sm100::pack_f16(r1[0], r1[1]);
      }
      *p0[k] = make_uint4(o0[0], o0[1], o0[2], o0[3]);
      *p1[k] = make_uint4(o1[0], o1[1], o1[2], o1[3]);
    }
  }
}

#ifndef NTB_ATTN_QDB
#define NTB_ATTN_QDB 1  // double-buffer Q in plain sdpa too (always with rope)
#endif
#ifndef NTB_ATTN_D64_QB2
#define NTB_ATTN_D64_QB2 1  // D = 64: two Q buffers + cross-unit S issue too (82.7-83.9 vs 89.8-90.6 us with one)
#endif
#ifndef NTB_ATTN_SEAM
#define NTB_ATTN_SEAM 1  // with two Q buffers: next unit's first S MMAs issued inside this unit
#endif

template <int D, bool ROPE = false>
struct Layout {
  static constexpr int DCH = D / 64;               // 128B chunks along D
  static constexpr int PCH = D == 64 ? NTB_ATTN_PCH64 : NTB_ATTN_PCH;
  static constexpr int Q_BYTES = BM * D * 2;       // one query tile
  static constexpr int CH = BN * 128;              // one 64-wide chunk of a K/V tile
  static constexpr int SLOT = DCH * CH;            // one K or V tile
  // Q buffers: with rope the next item's two query tiles are loaded and
  // rotated while the current item runs (the rotation is L2-latency bound,
  // ~5 us per item, and would otherwise stall the tensor core between items)
  // measured per shape: D = 128 runs best with two Q
  // buffers, the cross-unit S issue and the Q-buffer epilogue staging;
  // D = 64 (8 KV tiles per unit at the paper's shape) with one Q buffer and
  // the unit-by-unit order
  static constexpr int QB = (ROPE || (NTB_ATTN_QDB && (D == 128 || NTB_ATTN_D64_QB2))) ? 2 : 1;
  static constexpr bool SEAM = NTB_ATTN_SEAM && (D == 128 || ROPE || NTB_ATTN_D64_QB2);
  // (two Q buffers) EARLY_Q: the next unit's Q is requested right after this
  // unit's first K/V tile and each warp releases its staged O rows as soon
  // as the TMA has read them (D = 64, rope: 82 vs 87 us at the paper shape);
  // otherwise the next Q is requested after the unit's last K/V tile and the
  // staging is released during the next unit's second tile (D = 128: 6.92-
  // 6.95 vs 7.05-7.33 ms)
  static constexpr bool EARLY_Q = D == 64 || ROPE;
  static constexpr int NS = D == 128 ? (QB == 2 ? 3 : 5) : 8;  // K/V ring entries
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_KV = QB * 2 * Q_BYTES;
  static constexpr int SMEM = OFF_KV + NS * SLOT + 1024;
  static constexpr uint32_t T_S0 = 0, T_S1 = BN, T_O0 = 2 * BN, T_O1 = 2 * BN + D;
  static_assert(2 * BN + 2 * D <= 512, "TMEM budget");
  // D = 64 leaves 128 TMEM columns: each query tile gets its own P buffer
  // (BN/2 columns of packed 16-bit P), so S_{j+1} can overwrite the S
  // columns as soon as the softmax has read S_j - no wait for P.V + S
  static constexpr bool SEP_P = NTB_ATTN_PBUF && 2 * BN + 2 * D + BN <= 512;
  static constexpr uint32_t T_P0 = SEP_P ? 2 * BN + 2 * D : T_S0;
  static constexpr uint32_t T_P1 = SEP_P ? 2 * BN + 2 * D + BN / 2 : T_S1;
  static_assert(SMEM <= 227 * 1024 - 512, "shared memory budget");
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x for a pair on the FMA pipe: x clamped to [-125, .] (2^i with i >= -125
// keeps the exponent add from wrapping into the sign bit; masked keys, -inf,
// give ~2^-125 instead of 0, below the 16-bit P resolution), x = i + f with
// i = rint(x) (1.5*2^23 trick), f in [-0.5, 0.5]; 2^f by a cubic (rel. err
// 7.5e-5, below half an fp16 / bf16 ulp); 2^i added into the exponent.
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 magic = make_float2(12582912.0f, 12582912.0f);
  const float2 t = __fadd2_rn(x, magic);
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

// The CTA's it-th work unit: item and query tile (-1: both tiles, the
// ping-pong; 0 / 1: that tile alone, on softmax warpgroup 0 and TMEM S0/O0).
// A single-tile unit is always the CTA's last.
__device__ __forceinline__ int n_units(const AttnParams& p) {
  const int b = (int)blockIdx.x, g = (int)gridDim.x;
  return (b < p.n_full ? (p.n_full - b + g - 1) / g : 0) + (b < p.n_half ? 1 : 0);
}
__device__ __forceinline__ void unit_of(const AttnParams& p, int it, int& item, int& half) {
  const int b = (int)blockIdx.x, g = (int)gridDim.x;
  const int nf = b < p.n_full ? (p.n_full - b + g - 1) / g : 0;
  if (it < nf) {
    item = b + it * g;
    half = -1;
  } else {
    item = p.n_full + b / 2;
    half = b & 1;
  }
}

template <int D, bool BF16, bool ROPE>
__global__ void __launch_bounds__(384, 1)
    attn_fwd_kernel(const __grid_constant__ AttnMaps maps, const AttnParams p) {
  using namespace sm100;
  using L = Layout<D, ROPE>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t q_full[L::QB], q_empty[L::QB], kv_full[L::NS], kv_empty[L::NS],
      s_full[2], p_full[2][L::PCH], o_full[2], o_empty[2], q_rot[L::QB], s_free[2], pv_done[2];
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_kv = (p.Sk + BN - 1) / BN;

  if (threadIdx.x == 0) {
    for (int i = 0; i < L::QB; ++i) {
      mbar_init(&q_full[i], 1);
      // the MMA warp's commit after the unit's last S, plus (TMA-store
      // epilogue) the 8 softmax warps once their staged O rows were read
      mbar_init(&q_empty[i], p.o_tma ? 9 : 1);
      mbar_init(&q_rot[i], 2);                  // rope warps 2-3
    }
    for (int i = 0; i < L::NS; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int g = 0; g < 2; ++g) {
      mbar_init(&s_full[g], 1);
      for (int q = 0; q < L::PCH; ++q) mbar_init(&p_full[g][q], 4);
      mbar_init(&o_full[g], 1);
      mbar_init(&o_empty[g], 4);
      mbar_init(&s_free[g], 4);    // SEP_P: S columns read by the 4 softmax warps
      mbar_init(&pv_done[g], 1);   // SEP_P: P.V of a tile complete (P buffer free)
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
#if NTB_ATTN_PDL
  // launched with programmatic stream serialization: the set-up above
  // overlaps the previous kernel's tail; nothing global is read before this
  pdl_wait();
  pdl_trigger();
#endif
  // registers: the producer / MMA warpgroup gives its share to the softmax
  // warpgroups (one 128-column S row per thread lives in registers)
  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(NTB_ATTN_REG_LO));
  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch(&maps.q);
      tma_prefetch(&maps.k);
      tma_prefetch(&maps.v);
      uint32_t c = 0;  // K/V ring sequence number: K_j, V_j, K_{j+1}, ...
      const int nu = n_units(p);
      auto load_q = [&](int it) {
        int item, half;
        unit_of(p, it, item, half);
        const int qt = item % p.n_qt, bh = item / p.n_qt, h = bh % p.H, b = bh / p.H;
        const int qb = it % L::QB;
        mbar_wait(&q_empty[qb], ((it / L::QB) & 1) ^ 1);
        mbar_expect_tx(&q_full[qb], (half < 0 ? 2 : 1) * L::Q_BYTES);
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          if (half >= 0 && g == 1) break;
          const int tile = half < 0 ? g : half;   // a single tile goes to slot 0
#pragma unroll
          for (int ch = 0; ch < L::DCH; ++ch)
            tma_load_4d(smem + L::OFF_Q + (qb * 2 + g) * L::Q_BYTES + ch * (BM * 128), &maps.q,
                        &q_full[qb], ch * 64, qt * 2 * BM + tile * BM, h, b);
        }
      };
      // two Q buffers: the next unit's Q is requested before this unit's K/V
      if (L::QB == 2 && nu > 0) load_q(0);
      for (int it = 0; it < nu; ++it) {
        int item, half;
        unit_of(p, it, item, half);
        const int bh = item / p.n_qt, h = bh % p.H, b = bh / p.H;
        // one Q buffer: this unit's Q after its first K/V tile (the buffer frees
        // only when the previous unit's last S completed; K_0, V_0 need not
        // wait).  Two: the next unit's Q after this unit's last K/V tile (its
        // buffer frees when unit it-1's epilogue staging has been read).
        if (L::QB == 1 && (it == 0 || !L::SEAM)) load_q(it);


        for (int j = 0; j < n_kv; ++j) {
#if !NTB_ATTN_NO_QPREFETCH
          // the next unit's query rows into L2 a few tiles before its TMA
          // load, which is issued only when this unit's last S MMA frees the
          // Q buffer (earlier, the K/V stream of 148 CTAs evicts them again)
          if (L::SEAM && j == (n_kv > 4 ? n_kv - 4 : 0) && it + 1 < nu) {
            int nitem, nhalf;
            unit_of(p, it + 1, nitem, nhalf);
            const int nqt = nitem % p.n_qt, nbh = nitem / p.n_qt;
#pragma unroll
            for (int g = 0; g < 2; ++g) {
              if (nhalf >= 0 && g == 1) break;
              const int tile = nhalf < 0 ? g : nhalf;
#pragma unroll
              for (int ch = 0; ch < L::DCH; ++ch)
                tma_prefetch_4d(&maps.q, ch * 64, nqt * 2 * BM + tile * BM, nbh % p.H, nbh / p.H);
            }
          }
#endif
#pragma unroll
          for (int kv = 0; kv < 2; ++kv, ++c) {
            const uint32_t slot = c % L::NS;
            mbar_wait(&kv_empty[slot], ((c / L::NS) & 1) ^ 1);
            mbar_expect_tx(&kv_full[slot], L::SLOT);
            uint8_t* dst = smem + L::OFF_KV + slot * L::SLOT;
#pragma unroll
            for (int ch = 0; ch < L::DCH; ++ch)
              tma_load_4d(dst + ch * L::CH, kv ? &maps.v : &maps.k, &kv_full[slot], ch * 64, j * BN,
                          h, b);
          }
          if (L::QB == 1 && L::SEAM && it > 0 && j == 0) load_q(it);
          // two Q buffers: the next unit's Q after this unit's first (EARLY_Q)
          // or last K/V tile (its buffer frees when unit it-1's last S
          // completed and its epilogue's staged O rows were read; with rope
          // it is then rotated - ~5 us, L2-latency bound - well before use)
          // (EARLY_Q: a few tiles into the unit rather than at its first
          // tile - the producer runs ~NS/2 tiles ahead of the MMAs, and the
          // buffer is released by the previous unit's epilogue, so waiting
          // for it at tile 0 would stall this unit's next K/V loads)
          if (L::QB == 2 && j == (L::EARLY_Q ? (n_kv > L::NS / 2 ? L::NS / 2 : n_kv - 1) : n_kv - 1) &&
              it + 1 < nu)
            load_q(it + 1);
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc_s = idesc_f16(BF16, false, false, BM, BN);
      constexpr uint32_t idesc_o = idesc_f16(BF16, false, true, BM, D);
      uint32_t c = 0;  // ring sequence number of K_0 of the current item
      uint32_t t = 0;  // tiles consumed (p_full phase)
      int it = 0;
      auto slot_addr = [&](uint32_t seq) {
        return smem_u32(smem + L::OFF_KV + (seq % L::NS) * L::SLOT);
      };
      auto wait_kv = [&](uint32_t seq) {
        mbar_wait(&kv_full[seq % L::NS], (seq / L::NS) & 1);
        tc_fence_after();
      };
      int qb = 0;  // Q buffer of the current item
      auto issue_s = [&](int g, uint32_t kseq) {
        const uint32_t q_addr = smem_u32(smem + L::OFF_Q + (qb * 2 + g) * L::Q_BYTES);
        const uint32_t k_addr = slot_addr(kseq);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * (BM * 128) + (kk & 3) * 32;
          const uint32_t koff = (kk >> 2) * L::CH + (kk & 3) * 32;
          mma_f16_ss(tmem + (g ? L::T_S1 : L::T_S0), umma_desc_sw128(q_addr + off, 16, 1024),
                     umma_desc_sw128(k_addr + koff, 16, 1024), idesc_s, kk != 0);
        }
        mma_commit(&s_full[g]);
      };
      // P.V for one chunk of the keys (P is released by the softmax in L::PCH chunks)
      auto issue_pv = [&](int g, uint32_t vseq, bool first, int half) {
        const uint32_t v_addr = slot_addr(vseq);
#pragma unroll
        for (int k2 = 0; k2 < BN / 16 / L::PCH; ++k2) {
          const int kk = half * (BN / 16 / L::PCH) + k2;
          mma_f16_ts(tmem + (g ? L::T_O1 : L::T_O0), tmem + (g ? L::T_P1 : L::T_P0) + kk * 8,
                     umma_desc_sw128(v_addr + kk * 2048, L::CH, 1024), idesc_o,
                     !(first && kk == 0));
        }
      };
      const int nu = n_units(p);
      auto unit_two = [&](int u) {
        int i, h;
        unit_of(p, u, i, h);
        return h < 0;
      };
      auto wait_q = [&](int u) {
        const int b = u % L::QB;
        mbar_wait(ROPE ? &q_rot[b] : &q_full[b], (u / L::QB) & 1);
        tc_fence_after();
      };
      // S_g of KV tile jn of unit un (K at ring sequence kseq), then the
      // releases that follow the LAST S reading those buffers: K_jn after
      // S1 (S0 for a single-tile unit), the unit's Q after its last tile's S
      auto s_and_release = [&](int g, int un, int jn, bool two_un, uint32_t kseq) {
        qb = un % L::QB;
        issue_s(g, kseq);
        if (g == (two_un ? 1 : 0)) {
          mma_commit(&kv_empty[kseq % L::NS]);
          if (jn == n_kv - 1) mma_commit(&q_empty[qb]);
        }
      };
      // SEAM: the next unit's first S MMAs are issued right behind this unit's
      // last P.V of the same query tile, so the ping-pong runs on across unit
      // boundaries instead of restarting after both warpgroups' epilogues
      // (with one Q buffer, the next unit's Q is loaded - from L2, prefetched
      // a few tiles earlier - once this unit's last S has read the buffer).
      constexpr bool SEAM = L::SEAM;
      for (it = 0; it < nu; ++it) {
        // two: the ping-pong of both query tiles; otherwise tile 0 alone, and
        // the K / V / Q buffers are released after its own MMAs
        const bool two = unit_two(it);
        if (!SEAM || it == 0) {
          ITRM(it, 0)
          wait_q(it);
          ITRM(it, 1)
          wait_kv(c);
          ITRM(it, 2)
          s_and_release(0, it, 0, two, c);
          if (two) s_and_release(1, it, 0, two, c);
          ITRM(it, 3)
        }
        for (int j = 0; j < n_kv; ++j, ++t) {
          const bool more = j + 1 < n_kv;
          const bool nxt = SEAM && !more && it + 1 < nu;   // next S belongs to unit it + 1
          const bool hs = more || nxt;                      // a next S exists
          const int un = more ? it : it + 1, jn = more ? j + 1 : 0;
          const bool two_n = more ? two : (nxt ? unit_two(it + 1) : false);
          const uint32_t kseq = c + 2 * j, vseq = kseq + 1, knext = kseq + 2;
          auto next_s = [&](int g) {
            if (nxt && g == 0) {
              ITRM(it + 1, 1)
              wait_q(it + 1);
              ITRM(it + 1, 2)
            }
            if (g == 0 || two_n) s_and_release(g, un, jn, two_n, knext);
            if (nxt && g == 0) { ITRM(it + 1, 3) }
          };
          // ---- query tile 0
          TRACE_MMA(j, 0)
          if (L::SEP_P && hs && !nxt) {
            // S_0 columns already read by the softmax: next S right away
            mbar_wait(&s_free[0], t & 1);
            wait_kv(knext);
            next_s(0);
          }
          mbar_wait(&p_full[0][0], t & 1);
          tc_fence_after();
          TRACE_MMA(j, 1)
          if (j == 0 && it > 0) {
            mbar_wait(&o_empty[0], (it - 1) & 1);
            tc_fence_after();
          }
          wait_kv(vseq);
          issue_pv(0, vseq, j == 0, 0);
#pragma unroll
          for (int q = 1; q < L::PCH; ++q) {
            mbar_wait(&p_full[0][q], t & 1);
            tc_fence_after();
            issue_pv(0, vseq, j == 0, q);
          }
          TRACE_MMA(j, 2)
          if (!two) mma_commit(&kv_empty[vseq % L::NS]);
          if (L::SEP_P) mma_commit(&pv_done[0]);
          if (!more) mma_commit(&o_full[0]);   // before any next-unit S: O0 is final
          if (L::SEP_P && nxt) {
            mbar_wait(&s_free[0], t & 1);
            wait_kv(knext);
            next_s(0);
          }
          if (hs && !L::SEP_P) {
            wait_kv(knext);
            TRACE_MMA(j, 3)
            next_s(0);
          }
          if (!two) continue;
          // ---- query tile 1
          TRACE_MMA(j, 4)
          if (L::SEP_P && hs && two_n && !nxt) {
            mbar_wait(&s_free[1], t & 1);
            next_s(1);
          }
          mbar_wait(&p_full[1][0], t & 1);
          tc_fence_after();
          TRACE_MMA(j, 5)
          if (j == 0 && it > 0) {
            mbar_wait(&o_empty[1], (it - 1) & 1);
            tc_fence_after();
          }
          issue_pv(1, vseq, j == 0, 0);
#pragma unroll
          for (int q = 1; q < L::PCH; ++q) {
            mbar_wait(&p_full[1][q], t & 1);
            tc_fence_after();
            issue_pv(1, vseq, j == 0, q);
          }
          mma_commit(&kv_empty[vseq % L::NS]);
          if (L::SEP_P) mma_commit(&pv_done[1]);
          if (!more) mma_commit(&o_full[1]);
          if (L::SEP_P && nxt && two_n) {
            mbar_wait(&s_free[1], t & 1);
            next_s(1);
          }
          if (hs && two_n && !L::SEP_P) next_s(1);
          TRACE_MMA(j, 6)
        }
        c += 2 * n_kv;
      }
    }
  } else if (ROPE && (warp == 2 || warp == 3)) {
    // rotary embedding of the two Q tiles of every item, in shared memory
    // between the TMA load and the first S MMA.  (K is rotated once per
    // (b, h) by a pre-pass: rotating every K tile here measured 20.2 ms vs
    // 7.2 ms, because the 16 query blocks that share a K tile each redo it
    // and the table reads double the L2 stream.)
    const int t = (warp - 2) * 32 + lane;
    const int nu = n_units(p);
    for (int it = 0; it < nu; ++it) {
      int item, half;
      unit_of(p, it, item, half);
      const int qt = item % p.n_qt, qb = it % L::QB;
      mbar_wait(&q_full[qb], (it / L::QB) & 1);
#pragma unroll 1
      for (int g = 0; g < (half < 0 ? 2 : 1); ++g)
        rope_tile<D, BF16>(smem + L::OFF_Q + (qb * 2 + g) * L::Q_BYTES, BM * 128, BM,
                           qt * 2 * BM + (half < 0 ? g : half) * BM, p.Sq, p.sin_q, p.sq_rs,
                           p.cos_q, p.cq_rs, t, 64);
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&q_rot[qb]);
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(NTB_ATTN_REG_HI));
    const int g = (warp - 4) >> 2;          // query tile of this warpgroup
    const int quad = warp & 3;              // TMEM lane quadrant
    const int row = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const uint32_t t_s = tmem + (g ? L::T_S1 : L::T_S0) + lane_off;
    const uint32_t t_p = tmem + (g ? L::T_P1 : L::T_P0) + lane_off;
    const uint32_t t_o = tmem + (g ? L::T_O1 : L::T_O0) + lane_off;
    const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
    uint32_t t = 0;
    int stage_pending = -1;   // !EARLY_Q: Q buffer holding this warp's staged O rows
    const int nu = n_units(p);
    for (int it = 0; it < nu; ++it) {
      int item, half;
      unit_of(p, it, item, half);
      // a single-tile unit (always the last) runs on warpgroup 0 alone
      if (half >= 0 && g == 1) break;
      const int tile = half < 0 ? g : half;
      const int qt = item % p.n_qt, bh = item / p.n_qt, h = bh % p.H, b = bh / p.H;
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < n_kv; ++j, ++t) {
        TRACE_SM(g, j, 0)
        mbar_wait(&s_full[g], t & 1);
        tc_fence_after();
        TRACE_SM(g, j, 1)
        if (j == 0) { ITR(g, it, 0) }
        const int kvalid = p.Sk - j * BN;
        uint32_t v[BN];
#pragma unroll
        for (int ch = 0; ch < BN / 32; ++ch) tmem_ld_32x32b_x32(t_s + ch * 32, v + ch * 32);
        tmem_ld_wait();
        if (L::SEP_P) {
          // S is in registers: the MMA warp may write S_{j+1} now
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&s_free[g]);
        }
        TRACE_SM(g, j, 2)
        if (kvalid < BN) {
#pragma unroll
          for (int i = 0; i < BN; ++i)
            if (i >= kvalid) v[i] = 0xFF800000u;   // -inf: masked key
        }
        // row max: 8 independent chains (a single FMNMX chain is ~64 dependent ops)
        float mx8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) mx8[u] = __uint_as_float(v[u]);
#pragma unroll
        for (int i = 8; i < BN; i += 8)
#pragma unroll
          for (int u = 0; u < 8; ++u) mx8[u] = fmaxf(mx8[u], __uint_as_float(v[i + u]));
        const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                               fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        const float cand = mx * p.scale_log2;
        const bool warp_grow = __any_sync(0xffffffffu, cand > m_used + kRescaleThreshold);
        float alpha = 1.f, m_new = m_used;
        if (warp_grow) {
          m_new = fmaxf(m_used, cand);
          alpha = ex2(m_used - m_new);
          if (j > 0) {
            // rescale the O row before any of P_j is released (O is current:
            // S_{g,j} was issued after PV_{g,j-1}; with a separate P buffer
            // S_{g,j} may run ahead of it, so wait for that P.V)
            if (L::SEP_P) {
              mbar_wait(&pv_done[g], (t - 1) & 1);
              tc_fence_after();
            }
#pragma unroll
            for (int ch = 0; ch < D / 32; ++ch) {
              uint32_t w[32];
              tmem_ld_32x32b_x32(t_o + ch * 32, w);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) w[i] = __float_as_uint(__uint_as_float(w[i]) * alpha);
              tmem_st_32x32b_x32(t_o + ch * 32, w);
            }
          }
        }
        TRACE_SM(g, j, 3)
        const float2 nm2 = make_float2(-m_new, -m_new);
        float2 sum2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        if (L::SEP_P && t > 0) {
          // the P buffer is free once the previous tile's P.V completed (at
          // j = 0 that is the previous unit's last P.V, complete before
          // o_full: the wait returns at once, but every pv_done phase is
          // consumed before the next commit - compute-sanitizer synccheck)
          mbar_wait(&pv_done[g], (t - 1) & 1);
          tc_fence_after();
        }
#pragma unroll
        for (int half = 0; half < L::PCH; ++half) {
#pragma unroll
          for (int c2 = 0; c2 < BN / 32 / L::PCH; ++c2) {
            const int ch = half * (BN / 32 / L::PCH) + c2;
            uint32_t pk[16];
            // staged: all 16 scale/subtract FFMA2, then all 2^x, then the
            // sums and packs - independent work laid out for the scheduler
            float2 xs[16], es[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              const int i = ch * 32 + 2 * q;
              xs[q] = __ffma2_rn(make_float2(__uint_as_float(v[i]), __uint_as_float(v[i + 1])),
                                 sc2, nm2);
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
            tmem_st_32x32b_x16(t_p + ch * 16, pk);
          }
          // release this chunk of P_j to the MMA warp
          if (half == L::PCH - 1) { TRACE_SM(g, j, 6) }
          tmem_st_wait();
          if (half == L::PCH - 1) { TRACE_SM(g, j, 7) }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[g][half]);
          if (half == 0) { TRACE_SM(g, j, 4) }
        }
        l = fmaf(l, alpha, (sum2[0].x + sum2[0].y) + (sum2[1].x + sum2[1].y));
        m_used = m_new;
        if (!L::EARLY_Q && stage_pending >= 0 && (j >= 1 || j == n_kv - 1)) {
          // the previous unit's staged O rows: long read by the TMA by now;
          // release that Q buffer to the producer
          if (lane == 0) {
            bulk_wait_read<0>();
            mbar_arrive(&q_empty[stage_pending]);
          }
          stage_pending = -1;
        }

        TRACE_SM(g, j, 5)
      }
      // epilogue: O row -> registers, release O, then O / l -> global
      ITR(g, it, 1)
      mbar_wait(&o_full[g], it & 1);
      tc_fence_after();
      ITR(g, it, 2)
      uint32_t o[D];
#pragma unroll
      for (int ch = 0; ch < D / 32; ++ch) tmem_ld_32x32b_x32(t_o + ch * 32, o + ch * 32);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[g]);
      const float inv = 1.f / l;
      const int qrow = qt * 2 * BM + tile * BM + row;
      if (p.o_tma) {
        // stage this warp's 32 rows x D columns, 64 columns (128 B) per
        // 4 KB box, 128B-swizzled (row r's 16-byte chunk q at q ^ (r & 7):
        // conflict-free), in the unit's Q buffer - free once the unit's last
        // S MMA completed (o_full implies it) - and let the TMA store them
        // (rows past S_q clipped); the producer reloads the buffer only
        // after every warp's TMA has read its staging (q_empty)
        const int qbuf = it % L::QB;
        uint8_t* stage = smem + L::OFF_Q + qbuf * 2 * L::Q_BYTES +
                         ((g * 4 + quad) * L::DCH) * (32 * 128);
        const int row0 = qt * 2 * BM + tile * BM + quad * 32;
#pragma unroll
        for (int ch = 0; ch < L::DCH; ++ch) {
          const uint32_t base = smem_u32(stage + ch * (32 * 128)) + lane * 128;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
              w[e] = pack2<BF16>(__uint_as_float(o[ch * 64 + q * 8 + e * 2]) * inv,
                                 __uint_as_float(o[ch * 64 + q * 8 + e * 2 + 1]) * inv);
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(base + ((q ^ (lane & 7)) << 4)),
                         "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                         : "memory");
          }
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
#pragma unroll
          for (int ch = 0; ch < L::DCH; ++ch)
            tma_store_4d(&maps.o, stage + ch * (32 * 128), ch * 64, row0, h, b);
          bulk_commit();
          if (L::EARLY_Q) {
            // the Q buffer goes back to the producer once the TMA has read
            // the staged rows (a few hundred cycles)
            bulk_wait_read<0>();
            mbar_arrive(&q_empty[qbuf]);
          }
        }
        if (!L::EARLY_Q) stage_pending = qbuf;   // released during the next unit (below)
        ITR(g, it, 3)
      } else if (qrow < p.Sq) {
        char* obase = reinterpret_cast<char*>(p.o) +
                      ((int64_t)b * p.os[0] + (int64_t)h * p.os[1] + (int64_t)qrow * p.os[2]) * 2;
        if (D == 128 && p.os[3] == 1 && ((reinterpret_cast<uintptr_t>(obase) & 31) == 0)) {
          // 256-bit stores: every lane writes whole 32-byte sectors of its row
          // (with 128-bit stores each warp store half-filled 32 sectors, and
          // the warp's next barrier wait queued behind their drain)
#pragma unroll
          for (int u = 0; u < D / 16; ++u) {
            uint32_t q8[8];
#pragma unroll
            for (int e = 0; e < 8; ++e)
              q8[e] = pack2<BF16>(__uint_as_float(o[u * 16 + e * 2]) * inv,
                                  __uint_as_float(o[u * 16 + e * 2 + 1]) * inv);
            asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(obase + u * 32),
                         "r"(q8[0]), "r"(q8[1]), "r"(q8[2]), "r"(q8[3]), "r"(q8[4]), "r"(q8[5]),
                         "r"(q8[6]), "r"(q8[7])
                         : "memory");
          }
          ITR(g, it, 3)
        } else if (p.os[3] == 1 && ((reinterpret_cast<uintptr_t>(obase) & 15) == 0)) {
          uint4* dst = reinterpret_cast<uint4*>(obase);
#pragma unroll
          for (int u = 0; u < D / 8; ++u) {
            uint32_t q4[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
              q4[e] = pack2<BF16>(__uint_as_float(o[u * 8 + e * 2]) * inv,
                                  __uint_as_float(o[u * 8 + e * 2 + 1]) * inv);
            dst[u] = make_uint4(q4[0], q4[1], q4[2], q4[3]);
          }
          ITR(g, it, 3)
        } else {
#pragma unroll
          for (int i = 0; i < D; ++i) {
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
  if (p.o_tma && warp >= 4 && lane == 0) bulk_wait<0>();   // O stores complete before exit
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D, bool BF16, bool ROPE>
int launch_attn(const AttnMaps& maps, AttnParams p, cudaStream_t s) {
  using L = Layout<D, ROPE>;
  auto k = attn_fwd_kernel<D, BF16, ROPE>;
  static size_t attr[kMaxDevices] = {};
  cudaError_t e = smem_attr_once(k, L::SMEM, attr);
  if (e != cudaSuccess) return cuda_fail(e, "attention smem attribute");
  // the TMA-store epilogue stages in a second Q buffer or its own area
  if (L::QB != 2) p.o_tma = 0;
  // Tail split: when the last round of items would leave more than half of
  // the CTAs idle, its items run as two single-tile units each on twice as
  // many CTAs (a single-tile unit takes ~half to ~3/4 of an item: the chain
  // of one warpgroup instead of the ping-pong of two).  Small problems
  // (<= SMs / 2 items) run entirely as single-tile units.
  static const bool split = !getenv("NTB_ATTN_NO_SPLIT");
  const int sms = sm_count();
  int grid = p.n_items < sms ? p.n_items : sms;
  p.n_full = p.n_items;
  p.n_half = 0;
  if (split) {
    if (2 * p.n_items <= sms) {
      p.n_full = 0;
      p.n_half = 2 * p.n_items;
      grid = p.n_half;
    } else {
      const int rounds = (p.n_items + grid - 1) / grid;
      const int tail = p.n_items - (rounds - 1) * grid;
      if (rounds > 1 && 2 * tail <= grid) {
        p.n_full = (rounds - 1) * grid;
        p.n_half = 2 * tail;
      }
    }
  }
  if (NTB_ATTN_PDL) launch_pdl(k, dim3(grid), dim3(384), L::SMEM, s, maps, p);
  else k<<<grid, 384, L::SMEM, s>>>(maps, p);
#if NTB_ATTN_TRACE
  {
    static long long h[2 * 64 * 8 + 64 * 8];
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(h, g_attn_trace, sizeof(h));
    const long long t0 = h[1 * 8 + 0] ? h[0] : h[0];
    for (int j = 0; j < 40; ++j) {
      fprintf(stderr, "j=%2d", j);
      for (int g = 0; g < 2; ++g) {
        const long long* r = h + (g * 64 + j) * 8;
        fprintf(stderr, " | g%d wait@%7lld +%5lld ld %4lld max %4lld h0 %4lld h1c %4lld st %4lld fin %4lld", g,
                r[0] - t0, r[1] - r[0], r[2] - r[1], r[3] - r[2], r[4] - r[3], r[6] - r[4], r[7] - r[6], r[5] - r[7]);
      }
      const long long* m = h + 128 * 8 + j * 8;
      fprintf(stderr, " | mma p0@%7lld h0 +%4lld h1 +%4lld kv +%4lld p1@ +%4lld h0 +%4lld done +%4lld\n",
              m[0] - t0, m[1] - m[0], m[2] - m[1], m[3] - m[2], m[4] - m[3], m[5] - m[4], m[6] - m[5]);
    }
  }
#endif
#if NTB_ATTN_ITRACE
  {
    static long long h[3][16][4];
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(h, g_attn_items, sizeof(h));
    const long long t0 = h[0][0][0];
    for (int it = 0; it < 16; ++it)
      for (int g = 0; g < 2; ++g)
        fprintf(stderr, "unit %2d g%d: S0 ready @%9lld  tiles %7lld  o_full wait %6lld  epilogue %6lld  next S0 after %6lld\n",
                it, g, h[g][it][0] - t0, h[g][it][1] - h[g][it][0], h[g][it][2] - h[g][it][1],
                h[g][it][3] - h[g][it][2], it < 15 ? h[g][it + 1][0] - h[g][it][3] : 0);
    for (int it = 0; it < 16; ++it)
      fprintf(stderr, "unit %2d mma: start @%9lld  q wait %6lld  K0 wait %6lld  S issue %6lld\n", it,
              h[2][it][0] - t0, h[2][it][1] - h[2][it][0], h[2][it][2] - h[2][it][1],
              h[2][it][3] - h[2][it][2]);
  }
#endif
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

bool map4o(CUtensorMap* m, CUtensorMapDataType dt, void* base, int64_t D, int64_t S, int64_t H,
           int64_t B, const int64_t* st) {
  if (st[3] != 1) return false;
  for (int i = 0; i < 3; ++i)
    if ((st[i] * 2) % 16 || st[i] <= 0) return false;
  uint64_t dims[4] = {(uint64_t)D, (uint64_t)S, (uint64_t)H, (uint64_t)B};
  uint64_t str[3] = {(uint64_t)st[2] * 2, (uint64_t)st[1] * 2, (uint64_t)st[0] * 2};
  uint32_t box[4] = {64, 32, 1, 1};
  return encode_tmap(m, dt, 4, base, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

}  // namespace

int attn_sm100(const AttnDesc& a, int dtype, cudaStream_t s, const RopeTables* rope, bool dry_run) {
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
  // O through TMA stores when its layout allows a tensor map (unit inner
  // stride, 16-byte aligned base and strides)
  {
    int64_t os[4] = {a.os[0], a.os[1], a.os[2], a.os[3]};
    fix(os, a.B, a.H, a.Sq, a.D);
    static const bool direct = getenv("NTB_ATTN_DIRECT_STORE") != nullptr;
    p.o_tma = !direct && aligned16(a.o) && map4o(&maps.o, dt, a.o, a.D, a.Sq, a.H, a.B, os);
  }
  p.B = (int)a.B;
  p.H = (int)a.H;
  p.Sq = (int)a.Sq;
  p.Sk = (int)a.Sk;
  p.n_qt = (int)((a.Sq + 2 * BM - 1) / (2 * BM));
  if ((int64_t)p.n_qt * a.H * a.B >= (1LL << 31)) return NTB_ERR_UNSUPPORTED;
  p.n_items = p.n_qt * p.H * p.B;
  p.scale_log2 = a.scale * kLog2e;
  p.o = a.o;
  for (int i = 0; i < 4; ++i) p.os[i] = a.os[i];
  p.sin_q = p.cos_q = nullptr;
  p.sq_rs = p.cq_rs = 0;
  if (rope) {
    // tables (S, D/2): 16-byte aligned rows of contiguous columns, covering
    // every query / key position
    const void* tp[2] = {rope->sin_q, rope->cos_q};
    const int64_t* tr[2] = {rope->sq, rope->cq};
    for (int i = 0; i < 2; ++i) {
      const int64_t rows_needed = a.Sq;
      if (!aligned16(tp[i]) || tr[i][3] != 1 || tr[i][1] != a.D / 2 ||
          (tr[i][2] * 2) % 16 || (tr[i][0] < rows_needed))
        return NTB_ERR_UNSUPPORTED;
    }
    p.sin_q = rope->sin_q; p.sq_rs = rope->sq[2];
    p.cos_q = rope->cos_q; p.cq_rs = rope->cq[2];
    if (dry_run) return NTB_OK;
    if (a.D == 128)
      return bf16 ? launch_attn<128, true, true>(maps, p, s) : launch_attn<128, false, true>(maps, p, s);
    return bf16 ? launch_attn<64, true, true>(maps, p, s) : launch_attn<64, false, true>(maps, p, s);
  }
  if (dry_run) return NTB_OK;
  if (a.D == 128)
    return bf16 ? launch_attn<128, true, false>(maps, p, s) : launch_attn<128, false, false>(maps, p, s);
  return bf16 ? launch_attn<64, true, false>(maps, p, s) : launch_attn<64, false, false>(maps, p, s);
}

}  // namespace ntb
