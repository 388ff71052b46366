// Does a UMMA SWIZZLE_128B K-major operand descriptor accept a start
// address that is a multiple of 128 B but not of 1024 B (a row offset inside
// the 8-row swizzle atom)?  Writes a 256-row x 64-channel window with the
// 128B swizzle of its absolute smem address, then runs D = A * B_sub^T with
// B_sub = window rows [o, o+128) for o = 0..15, once with base_offset = 0
// and once with base_offset = (addr >> 7) & 7, and checks against the host.
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <stdio.h>
#include <stdint.h>
#include <stdlib.h>
#include <math.h>
#include "../../paper_2507_11978_b200/csrc/sm100_ptx.cuh"
using namespace ntb::sm100;

__device__ __forceinline__ uint32_t swz(uint32_t addr) {  // 128B swizzle of an absolute smem byte address
  return addr ^ (((addr >> 7) & 7) << 4);
}

__global__ void k(const __half* A, const __half* Wn, float* out, int o, int use_bo) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;               // 128 rows x 64 ch (we use K=16)
  uint8_t* sB = sm + 16384;       // 256 rows x 64 ch window
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) {
    int r = i / 64, c = i % 64;
    uint32_t ad = a0 + r * 128 + c * 2;
    *(__half*)(sm + (swz(ad) - smem_u32(sm))) = A[i];
  }
  for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) {
    int r = i / 64, c = i % 64;
    uint32_t ad = b0 + r * 128 + c * 2;
    *(__half*)(sm + (swz(ad) - smem_u32(sm))) = Wn[i];
  }
  fence_proxy_async();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, 128);
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_f16(false, false, false, 128, 128);
    uint64_t ad = umma_desc_sw128(a0, 16, 1024);
    uint32_t baddr = b0 + o * 128;
    uint64_t bd = umma_desc_sw128(baddr, 16, 1024);
    if (use_bo) bd |= (uint64_t)((baddr >> 7) & 7) << 49;
    mma_f16_ss(tm, ad, bd, idesc, 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (threadIdx.x < 128) {
    uint32_t v[32];
    for (int cc = 0; cc < 4; ++cc) {
      tmem_ld_32x32b_x32(tm + ((uint32_t)(threadIdx.x & ~31) << 16) + cc * 32, v);
      tmem_ld_wait();
      for (int i = 0; i < 32; ++i) out[threadIdx.x * 128 + cc * 32 + i] = __uint_as_float(v[i]);
    }
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tm, 128);
}

int main() {
  const int na = 128 * 64, nb = 256 * 64;
  __half *hA = (__half*)malloc(na * 2), *hB = (__half*)malloc(nb * 2);
  float* fA = (float*)malloc(na * 4); float* fB = (float*)malloc(nb * 4);
  srand(1);
  for (int i = 0; i < na; ++i) { fA[i] = (rand() % 17 - 8) / 8.f; hA[i] = __float2half(fA[i]); }
  for (int i = 0; i < nb; ++i) { fB[i] = (rand() % 17 - 8) / 8.f; hB[i] = __float2half(fB[i]); }
  __half *dA, *dB; float* dO;
  cudaMalloc(&dA, na * 2); cudaMalloc(&dB, nb * 2); cudaMalloc(&dO, 128 * 128 * 4);
  cudaMemcpy(dA, hA, na * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, nb * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 32768 + 1024);
  float* res = (float*)malloc(128 * 128 * 4);
  for (int bo = 0; bo < 2; ++bo) {
    for (int o = 0; o < 16; ++o) {
      k<<<1, 128, 16384 + 32768 + 1024>>>(dA, dB, dO, o, bo);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(res, dO, 128 * 128 * 4, cudaMemcpyDeviceToHost);
      double maxerr = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 128; ++n) {
          double ref = 0;
          for (int kk = 0; kk < 16; ++kk) ref += (double)fA[m * 64 + kk] * fB[(o + n) * 64 + kk];
          maxerr = fmax(maxerr, fabs(ref - res[m * 128 + n]));
        }
      printf("base_offset=%s o=%2d maxerr %.3g\n", bo ? "(addr>>7)&7" : "0", o, maxerr);
    }
  }
  return 0;
}
