// tcgen05.mma issue rate by shape: cycles per K=16 MMA for SS (A and B in
// shared memory) at M=128 and N = 64 / 128 / 256, and TS (A in TMEM).  One
// CTA per SM, one thread issues back to back, clock64 around the batch.
// Question it answers: does an M=128 N=64 SS MMA (attention with 64-key
// tiles) run at the tensor floor (32 cyc) or is it paced by shared memory?
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <stdio.h>
#include <stdint.h>
#include "../../paper_2507_11978_b200/csrc/sm100_ptx.cuh"
using namespace ntb::sm100;

template <int N, bool TS>
__global__ void k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x3c003c00u;
  fence_proxy_async();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_f16(false, false, false, 128, N);
    const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 16384);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (TS)
          mma_f16_ts(tm, tm + 256 + kk * 8, umma_desc_sw128(b0 + kk * 32, 16, 1024), idesc, 1);
        else
          mma_f16_ss(tm, umma_desc_sw128(a0 + kk * 32, 16, 1024),
                     umma_desc_sw128(b0 + kk * 32, 16, 1024), idesc, 1);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tm, 512);
}

template <int N, bool TS>
void run(const char* name, long long* d, int sms) {
  const int iters = 20000;
  cudaFuncSetAttribute(k<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 32768 + 1024);
  k<N, TS><<<sms, 128, 16384 + 32768 + 1024>>>(d, iters);
  k<N, TS><<<sms, 128, 16384 + 32768 + 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  if (e) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
  long long h[256];
  cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < sms; ++i) s += h[i];
  const double cyc = s / sms / (iters * 4.0);
  printf("%-14s N=%3d  %.1f cyc/mma  floor %d  -> %.0f flop/cyc/SM\n", name, N, cyc, 128 * N / 256,
         2.0 * 128 * N * 16 / cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d;
  cudaMalloc(&d, 256 * 8);
  run<64, false>("SS", d, sms);
  run<128, false>("SS", d, sms);
  run<256, false>("SS", d, sms);
  run<64, true>("TS", d, sms);
  run<128, true>("TS", d, sms);
  run<256, true>("TS", d, sms);
  return 0;
}
