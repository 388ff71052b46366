// Pipe-throughput microbenchmark (sm_100a): cycles per warp-instruction for
// the ops on the attention softmax path, with 1 or 2 warps per SMSP and 8
// independent chains per thread.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 pipes.cu
#include <cuda_fp16.h>
#include <stdio.h>
#include <stdint.h>

#define N_IT 4096
template <int OP>
__global__ void k(float* out, long long* cyc, float seed) {
  float a[8];
  uint32_t u[8];
  for (int i = 0; i < 8; ++i) { a[i] = seed + threadIdx.x * 1e-3f + i; u[i] = i; }
  float2 b[8];
  for (int i = 0; i < 8; ++i) b[i] = make_float2(a[i], a[i] + 1);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < N_IT; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (OP == 1) { asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(a[i]), "f"(__uint_as_float(u[i]))); }
      if (OP == 2) b[i] = __ffma2_rn(b[i], b[(i + 1) & 7], b[i]);
      if (OP == 3) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i]));
      if (OP == 4) asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(a[(i+3)&7]));
      if (OP == 5) { asm volatile("shl.b32 %0, %0, 3;" : "+r"(u[i])); }
      if (OP == 6) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i])); asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(a[i]), "f"(__uint_as_float(u[i]))); }
      if (OP == 7) { asm volatile("add.s32 %0, %0, %1;" : "+r"(u[i]) : "r"(u[(i+1)&7])); }
      if (OP == 8) { asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(a[i]), "f"(__uint_as_float(u[i]))); asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i])); }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i] + b[i].x + (float)u[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const char* names[] = {"MUFU.EX2", "F2FP f16x2", "FFMA2", "FFMA", "FMNMX", "SHL", "EX2+F2FP", "IADD", "F2FP+FFMA"};
  for (int op = 0; op < 9; ++op) {
    for (int wps = 1; wps <= 4; wps *= 2) {
      int threads = 128 * wps;
      for (int rep = 0; rep < 2; ++rep) {
        switch (op) {
          case 0: k<0><<<148, threads>>>(out, cyc, 0.1f); break;
          case 1: k<1><<<148, threads>>>(out, cyc, 0.1f); break;
          case 2: k<2><<<148, threads>>>(out, cyc, 0.1f); break;
          case 3: k<3><<<148, threads>>>(out, cyc, 0.1f); break;
          case 4: k<4><<<148, threads>>>(out, cyc, 0.1f); break;
          case 5: k<5><<<148, threads>>>(out, cyc, 0.1f); break;
          case 6: k<6><<<148, threads>>>(out, cyc, 0.1f); break;
          case 7: k<7><<<148, threads>>>(out, cyc, 0.1f); break;
          case 8: k<8><<<148, threads>>>(out, cyc, 0.1f); break;
        }
      }
      long long c;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      // per SMSP: wps warps x N_IT x 8 instructions
      printf("%-12s warps/SMSP=%d  cycles per warp-instr per SMSP = %.2f\n", names[op], wps,
             (double)c / (wps * (double)N_IT * 8));
    }
  }
  return 0;
}
