// Internal declarations shared by the libntb200 translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/ntb200.h"

namespace ntb {

// Thread-local error text; returns `code` so call sites can `return fail(...)`.
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);
void note_launch(int n = 1);

// Number of SMs of the current device (cached per device).
int sm_count();

// Check the last launch and return NTB_OK / NTB_ERR_CUDA.
int check_launch(const char* what, int path = -1);

// Per-family unpacked arguments (element strides).
struct Tensor1 { void* p; int64_t n, s; };
struct Tensor2 { void* p; int64_t n0, n1, s0, s1; };

struct LaunchArgs {
  int kernel, dtype;
  void* const* ptrs; int n_ptrs;
  const double* scalars; int n_scalars;
  const int64_t* sizes; const int64_t* strides; const int* ranks;
  const int64_t* meta; int n_meta;
  cudaStream_t stream;
  // offsets of each tensor param's sizes/strides in the flat arrays
  int64_t base[8];
};

int launch_elementwise(const LaunchArgs& a);   // add, silu
int launch_rowwise(const LaunchArgs& a);       // softmax, rms_norm
int launch_rope(const LaunchArgs& a);
int launch_gemm(const LaunchArgs& a);          // mm, bmm, addmm
int launch_conv2d(const LaunchArgs& a);
int launch_sdpa(const LaunchArgs& a);
int launch_sdpa_rope(const LaunchArgs& a);

// Device workspace (grown on demand, stream-ordered use only).
void* workspace(size_t bytes, cudaStream_t s);

}  // namespace ntb
