// Generic path for specs outside the native kernel families (SURVEY 8(f)
// rank 4): the host front end (paper_2507_11978_b200/codegen.py) prints a
// CheckedSpec's grid decode, index maps and application IR as CUDA C++; this
// layer compiles it with NVRTC for sm_100a, loads the cubin through the
// driver API and launches it.  It replaces the reference's Triton emitter +
// Triton JIT pair (emit.py:72-314) for non-catalog kernels.  No CPU path:
// a missing NVRTC or a failed compile is an error.
//
// NVRTC is opened with dlopen and the driver entry points come from
// cudaGetDriverEntryPoint (no -lnvrtc / -lcuda link dependency); compiled
// modules are cached per (source, device) behind a mutex.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "ntb_internal.h"

namespace ntb {
namespace {

typedef int nvrtcResult_t;
typedef struct _nvrtcProgram* nvrtcProgram_t;
struct Nvrtc {
  nvrtcResult_t (*create)(nvrtcProgram_t*, const char*, const char*, int, const char* const*,
                          const char* const*);
  nvrtcResult_t (*compile)(nvrtcProgram_t, int, const char* const*);
  nvrtcResult_t (*log_size)(nvrtcProgram_t, size_t*);
  nvrtcResult_t (*log)(nvrtcProgram_t, char*);
  nvrtcResult_t (*cubin_size)(nvrtcProgram_t, size_t*);
  nvrtcResult_t (*cubin)(nvrtcProgram_t, char*);
  nvrtcResult_t (*destroy)(nvrtcProgram_t*);
  bool ok = false;
};

static Nvrtc* nvrtc_load() {
  static Nvrtc n;
  const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"};
  void* h = nullptr;
  for (const char* nm : names)
    if ((h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
  if (!h) return nullptr;
  n.create = (decltype(n.create))dlsym(h, "nvrtcCreateProgram");
  n.compile = (decltype(n.compile))dlsym(h, "nvrtcCompileProgram");
  n.log_size = (decltype(n.log_size))dlsym(h, "nvrtcGetProgramLogSize");
  n.log = (decltype(n.log))dlsym(h, "nvrtcGetProgramLog");
  n.cubin_size = (decltype(n.cubin_size))dlsym(h, "nvrtcGetCUBINSize");
  n.cubin = (decltype(n.cubin))dlsym(h, "nvrtcGetCUBIN");
  n.destroy = (decltype(n.destroy))dlsym(h, "nvrtcDestroyProgram");
  n.ok = n.create && n.compile && n.log_size && n.log && n.cubin_size && n.cubin && n.destroy;
  return n.ok ? &n : nullptr;
}

struct Driver {
  CUresult (*load)(CUmodule*, const void*);
  CUresult (*getfn)(CUfunction*, CUmodule, const char*);
  CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                     unsigned, CUstream, void**, void**);
  bool ok = false;
};

static Driver* driver_load() {
  static Driver d;
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  if (cudaGetDriverEntryPoint("cuModuleLoadData", &p, cudaEnableDefault, &q) == cudaSuccess && p)
    d.load = (decltype(d.load))p;
  p = nullptr;
  if (cudaGetDriverEntryPoint("cuModuleGetFunction", &p, cudaEnableDefault, &q) == cudaSuccess && p)
    d.getfn = (decltype(d.getfn))p;
  p = nullptr;
  if (cudaGetDriverEntryPoint("cuLaunchKernel", &p, cudaEnableDefault, &q) == cudaSuccess && p)
    d.launch = (decltype(d.launch))p;
  d.ok = d.load && d.getfn && d.launch;
  return d.ok ? &d : nullptr;
}

// Function-local statics are initialised exactly once (thread-safe under
// C++11), so two threads doing their first compile never see a half-filled
// table.
Nvrtc* nvrtc() {
  static Nvrtc* const n = nvrtc_load();
  return n;
}
Driver* driver() {
  static Driver* const d = driver_load();
  return d;
}

std::mutex g_mu;
std::map<std::pair<std::string, int>, int64_t> g_cache;   // (source+name, device) -> handle
std::vector<CUfunction> g_funcs;

}  // namespace
}  // namespace ntb

using namespace ntb;

extern "C" {

int ntb_jit_compile(const char* source, const char* kernel_name, int64_t* handle_out) {
  if (!source || !kernel_name || !handle_out) return fail(NTB_ERR_ARG, "ntb_jit_compile: null argument");
  int dev = 0;
  cudaGetDevice(&dev);
  cudaFree(nullptr);   // make sure the primary context exists for the driver calls
  const std::string key = std::string(kernel_name) + "\n" + source;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_cache.find({key, dev});
    if (it != g_cache.end()) {
      *handle_out = it->second;
      return NTB_OK;
    }
  }
  Nvrtc* nv = nvrtc();
  if (!nv) return fail(NTB_ERR_UNSUPPORTED, "ntb_jit_compile: libnvrtc.so.12 not found");
  Driver* dr = driver();
  if (!dr) return fail(NTB_ERR_CUDA, "ntb_jit_compile: driver entry points unavailable");
  nvrtcProgram_t prog = nullptr;
  if (nv->create(&prog, source, "ntb_generated.cu", 0, nullptr, nullptr) != 0)
    return fail(NTB_ERR_CUDA, "ntb_jit_compile: nvrtcCreateProgram failed");
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-default-device",
                        "-lineinfo", "--include-path=/usr/local/cuda/include"};
  const int rc = nv->compile(prog, 5, opts);
  if (rc != 0) {
    size_t n = 0;
    nv->log_size(prog, &n);
    std::string log(n, '\0');
    if (n) nv->log(prog, &log[0]);
    nv->destroy(&prog);
    return fail(NTB_ERR_UNSUPPORTED, "ntb_jit_compile: NVRTC error:\n" + log);
  }
  size_t n = 0;
  nv->cubin_size(prog, &n);
  std::string cubin(n, '\0');
  nv->cubin(prog, &cubin[0]);
  nv->destroy(&prog);
  CUmodule mod;
  CUresult e = dr->load(&mod, cubin.data());
  if (e != CUDA_SUCCESS) return fail(NTB_ERR_CUDA, "ntb_jit_compile: cuModuleLoadData failed");
  CUfunction fn;
  e = dr->getfn(&fn, mod, kernel_name);
  if (e != CUDA_SUCCESS) return fail(NTB_ERR_CUDA, "ntb_jit_compile: kernel symbol not found");
  std::lock_guard<std::mutex> lk(g_mu);
  g_funcs.push_back(fn);
  const int64_t h = (int64_t)g_funcs.size() - 1;
  g_cache[{key, dev}] = h;
  *handle_out = h;
  return NTB_OK;
}

int ntb_jit_launch(int64_t handle, const int64_t* grid3, const int64_t* block3, void** args,
                   void* stream) {
  CUfunction fn;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (handle < 0 || handle >= (int64_t)g_funcs.size())
      return fail(NTB_ERR_ARG, "ntb_jit_launch: unknown handle");
    fn = g_funcs[handle];
  }
  Driver* dr = driver();
  if (!dr) return fail(NTB_ERR_CUDA, "ntb_jit_launch: driver entry points unavailable");
  if (grid3[0] < 1 || grid3[0] > 0x7FFFFFFF || grid3[1] < 1 || grid3[1] > 65535 || grid3[2] < 1 ||
      grid3[2] > 65535 || block3[0] * block3[1] * block3[2] > 1024)
    return fail(NTB_ERR_ARG, "ntb_jit_launch: grid / block out of range");
  CUresult e = dr->launch(fn, (unsigned)grid3[0], (unsigned)grid3[1], (unsigned)grid3[2],
                          (unsigned)block3[0], (unsigned)block3[1], (unsigned)block3[2], 0,
                          (CUstream)stream, args, nullptr);
  if (e != CUDA_SUCCESS) return fail(NTB_ERR_CUDA, "ntb_jit_launch: cuLaunchKernel failed");
  return check_launch("generated kernel", NTB_PATH_JIT);
}

}  // extern "C"
