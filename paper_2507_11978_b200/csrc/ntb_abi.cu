// libntb200: C ABI entry points, error plumbing, map VM host side and the
// GPU map probe.  See include/ntb200.h for the contract.
#include <cuda_runtime.h>
#include <stdio.h>

#include <atomic>
#include <mutex>
#include <map>
#include <vector>
#include <utility>
#include <string>

#include "mapvm.cuh"
#include "ntb_internal.h"

namespace ntb {

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};
static std::atomic<int64_t> g_paths[NTB_NUM_PATHS];

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return NTB_ERR_CUDA;
}

void note_launch(int n) { g_launches += n; }

int check_launch(const char* what, int path) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, what);
  note_launch();
  if (path >= 0 && path < NTB_NUM_PATHS) g_paths[path]++;
  return NTB_OK;
}

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : 148;
  }
  return cached[dev];
}

// Library-owned scratch (conv's repacked filter) is kept PER STREAM: within a
// stream, reuse is ordered by the stream; two streams never share a buffer.
// Eager growth frees the old buffer after a sync of its stream.  A buffer
// handed out while the stream is being CAPTURED into a CUDA graph is baked
// into that graph, so it is "pinned": it is never freed on growth (only
// retired, still allocated) and lives until ntb_release_workspace(), which
// therefore invalidates any graph captured over a workspace-using kernel.
// Growth during a capture allocates a fresh buffer (in relaxed capture mode
// for this thread: cudaMalloc is not a stream operation) instead of handing
// out another stream's buffer.  Graphs captured on the same stream share its
// buffer: replay them in order on one stream, not concurrently.
struct Ws {
  void* p = nullptr;
  size_t bytes = 0;
  bool pinned = false;
};
static std::mutex g_ws_mu;
// keyed by (device, stream): the legacy default stream is per device
static std::map<std::pair<int, cudaStream_t>, Ws> g_ws;
static std::vector<std::pair<int, void*>> g_ws_retired;

void* workspace(size_t bytes, cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_ws_mu);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cap);
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  Ws& w = g_ws[{dev, s}];
  if (bytes <= w.bytes) {
    w.pinned = w.pinned || capturing;
    return w.p;
  }
  if (w.p) {
    if (w.pinned || capturing) {
      g_ws_retired.emplace_back(dev, w.p);   // a graph (or in-flight work) may hold it
    } else {
      cudaStreamSynchronize(s);
      cudaFree(w.p);
    }
  }
  w = Ws{};
  void* p = nullptr;
  cudaError_t e;
  if (capturing) {
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    cudaThreadExchangeStreamCaptureMode(&mode);
    e = cudaMalloc(&p, bytes);
    cudaThreadExchangeStreamCaptureMode(&mode);
  } else {
    e = cudaMalloc(&p, bytes);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  w.p = p;
  w.bytes = bytes;
  w.pinned = capturing;
  return w.p;
}

// ---- GPU probe: one thread per (pid, nest, lane) point -------------------
__global__ void map_probe_kernel(const int64_t* blob, int64_t blob_len, int q,
                                 const int64_t* slots_in, int64_t n_slots,
                                 const int64_t* nest_ext, const int64_t* lane_ext,
                                 int64_t n_points, int64_t* offs, uint8_t* mask,
                                 int* status) {
  __shared__ Blob B;
  __shared__ int parse_rc;
  if (threadIdx.x == 0) parse_rc = parse_blob(blob, blob_len, &B);
  __syncthreads();
  if (parse_rc) {
    if (threadIdx.x == 0) atomicMax(status, 1);
    return;
  }
  int64_t slots[kMaxSlots];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_points;
       i += (int64_t)gridDim.x * blockDim.x) {
    for (int64_t s = 0; s < n_slots; ++s) slots[s] = slots_in[s];
    int64_t off = 0;
    uint8_t m = 0;
    int rc = eval_point(B, q, i, nest_ext, lane_ext, slots, &off, &m);
    if (rc) atomicMax(status, rc);
    offs[i] = off;
    mask[i] = m;
  }
}

}  // namespace ntb

using namespace ntb;

extern "C" {

int ntb_abi_version(void) { return NTB_ABI_VERSION; }

const char* ntb_last_error(void) { return g_err.c_str(); }

int64_t ntb_launch_count(void) { return g_launches.load(); }

int64_t ntb_path_count(int path) {
  if (path < 0 || path >= NTB_NUM_PATHS) return -1;
  return g_paths[path].load();
}

int ntb_expr_eval(const int64_t* code, int64_t code_len, const int64_t* slots,
                  int64_t n_slots, int64_t* out) {
  if (!code || !out || (n_slots > 0 && !slots)) return fail(NTB_ERR_ARG, "null argument");
  int rc = eval_code(code, code_len, slots, n_slots, out);
  if (rc == NTB_ERR_EVAL) return fail(rc, "division or modulo by zero");
  if (rc) return fail(NTB_ERR_ARG, "malformed expression code");
  return NTB_OK;
}

static int parse_checked(const int64_t* blob, int64_t blob_len, int64_t n_slots, Blob* B) {
  if (!blob) return fail(NTB_ERR_ARG, "null map blob");
  if (parse_blob(blob, blob_len, B)) return fail(NTB_ERR_ARG, "malformed map blob");
  if (n_slots < B->n_slots) return fail(NTB_ERR_ARG, "binding shorter than the blob's slot count");
  return NTB_OK;
}

static int eval_or_fail(const Expr& e, const int64_t* slots, int64_t n_slots, int64_t* v,
                        const char* what) {
  int rc = eval_code(e.code, e.len, slots, n_slots, v);
  if (rc == NTB_ERR_EVAL) return fail(rc, std::string(what) + ": division or modulo by zero");
  if (rc) return fail(NTB_ERR_ARG, std::string(what) + ": malformed expression code");
  return NTB_OK;
}

int ntb_grid_eval(const int64_t* blob, int64_t blob_len, const int64_t* slots, int64_t n_slots,
                  int64_t* grid_out, int64_t grid_cap, int64_t* n_grid_out) {
  Blob B;
  int rc = parse_checked(blob, blob_len, n_slots, &B);
  if (rc) return rc;
  for (int i = 0; i < B.n_checks; ++i) {
    int64_t l, r;
    if ((rc = eval_or_fail(B.check_lhs[i], slots, n_slots, &l, "launch check"))) return rc;
    if ((rc = eval_or_fail(B.check_rhs[i], slots, n_slots, &r, "launch check"))) return rc;
    if (l != r) {
      char buf[160];
      snprintf(buf, sizeof buf, "launch-time check %d failed: lhs = %lld but rhs = %lld", i,
               (long long)l, (long long)r);
      return fail(NTB_ERR_CHECK, buf);
    }
  }
  if (n_grid_out) *n_grid_out = B.n_grid;
  for (int i = 0; i < B.n_grid; ++i) {
    int64_t g;
    if ((rc = eval_or_fail(B.grid[i], slots, n_slots, &g, "grid size"))) return rc;
    if (g < 1) {
      char buf[96];
      snprintf(buf, sizeof buf, "grid dimension evaluated to %lld", (long long)g);
      return fail(NTB_ERR_CHECK, buf);
    }
    if (i < grid_cap && grid_out) grid_out[i] = g;
  }
  return NTB_OK;
}

// Shared sizing for enumerate/probe: fills scratch slots with the pid
// component values unknown yet; returns extents and the point count.
static int extents(const Blob& B, int q, const int64_t* slots, int64_t n_slots,
                   int64_t* nest_ext, int64_t* lane_ext, int64_t* n_points) {
  if (q < 0 || q >= B.n_params) return fail(NTB_ERR_ARG, "parameter index out of range");
  int rc;
  int64_t total = 1;
  for (int i = 0; i < B.n_grid; ++i) {
    int64_t g;
    if ((rc = eval_or_fail(B.grid[i], slots, n_slots, &g, "grid size"))) return rc;
    if (g < 1) return fail(NTB_ERR_CHECK, "grid dimension below 1");
    total *= g;
  }
  const ParamMap& m = B.params[q];
  for (int k = 0; k < m.n_nest; ++k) {
    if ((rc = eval_or_fail(m.nest[k], slots, n_slots, &nest_ext[k], "nest extent"))) return rc;
    if (nest_ext[k] < 1) return fail(NTB_ERR_CHECK, "nest extent below 1");
    total *= nest_ext[k];
  }
  for (int j = 0; j < m.n_lane; ++j) {
    if ((rc = eval_or_fail(m.lane[j], slots, n_slots, &lane_ext[j], "lane extent"))) return rc;
    if (lane_ext[j] < 1) return fail(NTB_ERR_CHECK, "lane extent below 1");
    total *= lane_ext[j];
  }
  *n_points = total;
  return NTB_OK;
}

int ntb_map_enumerate(const int64_t* blob, int64_t blob_len, int param, const int64_t* slots,
                      int64_t n_slots, int64_t* offs, uint8_t* mask, int64_t capacity,
                      int64_t* n_points) {
  Blob B;
  int rc = parse_checked(blob, blob_len, n_slots, &B);
  if (rc) return rc;
  int64_t nest_ext[8], lane_ext[8], n = 0;
  if ((rc = extents(B, param, slots, n_slots, nest_ext, lane_ext, &n))) return rc;
  if (n_points) *n_points = n;
  if (capacity == 0) return NTB_OK;
  if (capacity < n || !offs || !mask) return fail(NTB_ERR_ARG, "output capacity too small");
  int64_t scratch[kMaxSlots];
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t s = 0; s < n_slots && s < kMaxSlots; ++s) scratch[s] = slots[s];
    rc = eval_point(B, param, i, nest_ext, lane_ext, scratch, &offs[i], &mask[i]);
    if (rc == NTB_ERR_EVAL) return fail(rc, "map point: division or modulo by zero");
    if (rc) return fail(NTB_ERR_ARG, "map point: malformed expression code");
  }
  return NTB_OK;
}

int ntb_map_probe(const int64_t* blob, int64_t blob_len, int param, const int64_t* slots,
                  int64_t n_slots, int64_t* d_offs, uint8_t* d_mask, int64_t capacity,
                  int64_t* n_points, void* stream) {
  Blob B;
  int rc = parse_checked(blob, blob_len, n_slots, &B);
  if (rc) return rc;
  if (n_slots > kMaxSlots) return fail(NTB_ERR_ARG, "too many slots");
  int64_t nest_ext[8], lane_ext[8], n = 0;
  if ((rc = extents(B, param, slots, n_slots, nest_ext, lane_ext, &n))) return rc;
  if (n_points) *n_points = n;
  if (capacity == 0) return NTB_OK;
  if (capacity < n || !d_offs || !d_mask) return fail(NTB_ERR_ARG, "output capacity too small");
  cudaStream_t s = (cudaStream_t)stream;
  // stage blob, slots and extents in one device buffer
  size_t words = (size_t)blob_len + (size_t)n_slots + 16 + 1;
  int64_t* dbuf = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&dbuf, words * sizeof(int64_t), s);
  if (e != cudaSuccess) return cuda_fail(e, "probe alloc");
  int64_t* hbuf = new int64_t[words]();
  for (int64_t i = 0; i < blob_len; ++i) hbuf[i] = blob[i];
  for (int64_t i = 0; i < n_slots; ++i) hbuf[blob_len + i] = slots[i];
  for (int k = 0; k < 8; ++k) hbuf[blob_len + n_slots + k] = nest_ext[k];
  for (int k = 0; k < 8; ++k) hbuf[blob_len + n_slots + 8 + k] = lane_ext[k];
  hbuf[words - 1] = 0;  // status word
  e = cudaMemcpyAsync(dbuf, hbuf, words * sizeof(int64_t), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  delete[] hbuf;
  if (e != cudaSuccess) return cuda_fail(e, "probe upload");
  int threads = 128;
  int64_t blocks = (n + threads - 1) / threads;
  if (blocks > 4096) blocks = 4096;
  map_probe_kernel<<<(unsigned)blocks, threads, 0, s>>>(
      dbuf, blob_len, param, dbuf + blob_len, n_slots, dbuf + blob_len + n_slots,
      dbuf + blob_len + n_slots + 8, n, d_offs, d_mask, (int*)(dbuf + words - 1));
  if ((rc = check_launch("map probe", NTB_PATH_PROBE))) return rc;
  int64_t status = 0;
  e = cudaMemcpyAsync(&status, dbuf + words - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFreeAsync(dbuf, s);
  if (e != cudaSuccess) return cuda_fail(e, "probe status");
  if (status == NTB_ERR_EVAL) return fail(NTB_ERR_EVAL, "probe: division or modulo by zero");
  if (status) return fail(NTB_ERR_ARG, "probe: malformed map blob");
  return NTB_OK;
}

int ntb_launch(int kernel, int dtype, void* const* ptrs, int n_ptrs, const double* scalars,
               int n_scalars, const int64_t* sizes, const int64_t* strides, const int* ranks,
               const int64_t* meta, int n_meta, void* stream) {
  if (n_ptrs < 1 || n_ptrs > 8 || !ptrs || !sizes || !strides || !ranks)
    return fail(NTB_ERR_ARG, "bad tensor argument arrays");
  LaunchArgs a;
  a.kernel = kernel;
  a.dtype = dtype;
  a.ptrs = ptrs;
  a.n_ptrs = n_ptrs;
  a.scalars = scalars;
  a.n_scalars = n_scalars;
  a.sizes = sizes;
  a.strides = strides;
  a.ranks = ranks;
  a.meta = meta;
  a.n_meta = n_meta;
  a.stream = (cudaStream_t)stream;
  int64_t off = 0;
  for (int i = 0; i < n_ptrs; ++i) {
    if (ranks[i] < 1 || ranks[i] > 4) return fail(NTB_ERR_ARG, "tensor rank out of range");
    a.base[i] = off;
    off += ranks[i];
    int64_t numel = 1;
    for (int d = 0; d < ranks[i]; ++d) numel *= sizes[a.base[i] + d];
    // an empty tensor (e.g. the K = 0 operands of a zero-length contraction)
    // may have a null data pointer; nothing is read from it
    if (!ptrs[i] && numel > 0) return fail(NTB_ERR_ARG, "null tensor pointer");
  }
  switch (kernel) {
    case NTB_K_ADD:
    case NTB_K_SILU: return launch_elementwise(a);
    case NTB_K_SOFTMAX:
    case NTB_K_RMS_NORM: return launch_rowwise(a);
    case NTB_K_ROPE: return launch_rope(a);
    case NTB_K_MM:
    case NTB_K_BMM:
    case NTB_K_ADDMM: return launch_gemm(a);
    case NTB_K_CONV2D: return launch_conv2d(a);
    case NTB_K_SDPA: return launch_sdpa(a);
    case NTB_K_SDPA_ROPE: return launch_sdpa_rope(a);
    default: return fail(NTB_ERR_UNSUPPORTED, "unknown kernel family");
  }
}

int ntb_release_workspace(void) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto& kv : g_ws)
    if (kv.second.p) {
      cudaSetDevice(kv.first.first);
      cudaFree(kv.second.p);
    }
  for (auto& r : g_ws_retired) {
    cudaSetDevice(r.first);
    cudaFree(r.second);
  }
  cudaSetDevice(cur);
  g_ws.clear();
  g_ws_retired.clear();
  return NTB_OK;
}

}  // extern "C"
