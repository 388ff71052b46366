/*
 * ntb200.h - C ABI of the B200 (sm_100a) backend for the NineToothed kernel
 * set (arXiv 2507.11978).  Plain pointers, sizes and status codes; no torch
 * or C++ types cross this boundary.  Implemented by libntb200.so
 * (paper_2507_11978_b200/csrc/).
 *
 * The reference executes a CheckedSpec in two places that this library
 * replaces (see INTEGRATION.md for the bindings a maintainer would add):
 *
 *   - the emitted Triton launcher `{name}_launch(*params, *meta)`
 *       /root/reference/pkg/src/tiledsl/emit.py:267-293
 *     whose kernel-argument packing is emit.py:80-98 (pointers / scalars in
 *     parameter order, then every tensor's sizes, then its strides, then the
 *     constexpr meta) -> ntb_launch();
 *   - the CPU executor `sim.launch(checked, args, meta)`
 *       /root/reference/pkg/src/tiledsl/sim.py:163-236
 *     whose launch-time checks (sim.py:153-160), grid evaluation
 *     (sim.py:176-183) and per-parameter offset/mask maps (sim.py:185-221,
 *     249-266) are served by the map VM below (ntb_grid_eval,
 *     ntb_map_enumerate on the host; ntb_map_probe on the GPU).
 *
 * Integer semantics of the map VM follow symexpr.evaluate
 * (/root/reference/pkg/src/tiledsl/symexpr.py:127-161): Python floor
 * division and modulo, ceildiv(a, b) = -((-a) // b), zero divisor = error.
 */
#ifndef NTB200_H
#define NTB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NTB_ABI_VERSION 1

/* status codes (every entry point returns one; text via ntb_last_error) */
enum {
  NTB_OK = 0,
  NTB_ERR_ARG = 1,          /* malformed arguments / program blob          */
  NTB_ERR_CHECK = 2,        /* a recorded launch-time check failed
                               (reference LaunchError, sim.py:153-160)     */
  NTB_ERR_UNSUPPORTED = 3,  /* no sm_100a kernel for this family/dtype/shape */
  NTB_ERR_CUDA = 4,         /* CUDA runtime/driver error                   */
  NTB_ERR_EVAL = 5          /* zero divisor in a map expression
                               (reference EvalError, symexpr.py:168-173)   */
};

/* element types */
enum { NTB_F32 = 0, NTB_F16 = 1, NTB_BF16 = 2 };

/* kernel families (paper kernel set) */
enum {
  NTB_K_ADD = 1,      /* catalog.py:121-134 */
  NTB_K_SILU = 2,     /* catalog.py:137-152 */
  NTB_K_SOFTMAX = 3,  /* catalog.py:155-176 */
  NTB_K_RMS_NORM = 4, /* catalog.py:179-223 */
  NTB_K_MM = 5,       /* catalog.py:226-240 */
  NTB_K_BMM = 6,      /* catalog.py:243-257 */
  NTB_K_ADDMM = 7,    /* catalog.py:260-292 */
  NTB_K_CONV2D = 8,   /* catalog.py:295-330 */
  NTB_K_SDPA = 9,     /* builder-defined (absent upstream, catalog.py:36) */
  NTB_K_ROPE = 10,    /* builder-defined (absent upstream, catalog.py:36) */
  NTB_K_SDPA_ROPE = 11 /* sdpa(rope(q), rope(k), v) in one kernel: SURVEY 8(f) rank 1 */
};

/* ---- library ----------------------------------------------------------- */
int ntb_abi_version(void);
/* Thread-local text of the last error raised on this thread ("" if none). */
const char* ntb_last_error(void);
/* Number of kernels launched by this library since load (all threads). */
int64_t ntb_launch_count(void);

/* Launches per execution path since load (evidence of which kernel ran). */
enum {
  NTB_PATH_PROBE = 0,
  NTB_PATH_EW_VEC = 1, NTB_PATH_EW_GENERIC = 2,
  NTB_PATH_ROW_VEC = 3, NTB_PATH_ROW_GENERIC = 4,
  NTB_PATH_ROPE_VEC = 5, NTB_PATH_ROPE_GENERIC = 6,
  NTB_PATH_GEMM_TC = 7, NTB_PATH_GEMM_GENERIC = 8,
  NTB_PATH_CONV_TC = 9, NTB_PATH_CONV_GENERIC = 10,
  NTB_PATH_ATTN_TC = 11, NTB_PATH_ATTN_GENERIC = 12,
  NTB_PATH_REPACK = 13,
  NTB_PATH_ROW_STREAM = 14,
  NTB_PATH_JIT = 15,
  NTB_PATH_GEMM_TF32 = 16,  /* fp32 mm/bmm/addmm: 3xTF32 on tcgen05 */
  NTB_PATH_CONV_TF32 = 17,  /* fp32 conv2d: 3xTF32 implicit GEMM on tcgen05 */
  NTB_PATH_EW_STREAM = 18,  /* add / silu: bulk-copy (TMA) streaming kernel */
  NTB_NUM_PATHS = 19
};
int64_t ntb_path_count(int path);

/* ---- map VM: expressions ------------------------------------------------
 * An expression is postfix int64 code:
 *   0 k : push constant k      1 i : push slots[i]
 *   2 neg  3 add  4 sub  5 mul  6 floordiv  7 ceildiv  8 mod  9 min  10 max
 */
int ntb_expr_eval(const int64_t* code, int64_t code_len,
                  const int64_t* slots, int64_t n_slots, int64_t* out);

/* ---- map VM: a compiled CheckedSpec ("map blob") ------------------------
 * Layout (all int64), produced by paper_2507_11978_b200/bytecode.py:
 *   magic 0x4E544231, n_slots, n_grid, n_checks, n_params,
 *   slot_pid, slot_pid_i[n_grid], max_nest, slot_nest_k[max_nest],
 *   max_lane, slot_lane_j[max_lane],
 *   grid sizes      : n_grid   x expr
 *   checks          : n_checks x (expr lhs, expr rhs)
 *   pid components  : n_grid   x expr   (in terms of slot_pid)
 *   per parameter   : n_nest, n_lane, nest sizes (expr...), lane sizes
 *                     (expr...), offset expr, n_mask, n_mask x (lhs, bound)
 * where each "expr" is [len, code[len]].
 *
 * ntb_grid_eval: evaluates every check (NTB_ERR_CHECK on the first failure,
 * message "launch-time check failed: <lhs> = a but <rhs> = b" as in
 * sim.py:157-160 with the expressions indexed) and the grid sizes.
 */
int ntb_grid_eval(const int64_t* blob, int64_t blob_len,
                  const int64_t* slots, int64_t n_slots,
                  int64_t* grid_out, int64_t grid_cap, int64_t* n_grid_out);

/* Enumerate every (pid, nest, lane) point of parameter `param` (index into
 * the blob's parameter list) in row-major (pid, nest..., lane...) order and
 * write its flat element offset and mask bit (AND of lhs < bound,
 * emit.py:188-192).  `capacity` is the length of offs/mask; the number of
 * points is returned in *n_points (call with capacity 0 to size).        */
int ntb_map_enumerate(const int64_t* blob, int64_t blob_len, int param,
                      const int64_t* slots, int64_t n_slots,
                      int64_t* offs, uint8_t* mask, int64_t capacity,
                      int64_t* n_points);

/* Same enumeration evaluated by a GPU kernel (one thread per point) into
 * device buffers d_offs / d_mask: the on-device proof that the
 * tile-to-program and source-to-target maps are reproduced bit-exactly.  */
int ntb_map_probe(const int64_t* blob, int64_t blob_len, int param,
                  const int64_t* slots, int64_t n_slots,
                  int64_t* d_offs, uint8_t* d_mask, int64_t capacity,
                  int64_t* n_points, void* stream);

/* ---- kernel launch -------------------------------------------------------
 * Replaces the emitted launcher's kernel call (emit.py:283-291).
 *   ptrs    : device pointers of the tensor parameters, KernelSpec order
 *   scalars : rank-0 parameters by value, KernelSpec order (addmm beta,
 *             alpha; emit.py:84-85)
 *   sizes / strides : concatenated per tensor parameter, element units
 *   ranks   : rank of each tensor parameter
 *   meta    : constexpr meta values, KernelSpec.meta order
 * Caller owns all buffers (outputs preallocated).  Launches
 * asynchronously on `stream` (a cudaStream_t; NULL = legacy default).     */
int ntb_launch(int kernel, int dtype,
               void* const* ptrs, int n_ptrs,
               const double* scalars, int n_scalars,
               const int64_t* sizes, const int64_t* strides,
               const int* ranks,
               const int64_t* meta, int n_meta,
               void* stream);

/* ---- generic path --------------------------------------
 * Specs that match no native family are printed as CUDA C++ by the host front
 * end (codegen.py; replaces the reference's Triton emitter, emit.py:72-314) and
 * compiled here with NVRTC for sm_100a.  Handles are cached per (source,
 * device).  Errors: NTB_ERR_UNSUPPORTED (no NVRTC / compile error, text in
 * ntb_last_error), NTB_ERR_CUDA, NTB_ERR_ARG. */
int ntb_jit_compile(const char* source, const char* kernel_name, int64_t* handle_out);
/* grid3 / block3: launch dims; args: cuLaunchKernel-style pointers to each
 * kernel argument; stream: cudaStream_t or NULL. */
int ntb_jit_launch(int64_t handle, const int64_t* grid3, const int64_t* block3, void** args,
                   void* stream);

/* Device scratch used by ntb_launch (conv2d's repacked filter), kept per
 * (device, stream).  A buffer used while a stream is captured into a CUDA
 * graph stays allocated until this call, so calling it invalidates graphs
 * captured over conv2d; re-capture them afterwards.                       */
int ntb_release_workspace(void);

#ifdef __cplusplus
}
#endif
#endif /* NTB200_H */
