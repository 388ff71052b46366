// Map VM: evaluation of postfix int64 expression code with Python floor
// semantics (reference symexpr.py:127-161).  Shared by the host
// (ntb_map_enumerate / ntb_grid_eval) and the device probe kernel.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define NTB_HD __host__ __device__ __forceinline__
#else
#define NTB_HD inline
#endif

namespace ntb {

enum Op : int64_t {
  OP_CONST = 0, OP_SLOT = 1, OP_NEG = 2, OP_ADD = 3, OP_SUB = 4, OP_MUL = 5,
  OP_FLOORDIV = 6, OP_CEILDIV = 7, OP_MOD = 8, OP_MIN = 9, OP_MAX = 10
};

constexpr int kMaxStack = 64;
constexpr int kMaxSlots = 128;

NTB_HD int64_t floordiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}

NTB_HD int64_t floormod(int64_t a, int64_t b) {
  int64_t r = a % b;
  if (r != 0 && ((r < 0) != (b < 0))) r += b;
  return r;
}

// Returns 0 on success, 5 (NTB_ERR_EVAL) on zero divisor, 1 on malformed code.
NTB_HD int eval_code(const int64_t* code, int64_t len, const int64_t* slots,
                     int64_t n_slots, int64_t* out) {
  int64_t st[kMaxStack];
  int sp = 0;
  for (int64_t pc = 0; pc < len; ++pc) {
    int64_t op = code[pc];
    if (op == OP_CONST || op == OP_SLOT) {
      if (pc + 1 >= len || sp >= kMaxStack) return 1;
      int64_t v = code[++pc];
      if (op == OP_SLOT) {
        if (v < 0 || v >= n_slots) return 1;
        v = slots[v];
      }
      st[sp++] = v;
      continue;
    }
    if (op == OP_NEG) {
      if (sp < 1) return 1;
      st[sp - 1] = -st[sp - 1];
      continue;
    }
    if (sp < 2) return 1;
    int64_t b = st[--sp];
    int64_t a = st[sp - 1];
    int64_t r;
    switch (op) {
      case OP_ADD: r = a + b; break;
      case OP_SUB: r = a - b; break;
      case OP_MUL: r = a * b; break;
      case OP_FLOORDIV: if (b == 0) return 5; r = floordiv(a, b); break;
      case OP_CEILDIV: if (b == 0) return 5; r = -floordiv(-a, b); break;
      case OP_MOD: if (b == 0) return 5; r = floormod(a, b); break;
      case OP_MIN: r = a < b ? a : b; break;
      case OP_MAX: r = a > b ? a : b; break;
      default: return 1;
    }
    st[sp - 1] = r;
  }
  if (sp != 1) return 1;
  *out = st[0];
  return 0;
}

// Parsed view of a map blob (pointers into the int64 array).
struct Expr { const int64_t* code; int64_t len; };

struct ParamMap {
  int n_nest, n_lane, n_mask;
  Expr nest[8];
  Expr lane[8];
  Expr offset;
  Expr mask_lhs[8];
  Expr mask_bound[8];
};

struct Blob {
  int64_t n_slots, n_grid, n_checks, n_params;
  int64_t slot_pid;
  int64_t slot_pidc[8];
  int64_t max_nest, slot_nest[8];
  int64_t max_lane, slot_lane[8];
  Expr grid[8];
  Expr check_lhs[16], check_rhs[16];
  Expr pidc[8];
  ParamMap params[8];
};

constexpr int64_t kBlobMagic = 0x4E544231;

// Returns 0 on success, 1 on a malformed blob.
NTB_HD int parse_blob(const int64_t* b, int64_t n, Blob* out) {
  int64_t p = 0;
#define NTB_TAKE(dst) do { if (p >= n) return 1; (dst) = b[p++]; } while (0)
#define NTB_EXPR(dst) do { int64_t L_; NTB_TAKE(L_); if (L_ < 0 || p + L_ > n) return 1; \
    (dst).code = b + p; (dst).len = L_; p += L_; } while (0)
  int64_t magic;
  NTB_TAKE(magic);
  if (magic != kBlobMagic) return 1;
  NTB_TAKE(out->n_slots);
  NTB_TAKE(out->n_grid);
  NTB_TAKE(out->n_checks);
  NTB_TAKE(out->n_params);
  if (out->n_grid < 1 || out->n_grid > 8 || out->n_checks < 0 || out->n_checks > 16 ||
      out->n_params < 0 || out->n_params > 8 || out->n_slots > kMaxSlots)
    return 1;
  NTB_TAKE(out->slot_pid);
  for (int i = 0; i < out->n_grid; ++i) NTB_TAKE(out->slot_pidc[i]);
  NTB_TAKE(out->max_nest);
  if (out->max_nest < 0 || out->max_nest > 8) return 1;
  for (int i = 0; i < out->max_nest; ++i) NTB_TAKE(out->slot_nest[i]);
  NTB_TAKE(out->max_lane);
  if (out->max_lane < 0 || out->max_lane > 8) return 1;
  for (int i = 0; i < out->max_lane; ++i) NTB_TAKE(out->slot_lane[i]);
  for (int i = 0; i < out->n_grid; ++i) NTB_EXPR(out->grid[i]);
  for (int i = 0; i < out->n_checks; ++i) { NTB_EXPR(out->check_lhs[i]); NTB_EXPR(out->check_rhs[i]); }
  for (int i = 0; i < out->n_grid; ++i) NTB_EXPR(out->pidc[i]);
  for (int q = 0; q < out->n_params; ++q) {
    ParamMap& m = out->params[q];
    int64_t v;
    NTB_TAKE(v); m.n_nest = (int)v;
    NTB_TAKE(v); m.n_lane = (int)v;
    if (m.n_nest < 0 || m.n_nest > out->max_nest || m.n_lane < 0 || m.n_lane > out->max_lane)
      return 1;
    for (int i = 0; i < m.n_nest; ++i) NTB_EXPR(m.nest[i]);
    for (int i = 0; i < m.n_lane; ++i) NTB_EXPR(m.lane[i]);
    NTB_EXPR(m.offset);
    NTB_TAKE(v); m.n_mask = (int)v;
    if (m.n_mask < 0 || m.n_mask > 8) return 1;
    for (int i = 0; i < m.n_mask; ++i) { NTB_EXPR(m.mask_lhs[i]); NTB_EXPR(m.mask_bound[i]); }
  }
#undef NTB_TAKE
#undef NTB_EXPR
  return p == n ? 0 : 1;
}

// Evaluate the point `linear` (row-major over pid, nest..., lane...) of
// parameter `q`.  `slots` is a scratch copy the function mutates.
NTB_HD int eval_point(const Blob& B, int q, int64_t linear, const int64_t* nest_ext,
                      const int64_t* lane_ext, int64_t* slots, int64_t* off, uint8_t* mask) {
  const ParamMap& m = B.params[q];
  int64_t rest = linear;
  for (int j = m.n_lane - 1; j >= 0; --j) {
    slots[B.slot_lane[j]] = rest % lane_ext[j];
    rest /= lane_ext[j];
  }
  for (int k = m.n_nest - 1; k >= 0; --k) {
    slots[B.slot_nest[k]] = rest % nest_ext[k];
    rest /= nest_ext[k];
  }
  slots[B.slot_pid] = rest;
  int rc;
  for (int i = 0; i < B.n_grid; ++i) {
    int64_t v;
    rc = eval_code(B.pidc[i].code, B.pidc[i].len, slots, B.n_slots, &v);
    if (rc) return rc;
    slots[B.slot_pidc[i]] = v;
  }
  rc = eval_code(m.offset.code, m.offset.len, slots, B.n_slots, off);
  if (rc) return rc;
  uint8_t ok = 1;
  for (int i = 0; i < m.n_mask; ++i) {
    int64_t l, bnd;
    rc = eval_code(m.mask_lhs[i].code, m.mask_lhs[i].len, slots, B.n_slots, &l);
    if (rc) return rc;
    rc = eval_code(m.mask_bound[i].code, m.mask_bound[i].len, slots, B.n_slots, &bnd);
    if (rc) return rc;
    ok = ok && l >= 0 && l < bnd;   // sim.py _offsets_and_mask: (lhs >= 0) & (lhs < bound)
  }
  *mask = ok;
  return 0;
}

}  // namespace ntb
