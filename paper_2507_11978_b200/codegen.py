"""Generic path: CUDA C++ generated from a CheckedSpec, compiled with NVRTC.

SURVEY 8(f) rank 4.  Specs that match none of the native sm_100a kernel
families (backend._family_of) used to end in UnsupportedSpecError; this
module prints them as a CUDA kernel instead - the role the reference's
``emit_triton`` (emit.py:72-314) plays for Triton - and the C ABI
(``ntb_jit_compile`` / ``ntb_jit_launch``, csrc/ntb_jit.cu) compiles it for
sm_100a and launches it.  There is no CPU path.

Execution model (one CTA per program, the reference's program = one tile):

* the 1-D grid is decoded exactly like the reference launcher
  (emit.py:164-166): ``pid_i`` from ``blockIdx.x`` by ``Grid.pid_components``;
* the lane tile of the program is spread over the CTA's threads, ``E``
  elements per thread; ``lane_j`` are the row-major coordinates of an
  element inside the tile (a parameter whose tile is 1 along a lane axis
  sees ``lane_j = 0`` there: the reference's broadcast);
* every load / store uses the parameter's own lowered IndexMap: ``offset``
  (elements) and the mask ``AND (idx >= 0) & (idx < bound)`` (sim.py:249-266);
  masked loads yield the load's fill value, masked stores are dropped;
* integer map arithmetic is int64 with the reference's FLOOR ``//`` and
  ``%`` (symexpr.py:31-161), float math is fp32, loads/stores convert from /
  to the tensor dtype (f32, f16, bf16).

Supported application IR: Store at the top level (the reference forbids
stores in loops, tileir.py:425-426), Let / Assign / Accumulate anywhere; ``for`` loops over a nest (ForRange) with loads indexed by the loop
variable or constants; + - * / max min; exp, sqrt, rsqrt, log, sigmoid, neg,
abs, tanh, relu; numeric constants; ShapeOf; Zeros; Reduce (max / sum) over
the WHOLE tile (every other lane axis of extent 1, e.g. softmax / rms_norm-
style rows: element-wise partials + one block reduction) or along ONE axis of
any loaded tile (results in shared memory, one warp per result element,
broadcast back with the reference's right-aligned numpy rules, e.g. row sums
of a (BM, BN) tile stored as (BM,), or x - max(x, axis=0)); Dot of two (transposed) 2-D operand tiles into the 2-D output
tile - both operands staged in shared memory, fp32 FMA accumulation on the
CUDA cores (the paper's contractions run on the native tcgen05 kernels; this
is the path for OTHER contractions, e.g. a matmul with a fused epilogue).
Anything else raises UnsupportedSpecError with the reason.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass

from . import symbolic as se
from .arrange import Grid
from .spec import (Accumulate, Assign, BinOp, ConstF, Dot, ForRange, IConst, Let, Load, Local,
                   Reduce, ShapeOf, Store, UnOp, Var, Zeros)


class CodegenError(Exception):
    """The spec is outside what the generic path generates."""


_BIN = {"+": "({a} + {b})", "-": "({a} - {b})", "*": "({a} * {b})", "/": "({a} / {b})",
        "max": "fmaxf({a}, {b})", "min": "fminf({a}, {b})"}
_UN = {"exp": "__expf({a})", "sqrt": "sqrtf({a})", "rsqrt": "rsqrtf({a})", "log": "__logf({a})",
       "sigmoid": "(1.0f / (1.0f + __expf(-({a}))))", "neg": "(-({a}))", "abs": "fabsf({a})",
       "tanh": "tanhf({a})", "relu": "fmaxf({a}, 0.0f)"}
_CT = {0: "float", 1: "__half", 2: "__nv_bfloat16"}

PRELUDE = r"""
#include <cuda_fp16.h>
#include <cuda_bf16.h>
typedef long long i64;
#ifndef INFINITY
#define INFINITY __int_as_float(0x7f800000)
#endif
__device__ __forceinline__ i64 fdiv(i64 a, i64 b) {
  i64 q = a / b; return (q * b != a && ((a < 0) != (b < 0))) ? q - 1 : q;
}
__device__ __forceinline__ i64 fmodp(i64 a, i64 b) {
  i64 r = a % b; return (r != 0 && ((r < 0) != (b < 0))) ? r + b : r;
}
__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__half v) { return __half2float(v); }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ __half from_f<__half>(float v) { return __float2half_rn(v); }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}
"""


def _render(e, sym) -> str:
    """int64 C expression of a map expression; ``sym(name)`` renders a symbol."""
    def walk(n):
        k = n[0]
        if k == "const":
            return f"((i64){n[1]}LL)"
        if k == "sym":
            return sym(n[1])
        if k == "neg":
            return f"(-{walk(n[1])})"
        a, b = walk(n[1]), walk(n[2])
        if k == "add":
            return f"({a} + {b})"
        if k == "sub":
            return f"({a} - {b})"
        if k == "mul":
            return f"({a} * {b})"
        if k == "floordiv":
            return f"fdiv({a}, {b})"
        if k == "ceildiv":
            return f"(-fdiv(-({a}), {b}))"
        if k == "mod":
            return f"fmodp({a}, {b})"
        if k == "min":
            return f"min({a}, {b})"
        if k == "max":
            return f"max({a}, {b})"
        raise CodegenError(f"map expression node {k!r}")
    return walk(se.from_any(e).node)


@dataclass
class Generated:
    source: str
    name: str
    slot_names: tuple        # order of the int64 slot array argument
    tensor_params: tuple     # pointer arguments, in order
    scalar_params: tuple     # float arguments, in order
    block: int


def generate(checked, binding: dict, dtype: int) -> Generated:
    """CUDA source for ``checked`` specialised to the lane-tile extents and
    meta values of ``binding`` (sizes/strides stay runtime arguments except
    where they fix a tile extent)."""
    spec = checked.spec
    tensors = [p for p in spec.params if p.rank >= 1]
    scalars = [p for p in spec.params if p.rank == 0]
    tnames = [t.name for t in tensors]
    maps = {p.name: checked.index_maps[p.name] for p in tensors}

    def ev(e) -> int:
        return int(se.evaluate(se.from_any(e), binding))

    ext = {n: [ev(s) for s in m.lane_sizes] for n, m in maps.items()}

    # the element universe is the lane tile of the stored parameter(s)
    def stores(stmts):
        for st in stmts:
            if isinstance(st, Store):
                yield st
            elif isinstance(st, ForRange):
                yield from stores(st.body)
    stored_params = [st.param for st in stores(spec.application)]
    if not stored_params:
        raise CodegenError("the application stores nothing")
    uni = ext[stored_params[0]]
    for n in stored_params:
        if ext[n] != uni:
            raise CodegenError("stored parameters with different lane tiles")
    nd = len(uni)

    def bcast_ok(n):
        e = ext[n]
        return len(e) == nd and all(e[j] in (1, uni[j]) for j in range(nd))

    lane_total = math.prod(uni) if uni else 1
    if lane_total < 1:
        raise CodegenError("empty lane tile")
    def has_reduce(x):
        if isinstance(x, Reduce):
            return True
        return any(has_reduce(c) for c in (getattr(x, "a", None), getattr(x, "b", None))
                   if c is not None and not isinstance(c, (str, int, float)))

    def stmts_reduce(stmts):
        for st in stmts:
            if isinstance(st, ForRange):
                if stmts_reduce(st.body):
                    return True
            elif has_reduce(getattr(st, "expr", None)):
                return True
        return False
    # 8 warps when the program reduces (axis reductions run one warp per result)
    block = 256 if stmts_reduce(spec.application) else \
        32 * min(8, max(1, math.ceil(lane_total / 32)))
    per_thread = math.ceil(lane_total / block)
    if per_thread > 64:
        raise CodegenError(f"lane tile of {lane_total} elements is too large for one CTA")

    slot_names = []
    for p in tensors:
        for d in range(p.rank):
            slot_names.append(f"{p.name}_size_{d}")
        for d in range(p.rank):
            slot_names.append(f"{p.name}_stride_{d}")
    slot_idx = {n: i for i, n in enumerate(slot_names)}

    def gsym(name):
        if name in spec.meta:
            return f"((i64){int(binding[name])}LL)"
        if name in slot_idx:
            return f"S.v[{slot_idx[name]}]"
        if name.startswith("pid"):
            return name
        raise CodegenError(f"symbol {name!r} in a grid / map expression")

    grid = Grid(sizes=tuple(se.from_any(s) for s in checked.grid.sizes),
                total=se.lit(1), checks=())
    pidc = grid.pid_components(se.var("pid"))

    kind: dict = {}
    loopvar: dict = {}            # IR loop variable -> C variable
    body: list = []
    shared_decls: list = []
    smem_bytes = [0]
    tmp = [0]
    ind = ["  "]

    def fresh():
        tmp[0] += 1
        return f"t{tmp[0]}"

    def emit(line):
        body.append(ind[0] + line)

    def nest_c(n):
        if isinstance(n, IConst):
            return f"((i64){int(n.value)}LL)"
        if isinstance(n, Var):
            if n.name not in loopvar:
                raise CodegenError(f"unknown loop variable {n.name!r}")
            return loopvar[n.name]
        raise CodegenError("nest index must be a constant or a loop variable")

    def map_sym(param, nests, lane_expr):
        """Renderer for the symbols of ``param``'s map: nest_k from ``nests``,
        lane_j from ``lane_expr(j)``."""
        nc = {f"nest_{k}": nest_c(n) for k, n in enumerate(nests)}

        def sym(name):
            if name.startswith("lane_"):
                return lane_expr(int(name[5:]))
            if name.startswith("nest_"):
                return nc.get(name, "((i64)0LL)")
            return gsym(name)
        return sym

    def off_mask(param, sym):
        m = maps[param]
        off = _render(m.offset, sym)
        conds = [f"(({_render(lhs, sym)}) >= 0 && ({_render(lhs, sym)}) < ({_render(b, sym)}))"
                 for lhs, b in m.mask]
        return off, (" && ".join(conds) if conds else "true")

    def fill(v):
        v = float(v)
        if math.isinf(v):
            return "(-INFINITY)" if v < 0 else "INFINITY"
        return f"{v!r}f"

    # -- tile shapes (evaluated), the reference's typecheck rules ------------
    def bcast(a, b):
        out = []
        for i in range(1, max(len(a), len(b)) + 1):
            da = a[-i] if i <= len(a) else 1
            db = b[-i] if i <= len(b) else 1
            if da != db and 1 not in (da, db):
                raise CodegenError(f"cannot broadcast {tuple(a)} with {tuple(b)}")
            out.append(db if da == 1 else da)
        return tuple(reversed(out))

    def shp(x) -> tuple:
        if isinstance(x, Load):
            return () if spec.param(x.param).rank == 0 else tuple(ext[x.param])
        if isinstance(x, Local):
            k = kind.get(x.name)
            if isinstance(k, tuple):
                return k[2]
            return tuple(uni) if k in ("elem", "elemtmp") else ()
        if isinstance(x, (ConstF, ShapeOf)):
            return ()
        if isinstance(x, Zeros):
            return tuple(ev(d) for d in x.shape)
        if isinstance(x, BinOp):
            return bcast(shp(x.a), shp(x.b))
        if isinstance(x, UnOp):
            sa = shp(x.a)
            return tuple(reversed(sa)) if x.op == "trans" else sa
        if isinstance(x, Reduce):
            sa = shp(x.a)
            return sa[: x.axis] + sa[x.axis + 1:]
        if isinstance(x, Dot):
            return tuple(uni)
        raise CodegenError(f"expression {type(x).__name__}")

    def whole_tile(x: Reduce) -> bool:
        """The operand is the element universe and every other axis is 1: a
        row reduction evaluated element-wise + one block reduction."""
        return list(shp(x.a)) == list(uni) and all(uni[j] == 1 for j in range(nd) if j != x.axis)

    def to_uni(sr) -> bool:
        """A reduction result right-aligned against the universe (numpy rules)."""
        if len(sr) > nd:
            return False
        o = nd - len(sr)
        return all(sr[d] in (1, uni[o + d]) for d in range(len(sr)))

    def check_red_operand(y):
        """Operands of axis reductions are evaluated at explicit coordinates:
        loads of any lane tile, constants, tile-uniform locals, nested
        reductions."""
        if isinstance(y, Load):
            for n in y.nests:
                nest_c(n)
            return
        if isinstance(y, Local):
            if kind.get(y.name) != "scalar":
                raise CodegenError(f"element-wise local {y.name!r} inside an axis reduction")
            return
        if isinstance(y, (ConstF, ShapeOf, Zeros)):
            return
        if isinstance(y, BinOp):
            if y.op not in _BIN:
                raise CodegenError(f"binary op {y.op!r}")
            check_red_operand(y.a)
            check_red_operand(y.b)
            return
        if isinstance(y, UnOp):
            if y.op not in _UN:
                raise CodegenError(f"unary op {y.op!r}")
            check_red_operand(y.a)
            return
        if isinstance(y, Reduce):
            if y.op not in ("max", "sum"):
                raise CodegenError(f"reduction {y.op!r}")
            check_red_operand(y.a)
            return
        raise CodegenError(f"{type(y).__name__} inside an axis reduction")

    # -- kinds ---------------------------------------------------------------
    def ekind(x) -> str:
        if isinstance(x, Load):
            if spec.param(x.param).rank == 0:
                return "scalar"
            if not bcast_ok(x.param):
                raise CodegenError(f"{x.param!r} has a lane tile {ext[x.param]} that is neither "
                                   f"the output tile {uni} nor a dot operand")
            for n in x.nests:
                nest_c(n)
            return "elem"
        if isinstance(x, Local):
            if x.name not in kind:
                raise CodegenError(f"undefined local {x.name!r}")
            k = kind[x.name]
            return "elem" if isinstance(k, tuple) else k
        if isinstance(x, (ConstF, ShapeOf)):
            return "scalar"
        if isinstance(x, Zeros):
            return "elem" if x.shape else "scalar"
        if isinstance(x, BinOp):
            if x.op not in _BIN:
                raise CodegenError(f"binary op {x.op!r}")
            return "elem" if "elem" in (ekind(x.a), ekind(x.b)) else "scalar"
        if isinstance(x, UnOp):
            if x.op not in _UN:
                raise CodegenError(f"unary op {x.op!r}")
            return ekind(x.a)
        if isinstance(x, Reduce):
            if x.op not in ("max", "sum"):
                raise CodegenError(f"reduction {x.op!r}")
            if whole_tile(x):
                ekind(x.a)
                return "scalar"
            check_red_operand(x.a)
            sr = shp(x)
            if all(d == 1 for d in sr):
                return "scalar"
            if not to_uni(sr):
                raise CodegenError(f"reduction result {sr} does not broadcast to the stored "
                                   f"tile {tuple(uni)}")
            return "elem"
        if isinstance(x, Dot):
            return "elem"
        raise CodegenError(f"expression {type(x).__name__}")

    # -- element expressions -------------------------------------------------
    def elem_lane(param):
        e = ext[param]
        return lambda j: "((i64)0)" if e[j] == 1 and uni[j] != 1 else f"Larr{j}[e]"

    def expr(x) -> str:
        """C float expression of x for element e (inside an element loop)."""
        if isinstance(x, Load):
            if spec.param(x.param).rank == 0:
                return f"s_{x.param}"
            off, mask = off_mask(x.param, map_sym(x.param, x.nests, elem_lane(x.param)))
            v = fresh()
            emit(f"  const float {v} = ({mask}) ? to_f(p{tnames.index(x.param)}[{off}]) : "
                 f"{fill(x.other)};")
            return v
        if isinstance(x, Local):
            k = kind[x.name]
            if isinstance(k, tuple):
                return red_index(k, lambda j: f"Larr{j}[e]", nd)
            return f"v_{x.name}[e]" if k == "elem" else f"v_{x.name}"
        if isinstance(x, ConstF):
            return fill(x.value)
        if isinstance(x, Zeros):
            return "0.0f"
        if isinstance(x, ShapeOf):
            m = maps[x.param]
            if x.of == "source":
                return f"((float){gsym(f'{x.param}_size_{x.dim}')})"
            if x.of == "nest":
                return f"((float){_render(m.nest_sizes[x.dim], gsym)})"
            return f"{float(ev(m.lane_sizes[x.dim]))!r}f"
        if isinstance(x, BinOp):
            return _BIN[x.op].format(a=expr(x.a), b=expr(x.b))
        if isinstance(x, UnOp):
            return _UN[x.op].format(a=expr(x.a))
        raise CodegenError(f"expression {type(x).__name__}")

    def elem_loop(fn):
        emit("#pragma unroll")
        emit("for (int e = 0; e < E; ++e) {")
        emit("  if (!V[e]) continue;")
        ind[0] += "  "
        fn()
        ind[0] = ind[0][:-2]
        emit("}")

    # -- whole-tile reductions and dot products (hoisted) --------------------
    def reduce_code(x: Reduce) -> str:
        r = fresh()
        ident = "(-INFINITY)" if x.op == "max" else "0.0f"
        comb = "fmaxf({a}, {b})" if x.op == "max" else "({a} + {b})"
        inner = hoist(x.a)
        emit(f"float {r} = {ident};")
        elem_loop(lambda: emit(f"  {r} = {comb.format(a=r, b=expr(inner))};"))
        emit(f"{r} = block_reduce_{x.op}({r}, red);")
        return r

    def red_index(k, coord, ctx_rank):
        """Element of an axis-reduction result (kind ("red", array, shape)) at
        context coordinates coord(j), right-aligned (numpy broadcasting)."""
        _, arr, sr = k
        o = ctx_rank - len(sr)
        terms = []
        for d in range(len(sr)):
            if sr[d] == 1:
                continue
            stride = math.prod(sr[d + 1:]) if d + 1 < len(sr) else 1
            terms.append(f"(int)({coord(o + d)}) * {stride}")
        return f"{arr}[{' + '.join(terms) if terms else '0'}]"

    def expr_at(y, coord, ctx) -> str:
        """C float expression of y at context coordinates coord(j) of a
        context tile of shape ctx (y broadcasts into ctx, right-aligned)."""
        if isinstance(y, Load):
            if spec.param(y.param).rank == 0:
                return f"s_{y.param}"
            e = ext[y.param]
            o = len(ctx) - len(e)
            if o < 0:
                raise CodegenError(f"{y.param!r} tile {e} inside a context tile {ctx}")
            lane = (lambda j: "((i64)0)" if e[j] == 1 else f"((i64)({coord(o + j)}))")
            off, mask = off_mask(y.param, map_sym(y.param, y.nests, lane))
            v = fresh()
            emit(f"const float {v} = ({mask}) ? to_f(p{tnames.index(y.param)}[{off}]) : "
                 f"{fill(y.other)};")
            return v
        if isinstance(y, Local):
            k = kind[y.name]
            if isinstance(k, tuple):
                return red_index(k, coord, len(ctx))
            if k != "scalar":
                raise CodegenError(f"element-wise local {y.name!r} inside an axis reduction")
            return f"v_{y.name}"
        if isinstance(y, (ConstF, Zeros, ShapeOf)):
            return expr(y)
        if isinstance(y, BinOp):
            return _BIN[y.op].format(a=expr_at(y.a, coord, ctx), b=expr_at(y.b, coord, ctx))
        if isinstance(y, UnOp):
            return _UN[y.op].format(a=expr_at(y.a, coord, ctx))
        raise CodegenError(f"{type(y).__name__} inside an axis reduction")

    def axis_reduce_code(x: Reduce):
        """Reduction along one axis of a tile that is not the element universe
        (e.g. row sums of a (BM, BN) tile stored as (BM,), or column maxima
        broadcast back over rows): the results go to shared memory, one warp
        per result element, lanes striding the reduced axis."""
        inner = hoist(x.a)          # nested reductions first
        sa = shp(inner)
        ax = x.axis
        sr = sa[:ax] + sa[ax + 1:]
        nres = math.prod(sr) if sr else 1
        if smem_bytes[0] + 4 * nres > 46 * 1024:
            raise CodegenError(f"reduction result of {nres} elements exceeds the generic path's "
                               "shared-memory budget")
        smem_bytes[0] += 4 * nres
        n = fresh()
        arr = f"R{n}"
        shared_decls.append(f"  __shared__ float {arr}[{nres}];")
        ident = "(-INFINITY)" if x.op == "max" else "0.0f"
        comb = "fmaxf({a}, {b})" if x.op == "max" else "({a} + {b})"
        shfl = "fmaxf(a_, __shfl_xor_sync(0xffffffffu, a_, o_))" if x.op == "max" else \
               "a_ + __shfl_xor_sync(0xffffffffu, a_, o_)"
        emit("__syncthreads();")
        emit(f"for (int r_ = threadIdx.x >> 5; r_ < {nres}; r_ += NT / 32) {{")
        ind[0] += "  "
        rc = []
        for d in range(len(sr)):
            stride = math.prod(sr[d + 1:]) if d + 1 < len(sr) else 1
            emit(f"const int {n}_c{d} = (r_ / {stride}) % {sr[d]};")
            rc.append(f"{n}_c{d}")
        coords = rc[:ax] + ["k_"] + rc[ax:]
        emit(f"float a_ = {ident};")
        emit(f"for (int k_ = threadIdx.x & 31; k_ < {sa[ax]}; k_ += 32) {{")
        ind[0] += "  "
        val = expr_at(inner, lambda j: coords[j], sa)
        emit(f"a_ = {comb.format(a='a_', b=val)};")
        ind[0] = ind[0][:-2]
        emit("}")
        emit(f"for (int o_ = 16; o_; o_ >>= 1) a_ = {shfl};")
        emit(f"if ((threadIdx.x & 31) == 0) {arr}[r_] = a_;")
        ind[0] = ind[0][:-2]
        emit("}")
        emit("__syncthreads();")
        return ("red", arr, tuple(sr))

    def operand(x):
        """(Load, transposed) of a dot operand."""
        if isinstance(x, UnOp) and x.op == "trans" and isinstance(x.a, Load):
            return x.a, True
        if isinstance(x, Load):
            return x, False
        raise CodegenError("dot operands must be (transposed) loads")

    def dot_code(x: Dot) -> str:
        if nd != 2:
            raise CodegenError("dot needs a 2-D output tile")
        (la, ta), (lb, tb) = operand(x.a), operand(x.b)
        ea, eb = ext[la.param], ext[lb.param]
        if len(ea) != 2 or len(eb) != 2:
            raise CodegenError("dot operands must be 2-D tiles")
        M, K = (ea[1], ea[0]) if ta else (ea[0], ea[1])
        K2, N = (eb[1], eb[0]) if tb else (eb[0], eb[1])
        if K != K2 or M != uni[0] or N != uni[1]:
            raise CodegenError(f"dot shapes {ea}{'T' if ta else ''} x {eb}{'T' if tb else ''} "
                               f"do not produce the output tile {uni}")
        elt = 4 if dtype == 0 else 2
        need = (M * K + K * N) * elt
        if smem_bytes[0] + need > 46 * 1024:
            raise CodegenError(f"dot operand tiles of {need} bytes exceed the generic path's "
                               "shared-memory budget")
        smem_bytes[0] += need
        sa, sb, t = fresh(), fresh(), fresh()
        shared_decls.append(f"  __shared__ T s{sa}[{M * K}];")
        shared_decls.append(f"  __shared__ T s{sb}[{K * N}];")

        def stage(ld, trans, rows, cols, dst):
            # dst[r * cols + c] <- operand element (r, c) (transposed view if trans)
            lane = (lambda j: "(i64)c_" if j == 0 else "(i64)r_") if trans else \
                   (lambda j: "(i64)r_" if j == 0 else "(i64)c_")
            off, mask = off_mask(ld.param, map_sym(ld.param, ld.nests, lane))
            pi = tnames.index(ld.param)
            emit(f"for (int q_ = threadIdx.x; q_ < {rows * cols}; q_ += NT) {{")
            emit(f"  const int r_ = q_ / {cols}, c_ = q_ % {cols};")
            emit(f"  s{dst}[q_] = ({mask}) ? p{pi}[{off}] : from_f<T>({fill(ld.other)});")
            emit("}")

        emit("__syncthreads();")
        stage(la, ta, M, K, sa)
        stage(lb, tb, K, N, sb)
        emit("__syncthreads();")
        emit(f"float {t}[E];")

        def comp():
            emit(f"  const int i_ = (int)Larr0[e], j_ = (int)Larr1[e];")
            emit(f"  float acc_ = 0.0f;")
            emit(f"  #pragma unroll 8")
            emit(f"  for (int k_ = 0; k_ < {K}; ++k_)")
            emit(f"    acc_ = fmaf(to_f(s{sa}[i_ * {K} + k_]), to_f(s{sb}[k_ * {N} + j_]), acc_);")
            emit(f"  {t}[e] = acc_;")
        elem_loop(comp)
        kind[t] = "elemtmp"
        return t

    def hoist(x):
        """Evaluate reductions and dots first; return an element expression."""
        if isinstance(x, Reduce):
            name = fresh()
            if whole_tile(x):
                emit(f"const float v_{name} = {reduce_code(x)};")
                kind[name] = "scalar"
                return Local(name)
            k = axis_reduce_code(x)
            if all(d == 1 for d in k[2]):
                emit(f"const float v_{name} = {k[1]}[0];")
                kind[name] = "scalar"
            else:
                kind[name] = k
            return Local(name)
        if isinstance(x, Dot):
            t = dot_code(x)
            kind[t] = "elem"
            emit(f"float* v_{t} = {t};")
            return Local(t)
        if isinstance(x, BinOp):
            return BinOp(x.op, hoist(x.a), hoist(x.b))
        if isinstance(x, UnOp):
            return UnOp(x.op, hoist(x.a))
        return x

    def scalar_expr(x) -> str:
        if isinstance(x, Reduce):
            if whole_tile(x):
                return reduce_code(x)
            return f"{axis_reduce_code(x)[1]}[0]"
        if isinstance(x, BinOp):
            return _BIN[x.op].format(a=scalar_expr(x.a), b=scalar_expr(x.b))
        if isinstance(x, UnOp):
            return _UN[x.op].format(a=scalar_expr(x.a))
        if isinstance(x, Load) and spec.param(x.param).rank == 0:
            return f"s_{x.param}"
        if isinstance(x, Local):
            return f"v_{x.name}"
        if isinstance(x, ConstF):
            return fill(x.value)
        if isinstance(x, ShapeOf):
            return expr(x)
        if isinstance(x, Zeros):
            return "0.0f"
        raise CodegenError(f"scalar expression {type(x).__name__}")

    def statements(stmts, top):
        for st in stmts:
            if isinstance(st, ForRange):
                lv = f"lv_{st.var}"
                if isinstance(st.extent, ShapeOf) and st.extent.of == "nest":
                    ext_c = _render(maps[st.extent.param].nest_sizes[st.extent.dim], gsym)
                elif isinstance(st.extent, (int, IConst)):
                    ext_c = str(int(getattr(st.extent, "value", st.extent)))
                else:
                    ext_c = _render(st.extent, gsym)
                emit(f"for (i64 {lv} = 0; {lv} < ({ext_c}); ++{lv}) {{")
                loopvar[st.var] = lv
                ind[0] += "  "
                statements(st.body, False)
                ind[0] = ind[0][:-2]
                del loopvar[st.var]
                emit("}")
            elif isinstance(st, (Let, Assign, Accumulate)):
                k = ekind(st.expr)
                if isinstance(st, Let):
                    # inside a loop the C declaration is scoped to the loop
                    # body: a fresh binding per iteration, as in the sim
                    kind[st.name] = k
                    if k == "elem":
                        emit(f"float v_{st.name}[E];")
                elif st.name not in kind:
                    raise CodegenError(f"assignment to undefined local {st.name!r}")
                elif kind[st.name] == "scalar" and k == "elem":
                    raise CodegenError(f"local {st.name!r} changes from tile-scalar to "
                                       "element-wise")
                x = hoist(st.expr)
                if isinstance(st, Accumulate):
                    x = BinOp("+", Local(st.name), x)
                if kind[st.name] == "elem":
                    name = st.name
                    elem_loop(lambda: emit(f"  v_{name}[e] = {expr(x)};"))
                else:
                    decl = "float " if isinstance(st, Let) else ""
                    emit(f"{decl}v_{st.name} = {scalar_expr(x)};")
            elif isinstance(st, Store):
                if not top:
                    raise CodegenError("stores inside loops are not generated")
                ekind(st.expr)
                x = hoist(st.expr)
                off, mask = off_mask(st.param, map_sym(st.param, st.nests, elem_lane(st.param)))
                pi = tnames.index(st.param)
                elem_loop(lambda: emit(f"  if ({mask}) p{pi}[{off}] = from_f<T>({expr(x)});"))
            else:
                raise CodegenError(f"statement {type(st).__name__}")

    statements(spec.application, True)

    # lane coordinates of element e of this thread (row-major in the universe)
    lane_decode = []
    for e in range(per_thread):
        lane_decode.append(f"  const i64 li_{e} = (i64)threadIdx.x + {e * block}LL;")
        for j in range(nd):
            inner = math.prod(uni[j + 1:]) if j + 1 < nd else 1
            lane_decode.append(f"  const i64 L{j}_{e} = (li_{e} / {inner}LL) % {uni[j]}LL;")
    arrays = [f"  const i64 Larr{j}[E] = {{{', '.join(f'L{j}_{e}' for e in range(per_thread))}}};"
              for j in range(nd)]

    ctype = _CT[dtype]
    args = [f"T* __restrict__ p{i}" for i in range(len(tensors))]
    args += [f"float s_{p.name}" for p in scalars]
    args.append("Slots S")
    pid_lines = [f"  const i64 pid_{i} = {_render(c, lambda n: 'pid' if n == 'pid' else gsym(n))};"
                 for i, c in enumerate(pidc)]
    src = "\n".join([
        PRELUDE,
        f"struct Slots {{ i64 v[{max(1, len(slot_names))}]; }};",
        f"typedef {ctype} T;",
        f"constexpr int E = {per_thread};",
        f"constexpr int NT = {block};",
        f"constexpr i64 LANES = {lane_total}LL;",
        "__device__ __forceinline__ float block_reduce_max(float v, float* red) {",
        "  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));",
        "  __syncthreads(); if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v; __syncthreads();",
        "  float r = -INFINITY; for (int i = 0; i < NT / 32; ++i) r = fmaxf(r, red[i]); return r;",
        "}",
        "__device__ __forceinline__ float block_reduce_sum(float v, float* red) {",
        "  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);",
        "  __syncthreads(); if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v; __syncthreads();",
        "  float r = 0.0f; for (int i = 0; i < NT / 32; ++i) r += red[i]; return r;",
        "}",
        f"extern \"C\" __global__ void __launch_bounds__(NT) ntb_generated({', '.join(args)}) {{",
        "  __shared__ float red[NT / 32];",
        "  (void)red;",
        *shared_decls,
        "  const i64 pid = (i64)blockIdx.x;",
        *pid_lines,
        *lane_decode,
        *arrays,
        "  bool V[E];",
        *[f"  V[{e}] = li_{e} < LANES;" for e in range(per_thread)],
        *body,
        "}",
    ])
    return Generated(source=src, name="ntb_generated", slot_names=tuple(slot_names),
                     tensor_params=tuple(tnames), scalar_params=tuple(p.name for p in scalars),
                     block=block)


def source_digest(g: Generated) -> str:
    return hashlib.sha256(g.source.encode()).hexdigest()[:16]
