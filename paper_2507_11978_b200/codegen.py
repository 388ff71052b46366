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

Supported application IR: Let / Assign / Accumulate / Store at the top level;
Load with constant nest indices; + - * / max min; exp, sqrt, rsqrt, log,
sigmoid, neg, abs, tanh, relu; numeric constants; ShapeOf; Zeros; Reduce
(max / sum) over the WHOLE tile (every other lane axis of extent 1, e.g.
softmax / rms_norm-style rows).  Loops (ForRange) and Dot are not generated:
those families have native tensor-core kernels, and anything else raises
UnsupportedSpecError with the reason.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass

from . import symbolic as se
from .arrange import Grid
from .spec import (Accumulate, Assign, BinOp, ConstF, Dot, ForRange, IConst, Let, Load, Local,
                   Reduce, ShapeOf, Store, UnOp, Zeros)


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
    maps = {p.name: checked.index_maps[p.name] for p in tensors}

    def ev(e) -> int:
        return int(se.evaluate(se.from_any(e), binding))

    # lane universe: per-axis maximum; each parameter is 1 or the maximum there
    ndim = {len(m.lane_sizes) for m in maps.values()}
    if len(ndim) != 1:
        raise CodegenError("parameters with lane tiles of different rank")
    nd = ndim.pop()
    ext = {n: [ev(s) for s in m.lane_sizes] for n, m in maps.items()}
    uni = [max(ext[n][j] for n in ext) for j in range(nd)]
    for n, e in ext.items():
        for j in range(nd):
            if e[j] not in (1, uni[j]):
                raise CodegenError(f"lane tile of {n!r} ({e}) does not broadcast to {uni}")
    lane_total = math.prod(uni) if uni else 1
    if lane_total < 1:
        raise CodegenError("empty lane tile")
    block = 32 * min(8, max(1, math.ceil(lane_total / 32)))
    per_thread = math.ceil(lane_total / block)
    if per_thread > 64:
        raise CodegenError(f"lane tile of {lane_total} elements is too large for one CTA")

    # statement kinds (element vs whole-tile scalar) ---------------------------
    kind: dict = {}

    def ekind(x) -> str:
        if isinstance(x, Load):
            for n in x.nests:
                if not isinstance(n, IConst):
                    raise CodegenError("loads with loop-variable nest indices are not generated")
            return "scalar" if spec.param(x.param).rank == 0 else "elem"
        if isinstance(x, Local):
            return kind[x.name]
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
            if any(uni[j] != 1 for j in range(nd) if j != x.axis):
                raise CodegenError("only whole-tile reductions are generated")
            ekind(x.a)
            return "scalar"
        if isinstance(x, Dot):
            raise CodegenError("dot products run on the native tensor-core kernels only")
        raise CodegenError(f"expression {type(x).__name__}")

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

    body = []
    tmp = [0]

    def fresh():
        tmp[0] += 1
        return f"t{tmp[0]}"

    def load_code(x: Load, e: str) -> str:
        """Emit the offset/mask/load of element ``e`` of parameter x.param; returns the
        float variable holding the value."""
        m = maps[x.param]
        nests = {f"nest_{k}": int(n.value) for k, n in enumerate(x.nests)}
        bcast = ext[x.param]

        def sym(name):
            if name.startswith("lane_"):
                j = int(name[5:])
                return "((i64)0)" if bcast[j] == 1 and uni[j] != 1 else f"L{j}_{e}"
            if name.startswith("nest_"):
                return f"((i64){nests.get(name, 0)}LL)"
            return gsym(name)

        v = fresh()
        off = _render(m.offset, sym)
        conds = [f"(({_render(lhs, sym)}) >= 0 && ({_render(lhs, sym)}) < ({_render(b, sym)}))"
                 for lhs, b in m.mask]
        mask = " && ".join(conds) if conds else "true"
        pi = [t.name for t in tensors].index(x.param)
        body.append(f"  float {v} = ({mask}) ? to_f(p{pi}[{off}]) : {float(x.other)!r}f;"
                    .replace("inff", "INFINITY").replace("-INFINITY", "(-INFINITY)"))
        return v

    def expr(x, e: str) -> str:
        """C float expression of x at element index variable e (elem) or scalar."""
        if isinstance(x, Load):
            if spec.param(x.param).rank == 0:
                return f"s_{x.param}"
            return load_code(x, e)
        if isinstance(x, Local):
            return f"v_{x.name}[{e}]" if kind[x.name] == "elem" else f"v_{x.name}"
        if isinstance(x, ConstF):
            v = float(x.value)
            if math.isinf(v):
                return "(-INFINITY)" if v < 0 else "INFINITY"
            return f"{v!r}f"
        if isinstance(x, Zeros):
            return "0.0f"
        if isinstance(x, ShapeOf):
            m = maps[x.param]
            if x.of == "source":
                return f"((float){gsym(f'{x.param}_size_{x.dim}')})"
            if x.of == "nest":
                return f"{float(ev(m.nest_sizes[x.dim]))!r}f"
            return f"{float(ev(m.lane_sizes[x.dim]))!r}f"
        if isinstance(x, BinOp):
            return _BIN[x.op].format(a=expr(x.a, e), b=expr(x.b, e))
        if isinstance(x, UnOp):
            return _UN[x.op].format(a=expr(x.a, e))
        raise CodegenError(f"expression {type(x).__name__}")

    def elem_loop(stmt_fn):
        body.append(f"  #pragma unroll\n  for (int e = 0; e < E; ++e) {{")
        body.append("    if (!V[e]) continue;")
        stmt_fn("e")
        body.append("  }")

    def reduce_code(x: Reduce) -> str:
        r = fresh()
        ident = "(-INFINITY)" if x.op == "max" else "0.0f"
        comb = "fmaxf({a}, {b})" if x.op == "max" else "({a} + {b})"
        body.append(f"  float {r} = {ident};")
        saved = len(body)
        elem_loop(lambda e: body.append(
            f"    {r} = {comb.format(a=r, b=expr(x.a, e))};"))
        del saved
        body.append(f"  {r} = block_reduce_{x.op}({r}, red);")
        return r

    def scalar_expr(x) -> str:
        """Scalar-kind expression: reductions evaluated first."""
        if isinstance(x, Reduce):
            return reduce_code(x)
        if isinstance(x, BinOp):
            return _BIN[x.op].format(a=scalar_expr(x.a), b=scalar_expr(x.b))
        if isinstance(x, UnOp):
            return _UN[x.op].format(a=scalar_expr(x.a))
        return expr(x, "0")

    def hoist(x):
        """Replace whole-tile reductions inside an element expression by scalars."""
        if isinstance(x, Reduce):
            return Local(_hoisted(x))
        if isinstance(x, BinOp):
            return BinOp(x.op, hoist(x.a), hoist(x.b))
        if isinstance(x, UnOp):
            return UnOp(x.op, hoist(x.a))
        return x

    def _hoisted(x):
        name = fresh()
        body.append(f"  const float v_{name} = {reduce_code(x)};")
        kind[name] = "scalar"
        return name

    stored = set()
    for st in spec.application:
        if isinstance(st, ForRange):
            raise CodegenError("loops (ForRange) are not generated")
        if isinstance(st, (Let, Assign, Accumulate)):
            k = ekind(st.expr)
            if isinstance(st, Let):
                kind[st.name] = k
                if k == "elem":
                    body.append(f"  float v_{st.name}[E];")
            elif st.name not in kind:
                raise CodegenError(f"assignment to undefined local {st.name!r}")
            elif kind[st.name] == "scalar" and k == "elem":
                raise CodegenError(f"local {st.name!r} changes from tile-scalar to element-wise")
            x = hoist(st.expr)
            if isinstance(st, Accumulate):
                x = BinOp("+", Local(st.name), x)
            if kind[st.name] == "elem":
                name = st.name
                elem_loop(lambda e: body.append(f"    v_{name}[{e}] = {expr(x, e)};"))
            else:
                decl = "float " if isinstance(st, Let) else ""
                body.append(f"  {decl}v_{st.name} = {scalar_expr(x)};")
        elif isinstance(st, Store):
            m = maps[st.param]
            for n in st.nests:
                if not isinstance(n, IConst):
                    raise CodegenError("stores with loop-variable nest indices are not generated")
            ekind(st.expr)
            x = hoist(st.expr)
            nests = {f"nest_{k}": int(n.value) for k, n in enumerate(st.nests)}
            bcast = ext[st.param]
            pi = [t.name for t in tensors].index(st.param)

            def sym(name, nests=nests, bcast=bcast):
                if name.startswith("lane_"):
                    j = int(name[5:])
                    return "((i64)0)" if bcast[j] == 1 and uni[j] != 1 else f"L{j}_e"
                if name.startswith("nest_"):
                    return f"((i64){nests.get(name, 0)}LL)"
                return gsym(name)

            off = _render(m.offset, sym)
            conds = [f"(({_render(lhs, sym)}) >= 0 && ({_render(lhs, sym)}) < ({_render(b, sym)}))"
                     for lhs, b in m.mask]
            mask = " && ".join(conds) if conds else "true"

            def emit_store(e, x=x, off=off, mask=mask, pi=pi):
                body.append(f"    if ({mask}) p{pi}[{off}] = from_f<T>({expr(x, e)});")

            elem_loop(emit_store)
            stored.add(st.param)
        else:
            raise CodegenError(f"statement {type(st).__name__}")

    # lane coordinates of element e of this thread (row-major in the universe)
    lane_decode = []
    for e in range(per_thread):
        lane_decode.append(f"  const i64 li_{e} = (i64)threadIdx.x + {e * block}LL;")
        rem = f"li_{e}"
        for j in range(nd):
            inner = math.prod(uni[j + 1:]) if j + 1 < nd else 1
            lane_decode.append(f"  const i64 L{j}_{e} = ({rem} / {inner}LL) % {uni[j]}LL;")
    # the body refers to per-element lane variables as L{j}_e with e the loop
    # index: materialise them through small arrays
    arrays = []
    for j in range(nd):
        arrays.append(f"  i64 Larr{j}[E] = {{{', '.join(f'L{j}_{e}' for e in range(per_thread))}}};")
    text_body = "\n".join(body)
    for j in range(nd):
        text_body = text_body.replace(f"L{j}_e", f"Larr{j}[e]")

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
        "  const i64 pid = (i64)blockIdx.x;",
        *pid_lines,
        *lane_decode,
        *arrays,
        "  bool V[E];",
        *[f"  V[{e}] = li_{e} < LANES;" for e in range(per_thread)],
        text_body,
        "}",
    ])
    if not stored:
        raise CodegenError("the application stores nothing")
    name = "ntb_generated"
    return Generated(source=src, name=name, slot_names=tuple(slot_names),
                     tensor_params=tuple(p.name for p in tensors),
                     scalar_params=tuple(p.name for p in scalars), block=block)


def source_digest(g: Generated) -> str:
    return hashlib.sha256(g.source.encode()).hexdigest()[:16]
