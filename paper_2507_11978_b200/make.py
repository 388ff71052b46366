"""The paper's front door on the B200 backend: ``make(arrangement,
application, tensors)``.

    BLOCK_SIZE = Symbol("BLOCK_SIZE", constexpr=True)

    def arrangement(input, other, output, BLOCK_SIZE=BLOCK_SIZE):
        return input.tile((BLOCK_SIZE,)), other.tile((BLOCK_SIZE,)), output.tile((BLOCK_SIZE,))

    def application(input, other, output):
        output = input + other

    kernel = make(arrangement, application, (Tensor(1), Tensor(1), Tensor(1)))
    kernel(a, b, c, BLOCK_SIZE=1024)

* ``arrangement`` runs on symbolic tensors whose meta-operations are recorded
  (tile / expand / squeeze / permute / flatten / ravel; ``t.dtype`` is the
  next level down, and assigning to it rewrites that level).
* ``application`` is NOT executed: its Python AST is compiled into the tile
  IR (spec.py).  Supported: assignment (a parameter assigned to is an
  output -> Store), ``+=`` (Accumulate), ``for k in range(t.shape[i])``,
  ``t[k]`` nest loads, ``+ - * /``, numbers, ``t.shape[i]`` and the ``ntl``
  calls ``zeros, dot, exp, sqrt, sigmoid, log, rsqrt, abs, tanh, relu, max,
  sum`` and the elementwise ``maximum, minimum``.
* The result is typechecked into a CheckedSpec and executed by
  ``backend.launch``, which matches it STRUCTURALLY (names of locals,
  parameters and the kernel itself do not matter) to one of the native
  sm_100a kernel families; anything else raises UnsupportedSpecError - the
  backend has no interpreter fallback.
"""

from __future__ import annotations

import ast
import inspect
import textwrap

from . import backend
from . import symbolic as se
from .spec import (Accumulate, ArrangeOp, BinOp, ConstF, Dot, ForRange, KernelSpec, Let, Load,
                   Local, ParamSpec, Reduce, ShapeOf, SpecError, Store, UnOp, Var, Zeros,
                   apply_op, typecheck)
from .tensor import new_param


def Symbol(name: str, constexpr: bool = False) -> se.Expr:
    """A named size symbol.  Symbols used as keyword defaults of the
    arrangement are the kernel's constexpr meta-parameters."""
    return se.var(name)


class Tensor:
    """Placeholder for a kernel parameter: ``Tensor(ndim)``; ``Tensor(0)`` is a
    by-value scalar (addmm's beta / alpha)."""

    def __init__(self, ndim: int, dtype: str = "f32", other: float = 0.0):
        self.ndim = int(ndim)
        self.dtype_kind = dtype
        self.other = float(other)    # fill value of masked loads (e.g. -inf for softmax)


class float32:  # ntl.float32 marker
    pass


class _Lang:
    float32 = float32
    float16 = "f16"

    @staticmethod
    def zeros(*a, **k):  # pragma: no cover - only referenced, never executed
        raise RuntimeError("ntl calls are compiled, not executed")

    dot = exp = sqrt = sigmoid = max = sum = zeros
    log = rsqrt = abs = tanh = relu = maximum = minimum = zeros


language = _Lang()


# ---- arrangement recording ----------------------------------------------------

class _Arranged:
    """Symbolic tensor view that records meta-ops at a given level depth."""

    def __init__(self, root, depth=0, ops=None):
        self._root = root          # _Param
        self._depth = depth
        self._ops = list(ops or [])

    def _with(self, op):
        return _Arranged(self._root, self._depth, self._ops + [op])

    def _tensor(self):
        t = self._root.tensor
        for op in self._ops:
            t = apply_op(t, op)
        return t

    def tile(self, shape, strides=None):
        return self._with(ArrangeOp("tile", depth=self._depth, shape=tuple(shape),
                                    strides=None if strides is None else tuple(strides)))

    def expand(self, shape):
        return self._with(ArrangeOp("expand", depth=self._depth, shape=tuple(shape)))

    def squeeze(self, dim):
        return self._with(ArrangeOp("squeeze", depth=self._depth, dim=dim))

    def permute(self, order):
        return self._with(ArrangeOp("permute", depth=self._depth, order=tuple(order)))

    def flatten(self, start_dim=0, end_dim=None):
        return self._with(ArrangeOp("flatten", depth=self._depth, start=start_dim, end=end_dim))

    def ravel(self):
        return self._with(ArrangeOp("ravel", depth=self._depth))

    @property
    def shape(self):
        t = self._tensor()
        for _ in range(self._depth):
            t = t.inner()
        return t.shape

    @property
    def dtype(self):
        return _Arranged(self._root, self._depth + 1, self._ops)

    @dtype.setter
    def dtype(self, inner):
        if not isinstance(inner, _Arranged) or inner._root is not self._root:
            raise SpecError("dtype must be assigned a view of the same tensor")
        self._ops = list(inner._ops)


class _Param:
    def __init__(self, name, rank):
        self.name = name
        self.tensor = new_param(name, rank)


# ---- application compilation (Python AST -> tile IR) ---------------------------

class _Compiler(ast.NodeVisitor):
    def __init__(self, params, tile_shapes, fills=None):
        self.params = params            # name -> rank
        self.tiles = tile_shapes        # name -> innermost tile shape (Exprs)
        self.fills = fills or {}        # name -> masked-load fill value
        self.ranks: dict = {}           # local -> tile rank
        self.locals: set = set()
        self.loop_vars: set = set()
        self.outputs: list = []

    # statements
    def stmts(self, body):
        out = []
        for node in body:
            r = self.stmt(node)
            if r is not None:
                out.append(r)
        return tuple(out)

    def stmt(self, n):
        if isinstance(n, ast.Expr) and isinstance(n.value, ast.Constant):
            return None  # docstring
        if isinstance(n, ast.Assign):
            if len(n.targets) != 1 or not isinstance(n.targets[0], ast.Name):
                raise SpecError("only `name = expr` assignments are supported")
            name = n.targets[0].id
            val = self.expr(n.value)
            if name in self.params:
                if name not in self.outputs:
                    self.outputs.append(name)
                return Store(name, val)
            if name in self.locals:
                raise SpecError(f"local {name!r} assigned twice (use +=)")
            self.locals.add(name)
            self.ranks[name] = self.rank(val)
            return Let(name, val)
        if isinstance(n, ast.AugAssign) and isinstance(n.op, ast.Add):
            if not isinstance(n.target, ast.Name) or n.target.id not in self.locals:
                raise SpecError("+= needs a local defined earlier")
            return Accumulate(n.target.id, self.expr(n.value))
        if isinstance(n, ast.For):
            if not isinstance(n.target, ast.Name) or not (
                    isinstance(n.iter, ast.Call) and getattr(n.iter.func, "id", "") == "range"
                    and len(n.iter.args) == 1):
                raise SpecError("only `for k in range(extent)` loops are supported")
            extent = self.extent(n.iter.args[0])
            self.loop_vars.add(n.target.id)
            body = self.stmts(n.body)
            self.loop_vars.discard(n.target.id)
            return ForRange(n.target.id, extent, body)
        raise SpecError(f"unsupported statement {ast.dump(n)[:60]}")

    def extent(self, n):
        # t.shape[i] of an arranged parameter = its (single) nest extent
        if (isinstance(n, ast.Subscript) and isinstance(n.value, ast.Attribute)
                and n.value.attr == "shape" and isinstance(n.value.value, ast.Name)):
            return ShapeOf(n.value.value.id, self._int(n.slice), "nest")
        raise SpecError("loop extent must be `param.shape[i]`")

    def _int(self, n):
        if isinstance(n, ast.Constant) and isinstance(n.value, int):
            return n.value
        raise SpecError("expected an integer literal")

    # expressions
    def expr(self, n):
        if isinstance(n, ast.Name):
            if n.id in self.params:
                return Load(n.id, (), self.fills.get(n.id, 0.0))
            if n.id in self.locals:
                return Local(n.id)
            raise SpecError(f"unknown name {n.id!r}")
        if isinstance(n, ast.Constant) and isinstance(n.value, (int, float)):
            return ConstF(float(n.value))
        if isinstance(n, ast.BinOp):
            op = {ast.Add: "+", ast.Sub: "-", ast.Mult: "*", ast.Div: "/"}.get(type(n.op))
            if op is None:
                raise SpecError("unsupported binary operator")
            return BinOp(op, self.expr(n.left), self.expr(n.right))
        if isinstance(n, ast.UnaryOp) and isinstance(n.op, ast.USub):
            return UnOp("neg", self.expr(n.operand))
        if isinstance(n, ast.Subscript) and isinstance(n.value, ast.Name) and \
                n.value.id in self.params:
            idx = n.slice
            if isinstance(idx, ast.Name) and idx.id in self.loop_vars:
                return Load(n.value.id, (Var(idx.id),), self.fills.get(n.value.id, 0.0))
            raise SpecError("nest index must be a loop variable")
        if isinstance(n, ast.Attribute) and n.attr == "shape":
            raise SpecError("use param.shape only as a loop extent or in ntl.zeros")
        if isinstance(n, ast.Call):
            fn = n.func.attr if isinstance(n.func, ast.Attribute) else getattr(n.func, "id", "")
            if fn == "zeros":
                return Zeros(self.shape_arg(n.args[0]), "f32")
            if fn == "dot":
                return Dot(self.expr(n.args[0]), self.expr(n.args[1]))
            if fn in ("exp", "sqrt", "sigmoid", "log", "rsqrt", "abs", "tanh", "relu"):
                return UnOp(fn, self.expr(n.args[0]))
            if fn in ("maximum", "minimum"):
                return BinOp("max" if fn == "maximum" else "min", self.expr(n.args[0]),
                             self.expr(n.args[1]))
            if fn in ("max", "sum"):
                arg = self.expr(n.args[0])
                kw = [k.value for k in n.keywords if k.arg == "axis"]
                if len(n.args) > 1:
                    axis = self._int(n.args[1])
                elif kw:
                    axis = self._int(kw[0])
                else:
                    axis = self.rank(arg) - 1    # Triton-style default: innermost axis
                return Reduce(fn, axis, arg)
            raise SpecError(f"unsupported call {fn!r}")
        raise SpecError(f"unsupported expression {ast.dump(n)[:60]}")

    def rank(self, e):
        if isinstance(e, Load):
            return len(self.tiles[e.param]) if self.params.get(e.param, 0) else 0
        if isinstance(e, Local):
            return self.ranks.get(e.name, 0)
        if isinstance(e, (BinOp, Dot)):
            return max(self.rank(e.a), self.rank(e.b)) if not isinstance(e, Dot) else 2
        if isinstance(e, UnOp):
            return self.rank(e.a)
        if isinstance(e, Reduce):
            return self.rank(e.a) - 1
        if isinstance(e, Zeros):
            return len(e.shape)
        return 0

    def shape_arg(self, n):
        if isinstance(n, ast.Attribute) and n.attr == "shape" and isinstance(n.value, ast.Name):
            return tuple(self.tiles[n.value.id])
        if isinstance(n, ast.Tuple):
            return tuple(se.var(e.id) if isinstance(e, ast.Name) else se.lit(self._int(e))
                         for e in n.elts)
        raise SpecError("zeros shape must be `param.shape` or a tuple")


def make(arrangement, application, tensors, name: str = "kernel"):
    """Build a B200 kernel from an arrangement and an application."""
    sig = inspect.signature(arrangement)
    names = list(sig.parameters)[: len(tensors)]
    meta = [p.name for p in list(sig.parameters.values())[len(tensors):]
            if isinstance(p.default, se.Expr)]
    ranks = {n: t.ndim for n, t in zip(names, tensors)}
    views = {n: _Arranged(_Param(n, r)) for n, r in ranks.items() if r >= 1}
    call = [views.get(n) for n in names]
    kwargs = {m: sig.parameters[m].default for m in meta}
    arranged = arrangement(*call, **kwargs)
    if not isinstance(arranged, tuple):
        arranged = (arranged,)
    tensor_names = [n for n in names if ranks[n] >= 1]
    if len(arranged) != len(tensor_names):
        raise SpecError("arrangement must return one arranged tensor per tensor parameter")
    ops = {}
    tiles = {}
    for n, a in zip(tensor_names, arranged):
        if not isinstance(a, _Arranged) or a._root.name != n:
            raise SpecError(f"arrangement output for {n!r} is not a view of {n!r}")
        ops[n] = tuple(a._ops)
        t = a._tensor()
        tiles[n] = t.level_shape(len(t.levels) - 1)
    src = textwrap.dedent(inspect.getsource(application))
    fn = next(n for n in ast.parse(src).body if isinstance(n, ast.FunctionDef))
    comp = _Compiler(ranks, tiles, {n: t.other for n, t in zip(names, tensors)})
    body = comp.stmts(fn.body)
    params = tuple(ParamSpec(n, ranks[n], "f32", "out" if n in comp.outputs else "in")
                   for n in names)
    spec = KernelSpec(name, params, tuple(meta), ops, body)
    return Kernel(typecheck(spec))


class Kernel:
    """``kernel(*params, **meta)`` - positional tensors, meta by keyword
    (PAPER.md:341-348); returns the output tensor(s)."""

    def __init__(self, checked):
        self.checked = checked
        self.spec = checked.spec

    def __call__(self, *args, **meta):
        spec = self.spec
        if len(args) != len(spec.params):
            raise TypeError(f"kernel takes {len(spec.params)} tensors, got {len(args)}")
        backend.launch(self.checked, {p.name: a for p, a in zip(spec.params, args)}, meta)
        outs = [a for p, a in zip(spec.params, args) if p.role == "out"]
        return outs[0] if len(outs) == 1 else tuple(outs)
