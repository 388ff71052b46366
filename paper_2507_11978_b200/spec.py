"""Kernel specs: parameters, arrangement programs, application IR, typecheck.

The IR vocabulary mirrors the reference's tile IR (tileir.py:48-151) so a
spec reads the same on both front ends: ``Load(param, nests, other)``,
``Local``, ``ConstF``, ``BinOp(+,-,*,/)``, ``UnOp(exp,sqrt,neg,sigmoid)``,
``Dot``, ``Zeros``, ``Reduce(sum|max, axis)``, ``ShapeOf(param, dim,
nest|source)`` and statements ``Let / Accumulate / Store / ForRange``.  Two
extensions carry the builder-defined attention spec (the reference has no
sdpa, catalog.py:36): ``Assign`` (rebind a local, for the online-softmax
running max/sum) and the binary op ``max`` / unary ``trans``.

``typecheck`` replays each parameter's arrangement program on a fresh
symbolic parameter (tileir.py:263-272), infers the grid, lowers the index
maps (arrange.py) and records the innermost tile shapes; it enforces the
reference's launch-independent rules (every output stored exactly once at
top level, tileir.py:422-458; nest-index count per load, tileir.py:346-355).

The B200 backend never interprets the application: it executes the
``CheckedSpec`` by matching it to a hand-written sm_100a kernel family
(backend.py); the IR is the contract that says what that kernel computes.
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass
from typing import Optional, Union

from . import symbolic as se
from .arrange import Grid, IndexMap, infer_grid, lower
from .symbolic import Expr, lift, simplify
from .tensor import KINDS, Tensor, new_param

ROLES = ("in", "out")


class SpecError(Exception):
    pass


class TypecheckError(SpecError):
    pass


# --- nest index expressions ----------------------------------------------

@dataclass(frozen=True)
class Var:
    name: str


@dataclass(frozen=True)
class IConst:
    value: int


# --- tile expressions ------------------------------------------------------

@dataclass(frozen=True)
class Load:
    param: str
    nests: tuple = ()
    other: float = 0.0


@dataclass(frozen=True)
class Local:
    name: str


@dataclass(frozen=True)
class ConstF:
    value: float


@dataclass(frozen=True)
class BinOp:
    op: str
    a: object
    b: object


@dataclass(frozen=True)
class UnOp:
    op: str
    a: object


@dataclass(frozen=True)
class Dot:
    a: object
    b: object


@dataclass(frozen=True)
class Zeros:
    shape: tuple
    kind: str = "f32"


@dataclass(frozen=True)
class Reduce:
    op: str
    axis: int
    a: object


@dataclass(frozen=True)
class ShapeOf:
    param: str
    dim: int
    of: str = "nest"


# --- statements --------------------------------------------------------------

@dataclass(frozen=True)
class Let:
    name: str
    expr: object


@dataclass(frozen=True)
class Assign:
    name: str
    expr: object


@dataclass(frozen=True)
class Accumulate:
    name: str
    expr: object


@dataclass(frozen=True)
class Store:
    param: str
    expr: object
    nests: tuple = ()   # builder extension: store into one nest (rope halves)


@dataclass(frozen=True)
class ForRange:
    var: str
    extent: object
    body: tuple


# --- spec ------------------------------------------------------------------

@dataclass(frozen=True)
class ParamSpec:
    name: str
    rank: int
    kind: str
    role: str


@dataclass(frozen=True)
class ArrangeOp:
    op: str
    depth: int = 0
    shape: Optional[tuple] = None
    strides: Optional[tuple] = None
    dim: Optional[int] = None
    order: Optional[tuple] = None
    start: Optional[int] = None
    end: Optional[int] = None


def apply_op(t: Tensor, op: ArrangeOp) -> Tensor:
    """Apply one meta-op at ``op.depth`` levels below the outermost
    (reference tileir.py:244-260)."""
    if op.depth > 0:
        return t.with_inner(apply_op(t.inner(), dataclasses.replace(op, depth=op.depth - 1)))
    if op.op == "tile":
        return t.tile(op.shape, op.strides)
    if op.op == "expand":
        return t.expand(op.shape)
    if op.op == "squeeze":
        return t.squeeze(op.dim)
    if op.op == "permute":
        return t.permute(op.order)
    if op.op == "flatten":
        return t.flatten(op.start or 0, op.end)
    if op.op == "ravel":
        return t.ravel()
    raise SpecError(f"unknown arrangement op {op.op!r}")


@dataclass(frozen=True)
class KernelSpec:
    name: str
    params: tuple
    meta: tuple
    arrangement: dict
    application: tuple

    def param(self, name: str) -> ParamSpec:
        for p in self.params:
            if p.name == name:
                return p
        raise SpecError(f"unknown parameter {name!r}")

    def __post_init__(self):
        names = [p.name for p in self.params]
        if len(set(names)) != len(names):
            raise SpecError("duplicate parameter names")
        for p in self.params:
            if p.kind not in KINDS:
                raise SpecError(f"parameter {p.name!r} has unknown kind {p.kind!r}")
            if p.role not in ROLES:
                raise SpecError(f"parameter {p.name!r} has unknown role {p.role!r}")
        if len(set(self.meta)) != len(self.meta):
            raise SpecError("duplicate meta-parameter")
        tensors = {p.name for p in self.params if p.rank >= 1}
        if set(self.arrangement) != tensors:
            raise SpecError("arrangement must cover exactly the tensor parameters")


@dataclass(frozen=True)
class CheckedSpec:
    spec: KernelSpec
    arrangement: tuple
    grid: Grid
    index_maps: dict
    tile_shapes: dict


def build_arrangement(spec: KernelSpec) -> list:
    out = []
    for p in spec.params:
        if p.rank < 1:
            continue
        t = new_param(p.name, p.rank, p.kind)
        for op in spec.arrangement[p.name]:
            t = apply_op(t, op)
        out.append((p.name, t))
    return out


def typecheck(spec: KernelSpec) -> CheckedSpec:
    arrangement = build_arrangement(spec)
    grid = infer_grid(arrangement)
    maps = {m.param: m for m in lower(arrangement, grid)}
    tiles = {name: tuple(simplify(s) for s in t.level_shape(len(t.levels) - 1))
             for name, t in arrangement}
    for p in spec.params:
        if p.rank == 0:
            tiles[p.name] = ()
    stored = {p.name: [] for p in spec.params if p.role == "out"}
    loop_vars: set = set()

    def expr(e):
        if isinstance(e, Load):
            p = spec.param(e.param)
            want = len(maps[e.param].nest_sizes) if p.rank else 0
            if len(e.nests) != want:
                raise TypecheckError(
                    f"load of {e.param!r} takes {want} nest indices, got {len(e.nests)}")
            for n in e.nests:
                if isinstance(n, Var) and n.name not in loop_vars:
                    raise TypecheckError(f"unknown index variable {n.name!r}")
        elif isinstance(e, (BinOp, Dot)):
            expr(e.a)
            expr(e.b)
        elif isinstance(e, (UnOp, Reduce)):
            expr(e.a)

    def stmt(s, top):
        if isinstance(s, (Let, Assign, Accumulate)):
            expr(s.expr)
        elif isinstance(s, Store):
            if spec.param(s.param).role != "out":
                raise TypecheckError(f"store into input parameter {s.param!r}")
            if not top:
                raise TypecheckError(f"store into {s.param!r} inside a loop")
            expr(s.expr)
            key = tuple(getattr(s, "nests", ()))
            if key in stored[s.param]:
                raise TypecheckError(f"output parameter {s.param!r} stored twice")
            stored[s.param].append(key)
        elif isinstance(s, ForRange):
            loop_vars.add(s.var)
            for b in s.body:
                stmt(b, False)
            loop_vars.discard(s.var)
        else:
            raise TypecheckError(f"unknown statement {type(s).__name__}")

    for s in spec.application:
        stmt(s, True)
    for name, keys in stored.items():
        if not keys:
            raise TypecheckError(f"output parameter {name!r} must be stored exactly once, got 0")
    return CheckedSpec(spec, tuple(arrangement), grid, maps, tiles)


def ir_tree(node):
    """Structural form of an application IR (class name + fields), valid for
    this module's nodes and the reference's (tileir.py dataclasses)."""
    if isinstance(node, Expr) or getattr(node, "kind", None) in se.KINDS:
        return ["expr", se.to_tree(se.from_any(node))]
    if dataclasses.is_dataclass(node) and not isinstance(node, type):
        out = [type(node).__name__]
        for f in dataclasses.fields(node):
            v = getattr(node, f.name)
            if isinstance(node, Store) and f.name == "nests" and not v:
                continue  # builder extension; absent from the reference IR
            out.append([f.name, ir_tree(v)])
        return out
    if isinstance(node, (tuple, list)):
        return [ir_tree(x) for x in node]
    if isinstance(node, float) and node in (float("inf"), float("-inf")):
        return "-inf" if node < 0 else "inf"
    return node
