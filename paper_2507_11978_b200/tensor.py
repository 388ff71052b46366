"""Symbolic hierarchical tensors and the six meta-operations.

Behaviour follows the reference's ``htensor`` (htensor.py:111-274); the data
model is restated here for the B200 front end:

* a tensor is a tuple of levels (outermost first); a level is a tuple of axes;
  an axis is a tuple of ``Piece``s (more than one after ``flatten``);
* every piece contributes ``index * scale`` to an index ``Bucket``; a bucket
  splits its accumulated index mixed-radix over its ``Slot``s, and each slot
  either lands on a source dimension (``ToSource``) or feeds another bucket
  with a coefficient (``ToBucket``).  Tiling a flattened axis creates a fresh
  bucket over the constituent pieces (htensor.py:167-175), which is what lets
  conv2d's implicit-GEMM arrangement tile the (C, R, S) reduction axis.

Tile count: ``cdiv(size, tile)`` when the stride equals the tile, else the
sliding-window count ``(size - tile) // stride + 1`` (htensor.py:159-162).
``squeeze`` of a non-constant extent defers to a launch check
(htensor.py:206-211); ``flatten`` takes an exclusive end (htensor.py:222-229).

Symbols follow the reference ABI naming ``{p}_size_i`` / ``{p}_stride_i``
(htensor.py:262-263) because they are also the kernel-argument names of the
drop-in launcher (emit.py:88-96).
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Optional, Sequence

from .symbolic import ONE, ZERO, Expr, ceil_div, lift, simplify, var

FULL = -1
KEEP = -1
DEFAULT = -1

KINDS = ("f32", "f16", "bf16", "i32")


class TensorError(Exception):
    pass


class Bucket:
    """Index group; identity matters (shared by the pieces of one tiled axis)."""

    __slots__ = ("slots",)

    def __init__(self, slots):
        self.slots = tuple(slots)


@dataclass(frozen=True)
class ToSource:
    scale: Expr
    dim: int


@dataclass(frozen=True)
class ToBucket:
    coeff: Expr
    bucket: Bucket


@dataclass(frozen=True)
class Slot:
    extent: Expr
    dest: object  # ToSource | ToBucket


@dataclass(frozen=True)
class Piece:
    extent: Expr
    scale: Expr
    bucket: Bucket


def axis_extent(axis: tuple) -> Expr:
    out = axis[0].extent
    for p in axis[1:]:
        out = out * p.extent
    return simplify(out)


def _default(x) -> bool:
    return x is None or (isinstance(x, int) and not isinstance(x, bool) and x == -1)


@dataclass(frozen=True)
class Tensor:
    """Symbolic tensor parameter plus its arrangement so far."""

    name: str
    kind: str
    sizes: tuple
    strides: tuple
    levels: tuple  # tuple[tuple[axis, ...], ...], axis = tuple[Piece, ...]
    checks: tuple = ()

    @property
    def rank(self) -> int:
        return len(self.sizes)

    @property
    def shape(self) -> tuple:
        return tuple(axis_extent(a) for a in self.levels[0])

    def level_shape(self, i: int) -> tuple:
        return tuple(axis_extent(a) for a in self.levels[i])

    # ---- meta-operations ---------------------------------------------------

    def tile(self, tile_shape: Sequence, strides: Optional[Sequence] = None) -> "Tensor":
        axes = self.levels[0]
        if len(tile_shape) != len(axes):
            raise TensorError(f"tile shape has {len(tile_shape)} entries for {len(axes)} dims")
        if strides is not None and len(strides) != len(axes):
            raise TensorError("tile strides must match the tile shape length")
        outer, inner = [], []
        for d, axis in enumerate(axes):
            size = axis_extent(axis)
            t = size if _default(tile_shape[d]) else lift(tile_shape[d])
            s = DEFAULT if strides is None else strides[d]
            step = t if _default(s) else lift(s)
            t, step = simplify(t), simplify(step)
            if step.kind == "const" and step.value <= 0:
                raise TensorError(f"tile stride must be positive, got {step.value}")
            if step == t:
                count = simplify(ceil_div(size, t))
            else:
                count = simplify((size - t) // step + 1)
            if len(axis) == 1:
                p = axis[0]
                outer.append((Piece(count, simplify(p.scale * step), p.bucket),))
                inner.append((Piece(t, p.scale, p.bucket),))
            else:
                b = Bucket(Slot(p.extent, ToBucket(p.scale, p.bucket)) for p in axis)
                outer.append((Piece(count, step, b),))
                inner.append((Piece(t, ONE, b),))
        return replace(self, levels=(tuple(outer), tuple(inner)) + self.levels[1:])

    def expand(self, shape: Sequence) -> "Tensor":
        axes = self.levels[0]
        if len(shape) != len(axes):
            raise TensorError(f"expand shape has {len(shape)} entries for {len(axes)} dims")
        out = []
        for d, axis in enumerate(axes):
            if _default(shape[d]):
                out.append(axis)
                continue
            if len(axis) != 1 or axis_extent(axis) != ONE:
                raise TensorError(f"expand of non-singleton dim {d}")
            out.append((Piece(simplify(lift(shape[d])), ZERO, axis[0].bucket),))
        return replace(self, levels=(tuple(out),) + self.levels[1:])

    def squeeze(self, dim: int) -> "Tensor":
        axes = self.levels[0]
        if not 0 <= dim < len(axes):
            raise TensorError(f"squeeze dim {dim} out of range for {len(axes)} dims")
        axis = axes[dim]
        if len(axis) != 1:
            raise TensorError("squeeze of a flattened dim")
        size = axis_extent(axis)
        checks = self.checks
        if size.kind == "const":
            if size.value != 1:
                raise TensorError(f"squeeze of dim with size {size.value}")
        else:
            checks = checks + ((size, ONE),)
        return replace(self, levels=(axes[:dim] + axes[dim + 1:],) + self.levels[1:],
                       checks=checks)

    def permute(self, order: Sequence[int]) -> "Tensor":
        axes = self.levels[0]
        if sorted(order) != list(range(len(axes))):
            raise TensorError(f"{tuple(order)} is not a permutation of {len(axes)} dims")
        return replace(self, levels=(tuple(axes[i] for i in order),) + self.levels[1:])

    def flatten(self, start_dim: int = 0, end_dim: Optional[int] = None) -> "Tensor":
        axes = self.levels[0]
        end = len(axes) if end_dim is None else end_dim
        if not (0 <= start_dim < end <= len(axes)) or end - start_dim < 2:
            raise TensorError(f"flatten span [{start_dim}, {end}) is degenerate")
        merged = tuple(p for a in axes[start_dim:end] for p in a)
        return replace(self, levels=(axes[:start_dim] + (merged,) + axes[end:],) + self.levels[1:])

    def ravel(self) -> "Tensor":
        return replace(self, levels=(tuple(a for lvl in self.levels for a in lvl),))

    def inner(self) -> "Tensor":
        if len(self.levels) < 2:
            raise TensorError("inner level of a single-level tensor")
        return replace(self, levels=self.levels[1:])

    def with_inner(self, inner: "Tensor") -> "Tensor":
        if inner.name != self.name or inner.rank != self.rank:
            raise TensorError("with_inner with mismatched source identity")
        checks = self.checks + tuple(c for c in inner.checks if c not in self.checks)
        return replace(self, levels=self.levels[:1] + inner.levels, checks=checks)

    # paper-style aliases (htensor.py:235-244)
    get_inner = inner
    set_inner = with_inner


def new_param(name: str, rank: int, kind: str = "f32") -> Tensor:
    """Fresh single-level parameter with ABI-named size/stride symbols."""
    if rank < 1:
        raise TensorError(f"parameter rank must be >= 1, got {rank}")
    if kind not in KINDS:
        raise TensorError(f"unknown element kind {kind!r}")
    sizes = tuple(var(f"{name}_size_{i}") for i in range(rank))
    strides = tuple(var(f"{name}_stride_{i}") for i in range(rank))
    axes = tuple(
        (Piece(sizes[d], ONE, Bucket((Slot(sizes[d], ToSource(ONE, d)),))),)
        for d in range(rank)
    )
    return Tensor(name, kind, sizes, strides, (axes,))


def param_with_shape(name: str, shape: Sequence[int], kind: str = "f32") -> Tensor:
    """Parameter with constant sizes (strides stay symbolic)."""
    if not shape:
        raise TensorError("shape must have at least one dim")
    sizes = tuple(lift(int(s)) for s in shape)
    strides = tuple(var(f"{name}_stride_{i}") for i in range(len(shape)))
    axes = tuple(
        (Piece(sizes[d], ONE, Bucket((Slot(sizes[d], ToSource(ONE, d)),))),)
        for d in range(len(shape))
    )
    return Tensor(name, kind, sizes, strides, (axes,))
