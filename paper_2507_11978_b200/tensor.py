"""Arranged tensors: the six meta-operations as rewrites of index variables.

Design (this package's own; the reference's ``htensor`` keeps a graph of
index groups instead).  An arranged tensor is

* ``coords`` - one integer expression per SOURCE dimension, written over
  index variables (one variable per dimension of some level);
* ``levels`` - the hierarchy the meta-operations built, outermost first;
  each level is a tuple of ``Dim(var, extent, parts)``;
* ``env`` - the substitutions (``var -> expression``) the meta-operations
  recorded.  A variable is substituted at most once, so the environment is
  a set of equations; resolving ``coords`` under it (plus the launch
  binding of the surviving variables to ``pid_i`` / ``nest_k`` / ``lane_j``)
  gives the source index of every element a program touches.

Every meta-operation is one rewrite:

=========  ==================================================================
tile       dim v (extent S) -> outer o (count) and inner t (tile T), with
           v := o*step + t.  count = cdiv(S, T) when step == T, else the
           sliding-window count (S - T) // step + 1 (reference semantics,
           htensor.py:159-162)
expand     a size-1 dim gets a new extent; its old variable := 0 (every
           element of the new dim reads the same source element)
squeeze    a size-1 dim disappears; its variable := 0.  A symbolic extent
           becomes a launch-time check ``extent == 1`` (htensor.py:206-211)
permute    reorders the outermost level
flatten    dims [start, end) -> one dim; the merged variables are kept as
           ``parts`` and decoded mixed-radix (last part fastest, the leading
           digit not reduced, so an out-of-range index stays out of range for
           the bound check) only when the merged dim is consumed - by a later
           tile or by the launch binding.  A flatten of flattened dims just
           concatenates their parts, so the decode stays one level deep
ravel      concatenates all levels into one
=========  ==================================================================

Size and stride symbols keep the reference's ABI names ``{p}_size_i`` /
``{p}_stride_i`` (htensor.py:262-263): they are the kernel-argument names of
the drop-in launcher (emit.py:88-96).
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass, replace
from typing import Optional, Sequence

from . import symbolic as se
from .symbolic import ONE, ZERO, Expr, ceil_div, lift, simplify, var

FULL = -1

KINDS = ("f32", "f16", "bf16", "i32")

_fresh = itertools.count()


def fresh_var() -> str:
    """A new index-variable name (never visible after lowering)."""
    return f"ix_{next(_fresh)}_"


def is_index_var(name: str) -> bool:
    return name.startswith("ix_") and name.endswith("_")


class TensorError(Exception):
    pass


def _keep(x) -> bool:
    """None / -1 mean 'leave this dimension as it is' in shape arguments."""
    return x is None or (isinstance(x, int) and not isinstance(x, bool) and x == -1)


@dataclass(frozen=True)
class Dim:
    var: str
    extent: Expr
    parts: tuple = ()   # flattened dim: ((var, extent), ...) outermost first

    def decode(self, index: Expr) -> dict:
        """Substitutions that bind this dim's variable (and, for a flattened
        dim, every merged variable) to ``index``."""
        subs = {self.var: index}
        if self.parts:
            radix = [e for _, e in self.parts]
            below = ONE
            digits = []
            for j in range(len(radix) - 1, -1, -1):
                q = index if below == ONE else index // below
                digits.append(q if j == 0 else q % radix[j])
                below = simplify(radix[j] * below)
            for (v, _), d in zip(self.parts, reversed(digits)):
                subs[v] = simplify(d)
        return subs


@dataclass(frozen=True)
class Tensor:
    name: str
    kind: str
    sizes: tuple
    strides: tuple
    coords: tuple
    levels: tuple
    env: tuple = ()      # ((var, Expr), ...)
    checks: tuple = ()   # ((lhs, rhs), ...): launch-time equalities

    @property
    def rank(self) -> int:
        return len(self.sizes)

    @property
    def shape(self) -> tuple:
        return self.level_shape(0)

    def level_shape(self, i: int) -> tuple:
        return tuple(d.extent for d in self.levels[i])

    # ---- helpers ----------------------------------------------------------

    def _top(self) -> tuple:
        return self.levels[0]

    def _with_top(self, dims, *outer, env=(), checks=()) -> "Tensor":
        return replace(self, levels=tuple(outer) + (tuple(dims),) + self.levels[1:],
                       env=self.env + tuple(env), checks=self.checks + tuple(checks))

    def _need(self, seq, what: str):
        if len(seq) != len(self._top()):
            raise TensorError(f"{what} for {self.name!r}: {len(seq)} entries, but its "
                              f"outermost level has {len(self._top())} dims")

    def resolve(self, extra: Optional[dict] = None) -> tuple:
        """``coords`` with every recorded substitution (and ``extra``)
        applied until no substituted variable is left."""
        subs = dict(self.env)
        if extra:
            subs.update(extra)
        out = []
        for c in self.coords:
            for _ in range(len(subs) + 1):
                hit = se.symbols(c) & subs.keys()
                if not hit:
                    break
                c = se.subst(c, {v: subs[v] for v in hit})
            out.append(simplify(c))
        return tuple(out)

    # ---- meta-operations ----------------------------------------------------

    def tile(self, tile_shape: Sequence, strides: Optional[Sequence] = None) -> "Tensor":
        self._need(tile_shape, "tile shape")
        if strides is not None:
            self._need(strides, "tile strides")
        outer, inner, env = [], [], []
        for d, dim in enumerate(self._top()):
            size = dim.extent
            t = size if _keep(tile_shape[d]) else simplify(lift(tile_shape[d]))
            step = t if strides is None or _keep(strides[d]) else simplify(lift(strides[d]))
            if step.kind == "const" and step.value < 1:
                raise TensorError(f"tile step along dim {d} of {self.name!r} must be >= 1, "
                                  f"got {step.value}")
            count = ceil_div(size, t) if step == t else (size - t) // step + 1
            o, i = fresh_var(), fresh_var()
            outer.append(Dim(o, simplify(count)))
            inner.append(Dim(i, t))
            env.extend(dim.decode(var(o) * step + var(i)).items())
        return self._with_top(inner, tuple(outer), env=env)

    def expand(self, shape: Sequence) -> "Tensor":
        self._need(shape, "expand shape")
        dims, env = [], []
        for d, dim in enumerate(self._top()):
            if _keep(shape[d]):
                dims.append(dim)
                continue
            if dim.parts or dim.extent != ONE:
                raise TensorError(f"expand needs a size-1 dim; dim {d} of {self.name!r} has "
                                  f"extent {se.text(dim.extent)}")
            env.append((dim.var, ZERO))
            dims.append(Dim(fresh_var(), simplify(lift(shape[d]))))
        return self._with_top(dims, env=env)

    def squeeze(self, dim: int) -> "Tensor":
        top = self._top()
        if not 0 <= dim < len(top):
            raise TensorError(f"squeeze: {self.name!r} has no dim {dim} (outermost level has "
                              f"{len(top)})")
        victim = top[dim]
        if victim.parts:
            raise TensorError(f"squeeze: dim {dim} of {self.name!r} is a flattened dim")
        checks = ()
        if victim.extent.kind == "const":
            if victim.extent.value != 1:
                raise TensorError(f"squeeze: dim {dim} of {self.name!r} has extent "
                                  f"{victim.extent.value}, not 1")
        else:
            checks = ((victim.extent, ONE),)
        return self._with_top(top[:dim] + top[dim + 1:], env=((victim.var, ZERO),),
                              checks=checks)

    def permute(self, order: Sequence[int]) -> "Tensor":
        top = self._top()
        if sorted(order) != list(range(len(top))):
            raise TensorError(f"permute: {tuple(order)} does not reorder the {len(top)} dims "
                              f"of {self.name!r}")
        return self._with_top([top[i] for i in order])

    def flatten(self, start_dim: int = 0, end_dim: Optional[int] = None) -> "Tensor":
        top = self._top()
        end = len(top) if end_dim is None else end_dim
        if not 0 <= start_dim < end <= len(top) or end - start_dim < 2:
            raise TensorError(f"flatten: dims [{start_dim}, {end}) of {self.name!r} do not "
                              "name two or more dims")
        parts = []
        for dim in top[start_dim:end]:
            parts.extend(dim.parts or ((dim.var, dim.extent),))
        extent = parts[0][1]
        for _, e in parts[1:]:
            extent = extent * e
        merged = Dim(fresh_var(), simplify(extent), tuple(parts))
        return self._with_top(top[:start_dim] + (merged,) + top[end:])

    def ravel(self) -> "Tensor":
        return replace(self, levels=(tuple(d for lvl in self.levels for d in lvl),))

    def inner(self) -> "Tensor":
        if len(self.levels) < 2:
            raise TensorError(f"{self.name!r} has no inner level")
        return replace(self, levels=self.levels[1:])

    def with_inner(self, inner: "Tensor") -> "Tensor":
        if inner.name != self.name or inner.rank != self.rank:
            raise TensorError(f"with_inner: {inner.name!r} is not an inner view of "
                              f"{self.name!r}")
        env = dict(self.env)
        env.update(inner.env)
        checks = self.checks + tuple(c for c in inner.checks if c not in self.checks)
        return replace(self, levels=self.levels[:1] + inner.levels, env=tuple(env.items()),
                       checks=checks)

    # paper-style aliases
    get_inner = inner
    set_inner = with_inner


def _fresh_tensor(name: str, kind: str, sizes: tuple) -> Tensor:
    if kind not in KINDS:
        raise TensorError(f"element kind {kind!r} is not one of {KINDS}")
    strides = tuple(var(f"{name}_stride_{i}") for i in range(len(sizes)))
    vs = [fresh_var() for _ in sizes]
    return Tensor(name, kind, sizes, strides, coords=tuple(var(v) for v in vs),
                  levels=(tuple(Dim(v, s) for v, s in zip(vs, sizes)),))


def new_param(name: str, rank: int, kind: str = "f32") -> Tensor:
    """A parameter with ABI-named symbolic sizes and strides, one level."""
    if rank < 1:
        raise TensorError(f"tensor parameter {name!r} needs rank >= 1, got {rank}")
    return _fresh_tensor(name, kind, tuple(var(f"{name}_size_{i}") for i in range(rank)))


def param_with_shape(name: str, shape: Sequence[int], kind: str = "f32") -> Tensor:
    """A parameter with constant sizes (strides stay symbolic)."""
    if not shape:
        raise TensorError(f"tensor parameter {name!r} needs at least one dim")
    return _fresh_tensor(name, kind, tuple(lift(int(s)) for s in shape))
