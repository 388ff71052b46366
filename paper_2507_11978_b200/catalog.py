"""The paper's kernel set as arrangement programs + application IR.

The eight kernels the reference implements (catalog.py:35, 121-330) are
restated with the same meta-op sequences, so their lowered grids and index
maps are identical tree-for-tree to the reference's (pinned by
tests/test_maps.py against tests/golden/maps.json).  ``sdpa`` and ``rope``
are absent from the reference (catalog.py:36, OUT_OF_SCOPE) but evaluated in
the paper; their specs here are
builder-defined and documented in DESIGN.md:

* sdpa: ``O = softmax(Q K^T / sqrt(D)) V``, non-causal, (B, H, S, D) layout,
  one program per (b, h, BLOCK_SIZE_M query rows), K/V blocks of
  BLOCK_SIZE_N rows as the nest (FlashAttention-2 schedule).
* rope: half-split ("NeoX") rotary embedding of x (B, S, H, D) with
  sin/cos tables (S, D/2): ``y1 = x1*cos - x2*sin``, ``y2 = x1*sin + x2*cos``
  where x1/x2 are the two D/2 halves (PAPER.md:846 signature).
* sdpa_rope: ``sdpa(rope(q), rope(k), v)`` as ONE kernel (SURVEY 8(f) rank
  1: the rotated Q/K never go through HBM).  The tile IR has no program-id
  expression, so the rotary tables enter twice: ``sin_q``/``cos_q`` blocked
  like the query rows (outer level), ``sin_k``/``cos_k`` blocked like the key
  rows (nest level); callers pass the same (S, D/2) tables for both.  The
  rotation is written with two elementwise IR ops: ``rotate_half(x) =
  [-x2, x1]`` and ``dup2(t) = [t, t]`` along the last axis, so
  ``rope(x) = x * dup2(cos) + rotate_half(x) * dup2(sin)``.
"""

from __future__ import annotations

from functools import lru_cache

from .spec import (
    Accumulate, ArrangeOp, Assign, BinOp, ConstF, Dot, ForRange, IConst,
    KernelSpec, Let, Load, Local, ParamSpec, Reduce, ShapeOf, SpecError, Store,
    UnOp, Var, Zeros, apply_op, typecheck,
)
from .symbolic import var
from .tensor import FULL, new_param

CATALOG_NAMES = ("add", "silu", "softmax", "rms_norm", "mm", "bmm", "addmm", "conv2d")
EXTRA_NAMES = ("sdpa", "rope", "sdpa_rope")
ALL_NAMES = CATALOG_NAMES + EXTRA_NAMES

RMS_NORM_EPS = 1e-6


class Rec:
    """Records meta-ops while replaying them, so later ops can read the
    arranged shape of another parameter."""

    def __init__(self, name: str, rank: int):
        self.t = new_param(name, rank)
        self.ops: list = []

    def _do(self, op: ArrangeOp):
        self.t = apply_op(self.t, op)
        self.ops.append(op)
        return self

    def tile(self, shape, strides=None):
        return self._do(ArrangeOp("tile", shape=tuple(shape),
                                  strides=None if strides is None else tuple(strides)))

    def expand(self, shape):
        return self._do(ArrangeOp("expand", shape=tuple(shape)))

    def squeeze(self, dim, depth=0):
        return self._do(ArrangeOp("squeeze", depth=depth, dim=dim))

    def permute(self, order):
        return self._do(ArrangeOp("permute", order=tuple(order)))

    def flatten(self, start=0, end=None):
        return self._do(ArrangeOp("flatten", start=start, end=end))

    def ravel(self):
        return self._do(ArrangeOp("ravel"))

    @property
    def shape(self):
        return self.t.shape


def _matmul_arrangement(a: Rec, b: Rec, c: Rec, bm, bn, bk, lead=0):
    """c in (bm, bn) blocks; a as row panels of (bm, bk) blocks and b as
    column panels of (bk, bn) blocks, broadcast across the grid
    (reference catalog.py:82-106; PAPER.md Fig. matrix multiplication)."""
    keep = [-1] * lead
    one = [1] * lead
    c.tile(tuple(one + [bm, bn]))
    a.tile(tuple(one + [bm, bk]))
    a.tile(tuple(one + [1, FULL]))
    a.expand(tuple(keep + [-1, c.shape[lead + 1]]))
    for _ in range(lead):
        a.squeeze(0, depth=1)
    a.squeeze(0, depth=1)
    b.tile(tuple(one + [bk, bn]))
    b.tile(tuple(one + [FULL, 1]))
    b.expand(tuple(keep + [c.shape[lead], -1]))
    for _ in range(lead):
        b.squeeze(0, depth=1)
    b.squeeze(1, depth=1)
    for _ in range(lead):
        c.squeeze(0, depth=1)
        a.squeeze(0, depth=2)
        b.squeeze(0, depth=2)


def _matmul_body(a: str, b: str, c: str, bm, bn) -> tuple:
    return (
        Let("acc", Zeros((bm, bn), "f32")),
        ForRange("k", ShapeOf(a, 0, "nest"),
                 (Accumulate("acc", Dot(Load(a, (Var("k"),)), Load(b, (Var("k"),)))),)),
        Store(c, Local("acc")),
    )


def _ptab(*entries):
    return tuple(ParamSpec(n, r, "f32", role) for n, r, role in entries)


def spec_add() -> KernelSpec:
    bs = var("BLOCK_SIZE")
    recs = {n: Rec(n, 1).tile((bs,)) for n in ("input", "other", "output")}
    return KernelSpec(
        "add", _ptab(("input", 1, "in"), ("other", 1, "in"), ("output", 1, "out")),
        ("BLOCK_SIZE",), {n: tuple(r.ops) for n, r in recs.items()},
        (Store("output", BinOp("+", Load("input"), Load("other"))),))


def spec_silu() -> KernelSpec:
    bs = var("BLOCK_SIZE")
    recs = {n: Rec(n, 1).tile((bs,)) for n in ("input", "output")}
    return KernelSpec(
        "silu", _ptab(("input", 1, "in"), ("output", 1, "out")),
        ("BLOCK_SIZE",), {n: tuple(r.ops) for n, r in recs.items()},
        (Let("x", Load("input")),
         Store("output", BinOp("*", Local("x"), UnOp("sigmoid", Local("x"))))))


def spec_softmax() -> KernelSpec:
    cp = var("COLS_PADDED")
    recs = {n: Rec(n, 2).tile((1, cp)) for n in ("input", "output")}
    return KernelSpec(
        "softmax", _ptab(("input", 2, "in"), ("output", 2, "out")),
        ("COLS_PADDED",), {n: tuple(r.ops) for n, r in recs.items()},
        (Let("x", Load("input", other=float("-inf"))),
         Let("m", Reduce("max", 1, Local("x"))),
         Let("e", UnOp("exp", BinOp("-", Local("x"), Local("m")))),
         Let("s", Reduce("sum", 1, Local("e"))),
         Store("output", BinOp("/", Local("e"), Local("s")))))


def spec_rms_norm() -> KernelSpec:
    cp = var("COLS_PADDED")
    rows = var("input_size_0")
    recs = {}
    for n in ("input", "output"):
        r = Rec(n, 2).tile((1, cp))
        r.squeeze(1)
        r.squeeze(0, depth=1)
        recs[n] = r
    w = Rec("weight", 1).tile((cp,))
    w.tile((FULL,))
    w.expand((rows,))
    w.squeeze(0, depth=1)
    body = (
        Let("x", Load("input")),
        Let("ss", Reduce("sum", 0, BinOp("*", Local("x"), Local("x")))),
        Let("ms", BinOp("/", Local("ss"), ShapeOf("input", 1, "source"))),
        Store("output", BinOp(
            "*",
            BinOp("/", Local("x"),
                  UnOp("sqrt", BinOp("+", Local("ms"), ConstF(RMS_NORM_EPS)))),
            Load("weight"))),
    )
    return KernelSpec(
        "rms_norm", _ptab(("input", 2, "in"), ("weight", 1, "in"), ("output", 2, "out")),
        ("COLS_PADDED",),
        {"input": tuple(recs["input"].ops), "weight": tuple(w.ops),
         "output": tuple(recs["output"].ops)},
        body)


_MNK = ("BLOCK_SIZE_M", "BLOCK_SIZE_N", "BLOCK_SIZE_K")


def spec_mm() -> KernelSpec:
    bm, bn, bk = (var(s) for s in _MNK)
    a, b, c = Rec("input", 2), Rec("other", 2), Rec("output", 2)
    _matmul_arrangement(a, b, c, bm, bn, bk)
    return KernelSpec(
        "mm", _ptab(("input", 2, "in"), ("other", 2, "in"), ("output", 2, "out")), _MNK,
        {"input": tuple(a.ops), "other": tuple(b.ops), "output": tuple(c.ops)},
        _matmul_body("input", "other", "output", bm, bn))


def spec_bmm() -> KernelSpec:
    bm, bn, bk = (var(s) for s in _MNK)
    a, b, c = Rec("input", 3), Rec("other", 3), Rec("output", 3)
    _matmul_arrangement(a, b, c, bm, bn, bk, lead=1)
    return KernelSpec(
        "bmm", _ptab(("input", 3, "in"), ("other", 3, "in"), ("output", 3, "out")), _MNK,
        {"input": tuple(a.ops), "other": tuple(b.ops), "output": tuple(c.ops)},
        _matmul_body("input", "other", "output", bm, bn))


def spec_addmm() -> KernelSpec:
    bm, bn, bk = (var(s) for s in _MNK)
    a, b, c = Rec("mat1", 2), Rec("mat2", 2), Rec("output", 2)
    _matmul_arrangement(a, b, c, bm, bn, bk)
    addend = Rec("input", 2).tile((bm, bn))
    core = _matmul_body("mat1", "mat2", "output", bm, bn)
    epilogue = Store("output", BinOp(
        "+", BinOp("*", Load("beta"), Load("input")), BinOp("*", Load("alpha"), Local("acc"))))
    return KernelSpec(
        "addmm",
        _ptab(("input", 2, "in"), ("mat1", 2, "in"), ("mat2", 2, "in"), ("beta", 0, "in"),
              ("alpha", 0, "in"), ("output", 2, "out")),
        _MNK,
        {"input": tuple(addend.ops), "mat1": tuple(a.ops), "mat2": tuple(b.ops),
         "output": tuple(c.ops)},
        core[:-1] + (epilogue,))


def conv2d_pre():
    """Implicit GEMM view: image -> (N*P*Q, C*R*S) via a sliding-window tile,
    filter -> (C*R*S, K), output -> (N*P*Q, K) (reference catalog.py:295-312)."""
    f1, f2, f3 = var("filter_size_1"), var("filter_size_2"), var("filter_size_3")
    img = Rec("input", 4)
    img.tile((1, f1, f2, f3), strides=(-1, -1, 1, 1))
    img.squeeze(1)
    img.squeeze(0, depth=1)
    img.ravel()
    img.flatten(0, 3)
    img.flatten(1, None)
    flt = Rec("filter", 4)
    flt.flatten(1, None)
    flt.permute((1, 0))
    out = Rec("output", 4)
    out.permute((0, 2, 3, 1))
    out.flatten(0, 3)
    return img, flt, out


def spec_conv2d() -> KernelSpec:
    bm, bn, bk = (var(s) for s in _MNK)
    img, flt, out = conv2d_pre()
    _matmul_arrangement(img, flt, out, bm, bn, bk)
    return KernelSpec(
        "conv2d", _ptab(("input", 4, "in"), ("filter", 4, "in"), ("output", 4, "out")), _MNK,
        {"input": tuple(img.ops), "filter": tuple(flt.ops), "output": tuple(out.ops)},
        _matmul_body("input", "filter", "output", bm, bn))


def spec_sdpa() -> KernelSpec:
    """Builder-defined (no reference spec, catalog.py:36)."""
    bm, bn = var("BLOCK_SIZE_M"), var("BLOCK_SIZE_N")
    recs = {}
    for n in ("q", "o"):
        r = Rec(n, 4).tile((1, 1, bm, FULL))
        r.squeeze(3)
        r.squeeze(0, depth=1)
        r.squeeze(0, depth=1)
        recs[n] = r
    m_tiles = recs["o"].shape[2]
    for n in ("k", "v"):
        r = Rec(n, 4).tile((1, 1, bn, FULL))
        r.tile((1, 1, FULL, 1))
        r.expand((-1, -1, m_tiles, -1))
        r.squeeze(3)
        r.squeeze(0, depth=1)           # middle level (1, 1, Nt, 1) -> (Nt,)
        r.squeeze(0, depth=1)
        r.squeeze(1, depth=1)
        r.squeeze(0, depth=2)           # innermost (1, 1, BN, D) -> (BN, D)
        r.squeeze(0, depth=2)
        recs[n] = r
    d = ShapeOf("q", 3, "source")
    body = (
        Let("qt", Load("q")),
        Let("scale", BinOp("/", ConstF(1.0), UnOp("sqrt", d))),
        Let("acc", Zeros((bm, var("q_size_3")), "f32")),
        Let("l", Zeros((bm,), "f32")),
        Let("m", BinOp("-", Zeros((bm,), "f32"), ConstF(float("inf")))),
        ForRange("j", ShapeOf("k", 0, "nest"), (
            Let("s", BinOp("*", Dot(Local("qt"), UnOp("trans", Load("k", (Var("j"),), float("-inf")))),
                           Local("scale"))),
            Let("m_new", BinOp("max", Local("m"), Reduce("max", 1, Local("s")))),
            Let("p", UnOp("exp", BinOp("-", Local("s"), Local("m_new")))),
            Let("alpha", UnOp("exp", BinOp("-", Local("m"), Local("m_new")))),
            Assign("l", BinOp("+", BinOp("*", Local("l"), Local("alpha")), Reduce("sum", 1, Local("p")))),
            Assign("acc", BinOp("+", BinOp("*", Local("acc"), Local("alpha")),
                                Dot(Local("p"), Load("v", (Var("j"),))))),
            Assign("m", Local("m_new")),
        )),
        Store("o", BinOp("/", Local("acc"), Local("l"))),
    )
    params = tuple(ParamSpec(n, 4, "f16", "out" if n == "o" else "in") for n in ("q", "k", "v", "o"))
    return KernelSpec("sdpa", params, ("BLOCK_SIZE_M", "BLOCK_SIZE_N"),
                      {n: tuple(recs[n].ops) for n in ("q", "k", "v", "o")}, body)


def spec_rope() -> KernelSpec:
    """Builder-defined half-split rotary embedding."""
    half = var("HALF_D")
    xs = {}
    for n in ("input", "output"):
        r = Rec(n, 4).tile((1, 1, 1, FULL))     # outer (B, S, H, 1), inner (1, 1, 1, D)
        r.squeeze(3)
        r.permute((1, 0, 2))                    # (S, B, H)
        r.flatten(1, None)                      # (S, B*H)
        xs[n] = r
    for r in xs.values():
        r._do(ArrangeOp("tile", depth=1, shape=(1, 1, 1, half)))   # mid (1,1,1,2), inner (1,1,1,HALF)
        for _ in range(3):
            r.squeeze(0, depth=1)
        for _ in range(3):
            r.squeeze(0, depth=2)
    bh = xs["input"].shape[1]
    tabs = {}
    for n in ("sin", "cos"):
        r = Rec(n, 2).tile((1, FULL))           # outer (S, 1), inner (1, D/2)
        r.expand((-1, bh))
        r.squeeze(0, depth=1)
        tabs[n] = r
    x0, x1 = Load("input", (IConst(0),)), Load("input", (IConst(1),))
    body = (
        Let("c", Load("cos")), Let("s", Load("sin")),
        Let("x0", x0), Let("x1", x1),
        Store("output", BinOp("-", BinOp("*", Local("x0"), Local("c")),
                              BinOp("*", Local("x1"), Local("s"))), (IConst(0),)),
        Store("output", BinOp("+", BinOp("*", Local("x0"), Local("s")),
                              BinOp("*", Local("x1"), Local("c"))), (IConst(1),)),
    )
    params = (ParamSpec("input", 4, "f16", "in"), ParamSpec("sin", 2, "f16", "in"),
              ParamSpec("cos", 2, "f16", "in"), ParamSpec("output", 4, "f16", "out"))
    return KernelSpec("rope", params, ("HALF_D",),
                      {"input": tuple(xs["input"].ops), "sin": tuple(tabs["sin"].ops),
                       "cos": tuple(tabs["cos"].ops), "output": tuple(xs["output"].ops)},
                      body)


def _rope_ir(x, c, s):
    """x * dup2(c) + rotate_half(x) * dup2(s) (half-split rotary embedding)."""
    return BinOp("+", BinOp("*", x, UnOp("dup2", c)),
                 BinOp("*", UnOp("rotate_half", x), UnOp("dup2", s)))


def spec_sdpa_rope() -> KernelSpec:
    """Builder-defined sdpa(rope(q), rope(k), v)."""
    bm, bn = var("BLOCK_SIZE_M"), var("BLOCK_SIZE_N")
    recs = {}
    for n in ("q", "o"):
        r = Rec(n, 4).tile((1, 1, bm, FULL))    # outer (B, H, Mt, 1), inner (1, 1, bm, D)
        r.squeeze(3)
        r.flatten(0, 2)                          # outer (B*H, Mt)
        r.squeeze(0, depth=1)
        r.squeeze(0, depth=1)                    # inner (bm, D)
        recs[n] = r
    bh, m_tiles = recs["o"].shape
    for n in ("k", "v"):
        r = Rec(n, 4).tile((1, 1, bn, FULL))
        r.tile((1, 1, FULL, 1))
        r.expand((-1, -1, m_tiles, -1))
        r.squeeze(3)
        r.flatten(0, 2)                          # outer (B*H, Mt)
        r.squeeze(0, depth=1)
        r.squeeze(0, depth=1)
        r.squeeze(1, depth=1)                    # nest (Nt,)
        r.squeeze(0, depth=2)
        r.squeeze(0, depth=2)                    # inner (bn, D)
        recs[n] = r
    for n in ("sin_q", "cos_q"):
        r = Rec(n, 2).tile((bm, FULL))           # outer (Mt, 1), inner (bm, D/2)
        r.permute((1, 0))
        r.expand((bh, -1))                       # outer (B*H, Mt)
        recs[n] = r
    for n in ("sin_k", "cos_k"):
        r = Rec(n, 2).tile((bn, FULL))           # outer (Nt, 1), inner (bn, D/2)
        r.tile((FULL, 1))                        # outer (1, 1), nest (Nt, 1)
        r.expand((bh, m_tiles))
        r.squeeze(1, depth=1)                    # nest (Nt,)
        recs[n] = r
    d = ShapeOf("q", 3, "source")
    kj = Load("k", (Var("j"),), float("-inf"))
    krot = _rope_ir(kj, Load("cos_k", (Var("j"),)), Load("sin_k", (Var("j"),)))
    body = (
        Let("qt", _rope_ir(Load("q"), Load("cos_q"), Load("sin_q"))),
        Let("scale", BinOp("/", ConstF(1.0), UnOp("sqrt", d))),
        Let("acc", Zeros((bm, var("q_size_3")), "f32")),
        Let("l", Zeros((bm,), "f32")),
        Let("m", BinOp("-", Zeros((bm,), "f32"), ConstF(float("inf")))),
        ForRange("j", ShapeOf("k", 0, "nest"), (
            Let("s", BinOp("*", Dot(Local("qt"), UnOp("trans", krot)), Local("scale"))),
            Let("m_new", BinOp("max", Local("m"), Reduce("max", 1, Local("s")))),
            Let("p", UnOp("exp", BinOp("-", Local("s"), Local("m_new")))),
            Let("alpha", UnOp("exp", BinOp("-", Local("m"), Local("m_new")))),
            Assign("l", BinOp("+", BinOp("*", Local("l"), Local("alpha")), Reduce("sum", 1, Local("p")))),
            Assign("acc", BinOp("+", BinOp("*", Local("acc"), Local("alpha")),
                                Dot(Local("p"), Load("v", (Var("j"),))))),
            Assign("m", Local("m_new")),
        )),
        Store("o", BinOp("/", Local("acc"), Local("l"))),
    )
    names = ("q", "k", "v", "sin_q", "cos_q", "sin_k", "cos_k", "o")
    params = tuple(ParamSpec(n, 2 if n.startswith(("sin", "cos")) else 4, "f16",
                             "out" if n == "o" else "in") for n in names)
    return KernelSpec("sdpa_rope", params, ("BLOCK_SIZE_M", "BLOCK_SIZE_N"),
                      {n: tuple(recs[n].ops) for n in names}, body)


_MAKERS = {
    "add": spec_add, "silu": spec_silu, "softmax": spec_softmax, "rms_norm": spec_rms_norm,
    "mm": spec_mm, "bmm": spec_bmm, "addmm": spec_addmm, "conv2d": spec_conv2d,
    "sdpa": spec_sdpa, "rope": spec_rope, "sdpa_rope": spec_sdpa_rope,
}


def catalog(name: str) -> KernelSpec:
    try:
        return _MAKERS[name]()
    except KeyError:
        raise SpecError(f"unknown kernel {name!r}; available: {', '.join(ALL_NAMES)}") from None


@lru_cache(maxsize=None)
def checked(name: str):
    return typecheck(catalog(name))
