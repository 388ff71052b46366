"""Golden cases for the GENERIC path (specs outside the native families),
produced by the reference's own simulator.

Run in the build container only (the reference tree does not exist on the GPU
box); the output is committed:

    python tests/golden/gen_generic.py      # -> tests/golden/generic_cases.npz

Specs written directly in the reference's IR (tiledsl.tileir
KernelSpec / ArrangeOp / Reduce / BinOp, the `catalog._Builder` pattern,
catalog.py:45-79), each exercising a reduction along ONE axis of a loaded
tile - the broadcasting of the result follows tileir._broadcast
(tileir.py:290-306) and sim.py:324-328 (numpy):

* fma, gelu (x * sigmoid(1.702 x)), temp_softmax (exp(z - max z) / sum,
  z = x / 2, on (1, BLOCK) rows), l2norm (x / sqrt(sum x^2 + 1e-6)): the
  element-wise and whole-tile-reduction subset
* rowsum    x (M, N) tiled (BM, BN) and squeezed to a 1-D grid, out (M,)
            tiled (BM,): out = sum(x, axis=1)
* colexp    x, out (M, N) tiled (BM, BN): out = exp(x - max(x, axis=0))
            (masked loads fill -inf)
* rowcenter a, c (M, M) tiled (B, B): c = a - sum(a, axis=1) - the (B,)
            row sums broadcast right-aligned, i.e. along the last axis

Inputs are uniform(-1, 1) float32 from default_rng(seed) (verify.py:153-168
style); sim.launch runs them in f32 / f64 exactly as the reference does.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")


def main():
    from tiledsl import sim
    from tiledsl.catalog import _Builder
    from tiledsl.symexpr import sym
    from tiledsl.tileir import (BinOp, ConstF, KernelSpec, Let, Load, Local, ParamSpec, Reduce,
                                Store, UnOp, typecheck)

    BM, BN, B = sym("BM"), sym("BN"), sym("B")

    def rowsum():
        x = _Builder("x", 2).tile((BM, BN)).squeeze(1)
        o = _Builder("out", 1).tile((BM,))
        return KernelSpec(
            name="rowsum",
            params=(ParamSpec("x", 2, "f32", "in"), ParamSpec("out", 1, "f32", "out")),
            meta=("BM", "BN"), arrangement={"x": tuple(x.ops), "out": tuple(o.ops)},
            application=(Store("out", Reduce("sum", 1, Load("x"))),))

    def colexp():
        x = _Builder("x", 2).tile((BM, BN))
        o = _Builder("out", 2).tile((BM, BN))
        return KernelSpec(
            name="colexp",
            params=(ParamSpec("x", 2, "f32", "in"), ParamSpec("out", 2, "f32", "out")),
            meta=("BM", "BN"), arrangement={"x": tuple(x.ops), "out": tuple(o.ops)},
            application=(Store("out", UnOp("exp", BinOp(
                "-", Load("x", other=float("-inf")),
                Reduce("max", 0, Load("x", other=float("-inf")))))),))

    def rowcenter():
        a = _Builder("a", 2).tile((B, B))
        c = _Builder("c", 2).tile((B, B))
        return KernelSpec(
            name="rowcenter",
            params=(ParamSpec("a", 2, "f32", "in"), ParamSpec("c", 2, "f32", "out")),
            meta=("B",), arrangement={"a": tuple(a.ops), "c": tuple(c.ops)},
            application=(Store("c", BinOp("-", Load("a"), Reduce("sum", 1, Load("a")))),))

    BLOCK = sym("BLOCK")

    def fma():
        bs = {n: _Builder(n, 1).tile((BLOCK,)) for n in ("x", "y", "z", "out")}
        return KernelSpec(
            name="fma", params=tuple(ParamSpec(n, 1, "f32", "out" if n == "out" else "in")
                                     for n in ("x", "y", "z", "out")),
            meta=("BLOCK",), arrangement={n: tuple(b.ops) for n, b in bs.items()},
            application=(Store("out", BinOp("+", BinOp("*", Load("x"), Load("y")), Load("z"))),))

    def gelu():
        bs = {n: _Builder(n, 1).tile((BLOCK,)) for n in ("x", "out")}
        return KernelSpec(
            name="gelu", params=(ParamSpec("x", 1, "f32", "in"), ParamSpec("out", 1, "f32", "out")),
            meta=("BLOCK",), arrangement={n: tuple(b.ops) for n, b in bs.items()},
            application=(Store("out", BinOp("*", Load("x"), UnOp("sigmoid", BinOp(
                "*", ConstF(1.702), Load("x"))))),))

    def temp_softmax():
        bs = {n: _Builder(n, 2).tile((1, BLOCK)) for n in ("x", "out")}
        xl = Load("x", other=float("-inf"))
        return KernelSpec(
            name="temp_softmax",
            params=(ParamSpec("x", 2, "f32", "in"), ParamSpec("out", 2, "f32", "out")),
            meta=("BLOCK",), arrangement={n: tuple(b.ops) for n, b in bs.items()},
            application=(
                Let("z", BinOp("*", xl, ConstF(0.5))),
                Let("e", UnOp("exp", BinOp("-", Local("z"), Reduce("max", 1, Local("z"))))),
                Store("out", BinOp("/", Local("e"), Reduce("sum", 1, Local("e"))))))

    def l2norm():
        bs = {n: _Builder(n, 2).tile((1, BLOCK)) for n in ("x", "out")}
        return KernelSpec(
            name="l2norm",
            params=(ParamSpec("x", 2, "f32", "in"), ParamSpec("out", 2, "f32", "out")),
            meta=("BLOCK",), arrangement={n: tuple(b.ops) for n, b in bs.items()},
            application=(Store("out", BinOp("/", Load("x"), UnOp("sqrt", BinOp(
                "+", Reduce("sum", 1, BinOp("*", Load("x"), Load("x"))), ConstF(1e-6))))),))

    cases = [
        ("fma", fma(), {"x": (5000,), "y": (5000,), "z": (5000,)}, {"out": (5000,)},
         {"BLOCK": 1024}, 21),
        ("gelu", gelu(), {"x": (777,)}, {"out": (777,)}, {"BLOCK": 256}, 22),
        ("temp_softmax", temp_softmax(), {"x": (33, 1000)}, {"out": (33, 1000)}, {"BLOCK": 1024}, 23),
        ("l2norm", l2norm(), {"x": (7, 4096)}, {"out": (7, 4096)}, {"BLOCK": 4096}, 24),
        ("rowsum", rowsum(), {"x": (100, 300)}, {"out": (100,)}, {"BM": 16, "BN": 512}, 11),
        ("colexp", colexp(), {"x": (100, 300)}, {"out": (100, 300)}, {"BM": 64, "BN": 32}, 12),
        ("rowcenter", rowcenter(), {"a": (40, 40)}, {"c": (40, 40)}, {"B": 16}, 13),
    ]
    out = {}
    for name, spec, ins, outs, meta, seed in cases:
        checked = typecheck(spec)
        rng = np.random.default_rng(seed)
        arrays = {k: rng.uniform(-1, 1, shp).astype(np.float32) for k, shp in ins.items()}
        args = {k: sim.ConcreteTensor.from_array(v) for k, v in arrays.items()}
        for k, shp in outs.items():
            args[k] = sim.ConcreteTensor.from_array(np.zeros(shp, np.float32))
        sim.launch(checked, args, meta)
        for k, v in arrays.items():
            out[f"{name}.in.{k}"] = v
        for k, shp in outs.items():
            t = args[k]
            out[f"{name}.out.{k}"] = np.asarray(t.buffer, np.float32).reshape(shp)
        out[f"{name}.meta"] = np.array([meta[m] for m in spec.meta], np.int64)
        print(name, {k: out[f'{name}.out.{k}'].shape for k in outs})
    np.savez_compressed(HERE / "generic_cases.npz", **out)


if __name__ == "__main__":
    main()
