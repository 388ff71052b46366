"""Golden cases for the GENERIC path (specs outside the native families),
produced by the reference's own simulator.

Run in the build container only (the reference tree does not exist on the GPU
box); the output is committed:

    python tests/golden/gen_generic.py      # -> tests/golden/generic_cases.npz

Three specs written directly in the reference's IR (tiledsl.tileir
KernelSpec / ArrangeOp / Reduce / BinOp, the `catalog._Builder` pattern,
catalog.py:45-79), each exercising a reduction along ONE axis of a loaded
tile - the broadcasting of the result follows tileir._broadcast
(tileir.py:290-306) and sim.py:324-328 (numpy):

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
    from tiledsl.tileir import (BinOp, KernelSpec, Load, ParamSpec, Reduce, Store, UnOp,
                                typecheck)

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

    cases = [
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
