"""Compile a CheckedSpec's grid / checks / index maps into the C-ABI map blob.

This replaces the reference's two consumers of the same expressions:
the Triton text renderer (emit.py:157-262, which prints them into kernel
source) and the simulator's eval-compiled numpy lambdas (sim.py:87-97,
185-221).  Here every expression becomes postfix int64 code (opcodes in
include/ntb200.h) evaluated by the native map VM on the host
(``ntb_grid_eval``, ``ntb_map_enumerate``) or on the GPU (``ntb_map_probe``).

Accepts both this package's ``CheckedSpec`` and the reference's (duck typed:
``.spec.params/.spec.meta``, ``.grid.sizes/.checks``, ``.index_maps``), so a
spec built by either front end reaches the same native layer.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import symbolic as se
from .arrange import Grid

MAGIC = 0x4E544231
OPS = {"neg": 2, "add": 3, "sub": 4, "mul": 5, "floordiv": 6, "ceildiv": 7, "mod": 8,
       "min": 9, "max": 10}


def compile_expr(e, slot_of) -> list:
    code: list = []

    def walk(n):
        k = n[0]
        if k == "const":
            code.extend((0, n[1]))
        elif k == "sym":
            code.extend((1, slot_of(n[1])))
        elif k == "neg":
            walk(n[1])
            code.append(OPS["neg"])
        else:
            walk(n[1])
            walk(n[2])
            code.append(OPS[k])

    walk(se.from_any(e).node)
    return code


@dataclass
class MapProgram:
    blob: np.ndarray            # int64 map blob
    slot_names: tuple           # slot index -> symbol name
    params: tuple               # tensor parameter names, blob order
    grid: Grid                  # this package's view of the grid
    checks_text: tuple          # rendered (lhs, rhs) of each launch check

    def slots(self, binding: dict) -> np.ndarray:
        out = np.zeros(len(self.slot_names), dtype=np.int64)
        for i, name in enumerate(self.slot_names):
            if name in binding:
                out[i] = int(binding[name])
        return out


def build_program(checked) -> MapProgram:
    spec = checked.spec
    sizes = tuple(se.from_any(s) for s in checked.grid.sizes)
    checks = tuple((se.from_any(a), se.from_any(b)) for a, b in checked.grid.checks)
    total = sizes[0]
    for s in sizes[1:]:
        total = total * s
    grid = Grid(sizes=sizes, total=se.simplify(total), checks=checks)
    pidc = grid.pid_components(se.var("pid"))
    tensor_params = [p.name for p in spec.params if p.rank >= 1]
    maps = [checked.index_maps[n] for n in tensor_params]
    max_nest = max((len(m.nest_sizes) for m in maps), default=0)
    max_lane = max((len(m.lane_sizes) for m in maps), default=0)

    names: list = []
    for p in spec.params:
        for i in range(p.rank):
            names.append(f"{p.name}_size_{i}")
        for i in range(p.rank):
            names.append(f"{p.name}_stride_{i}")
    names.extend(spec.meta)
    names.append("pid")
    names.extend(f"pid_{i}" for i in range(len(sizes)))
    names.extend(f"nest_{k}" for k in range(max_nest))
    names.extend(f"lane_{j}" for j in range(max_lane))
    index = {n: i for i, n in enumerate(names)}

    def slot_of(name):
        try:
            return index[name]
        except KeyError:
            raise se.ExprError(f"map expression uses unknown symbol {name!r}") from None

    out: list = [MAGIC, len(names), len(sizes), len(checks), len(maps), index["pid"]]
    out.extend(index[f"pid_{i}"] for i in range(len(sizes)))
    out.append(max_nest)
    out.extend(index[f"nest_{k}"] for k in range(max_nest))
    out.append(max_lane)
    out.extend(index[f"lane_{j}"] for j in range(max_lane))

    def emit(e):
        c = compile_expr(e, slot_of)
        out.append(len(c))
        out.extend(c)

    for s in sizes:
        emit(s)
    for a, b in checks:
        emit(a)
        emit(b)
    for c in pidc:
        emit(c)
    for m in maps:
        out.extend((len(m.nest_sizes), len(m.lane_sizes)))
        for s in m.nest_sizes:
            emit(s)
        for s in m.lane_sizes:
            emit(s)
        emit(m.offset)
        out.append(len(m.mask))
        for lhs, bound in m.mask:
            emit(lhs)
            emit(bound)
    return MapProgram(
        blob=np.asarray(out, dtype=np.int64),
        slot_names=tuple(names),
        params=tuple(tensor_params),
        grid=grid,
        checks_text=tuple((se.text(a), se.text(b)) for a, b in checks),
    )
