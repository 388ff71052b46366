"""Generate the golden fixtures under tests/golden/ from the reference itself.

Run in the build container only (the reference tree does not exist on the GPU
box); the outputs are committed so the tests never read /root/reference:

    python tests/golden/gen_golden.py

What is dumped (all produced by the reference `tiledsl` package, imported from
/root/reference/pkg/src with PYTHONHASHSEED=0 because
`verify.sample_configs` seeds with `hash(kernel)`, verify.py:76):

* maps.json        - per catalog kernel: grid sizes / checks / pid components
                     and per-parameter index maps (offset, mask, source index,
                     lane and nest extents), each as the reference's JSON tree
                     (symexpr.py:251-256) and rendered text (symexpr.py:292),
                     plus the application IR as a structural tuple.
* map_points.npz   - numeric evaluation of those maps at small, odd shapes:
                     for every (pid, nest, lane) point the flat offset and the
                     mask bit, exactly as arrange/_covered_offsets in
                     test_arrange.py:26-57 enumerates them.
* sim_cases.npz    - the acceptance matrix (test_acceptance.py:26-27, 44-64:
                     20 configs per kernel, seed 2024+i) plus the
                     non-divisible cases of test_sim.py:36-56: inputs, meta,
                     sim.launch output and oracle output.
* expr_cases.json  - 1000 random (expression, binding, value) triples using the
                     generator of tests/helpers.py, pinning floor-division /
                     ceildiv / mod semantics (symexpr.py:150-156).
"""

from __future__ import annotations

import json
import os
import random
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"


def _reexec_with_hashseed():
    if os.environ.get("PYTHONHASHSEED") != "0":
        env = dict(os.environ, PYTHONHASHSEED="0")
        sys.exit(subprocess.call([sys.executable, __file__] + sys.argv[1:], env=env))


def _ir(node):
    """Structural tuple of an application IR node (class name + fields)."""
    import dataclasses

    from tiledsl.symexpr import SymExpr, to_json

    if isinstance(node, SymExpr):
        return ["expr", to_json(node)]
    if dataclasses.is_dataclass(node):
        out = [type(node).__name__]
        for f in dataclasses.fields(node):
            out.append([f.name, _ir(getattr(node, f.name))])
        return out
    if isinstance(node, (tuple, list)):
        return [_ir(x) for x in node]
    if isinstance(node, float):
        if node == float("-inf"):
            return "-inf"
        if node == float("inf"):
            return "inf"
    return node


def dump_maps(vf, out):
    from tiledsl.catalog import CATALOG_NAMES
    from tiledsl.emit import _TL
    from tiledsl.symexpr import render, sym, to_json

    kernels = {}
    for k in CATALOG_NAMES:
        checked = vf.checked_catalog(k)
        spec = checked.spec
        grid = checked.grid
        entry = {
            "params": [[p.name, p.rank, p.kind, p.role] for p in spec.params],
            "meta": list(spec.meta),
            "grid": {
                "sizes": [to_json(s) for s in grid.sizes],
                "sizes_text": [render(s) for s in grid.sizes],
                "total": to_json(grid.total),
                "checks": [[to_json(a), to_json(b)] for a, b in grid.checks],
                "checks_text": [[render(a), render(b)] for a, b in grid.checks],
                "pid_components": [to_json(c) for c in grid.pid_components(sym("pid"))],
                "pid_components_text": [render(c, _TL) for c in grid.pid_components(sym("pid"))],
            },
            "maps": {},
            "tile_shapes": {n: [to_json(s) for s in sh] for n, sh in checked.tile_shapes.items()},
            "application": _ir(spec.application),
        }
        for name, imap in checked.index_maps.items():
            entry["maps"][name] = {
                "lane_sizes": [to_json(s) for s in imap.lane_sizes],
                "nest_sizes": [to_json(s) for s in imap.nest_sizes],
                "source_index": [to_json(s) for s in imap.source_index],
                "offset": to_json(imap.offset),
                "offset_text": render(imap.offset),
                "mask": [[to_json(a), to_json(b)] for a, b in imap.mask],
                "mask_text": [[render(a), render(b)] for a, b in imap.mask],
            }
        kernels[k] = entry
    (out / "maps.json").write_text(json.dumps(kernels, indent=1, sort_keys=True) + "\n")


MAP_POINT_CASES = [
    ("add", {"N": 37}, {"BLOCK_SIZE": 8}),
    ("add", {"N": 10}, {"BLOCK_SIZE": 3}),
    ("silu", {"N": 5}, {"BLOCK_SIZE": 2}),
    ("softmax", {"R": 5, "C": 13}, {"COLS_PADDED": 16}),
    ("softmax", {"R": 3, "C": 20}, {"COLS_PADDED": 8}),
    ("rms_norm", {"R": 4, "C": 13}, {"COLS_PADDED": 16}),
    ("mm", {"M": 7, "N": 9, "K": 11}, {"BLOCK_SIZE_M": 3, "BLOCK_SIZE_N": 4, "BLOCK_SIZE_K": 2}),
    ("mm", {"M": 4, "N": 6, "K": 8}, {"BLOCK_SIZE_M": 2, "BLOCK_SIZE_N": 2, "BLOCK_SIZE_K": 3}),
    ("bmm", {"B": 3, "M": 7, "N": 9, "K": 11}, {"BLOCK_SIZE_M": 4, "BLOCK_SIZE_N": 4, "BLOCK_SIZE_K": 4}),
    ("addmm", {"M": 7, "N": 9, "K": 11}, {"BLOCK_SIZE_M": 4, "BLOCK_SIZE_N": 8, "BLOCK_SIZE_K": 3}),
    ("conv2d", {"N": 2, "C": 3, "H": 6, "W": 5, "K": 4, "R": 3, "S": 2},
     {"BLOCK_SIZE_M": 3, "BLOCK_SIZE_N": 2, "BLOCK_SIZE_K": 4}),
    ("conv2d", {"N": 1, "C": 2, "H": 5, "W": 5, "K": 3, "R": 3, "S": 3},
     {"BLOCK_SIZE_M": 4, "BLOCK_SIZE_N": 4, "BLOCK_SIZE_K": 8}),
]


def _binding(vf, kernel, dims, meta):
    from tiledsl.sim import binding_for

    args = vf.to_concrete(vf.make_inputs(kernel, vf.Config(kernel, dims, meta), 0))
    return binding_for(vf.checked_catalog(kernel), args, meta)


def dump_map_points(vf, out):
    import numpy as np

    from tiledsl.arrange import decompose_pid
    from tiledsl.symexpr import evaluate

    arrays = {}
    index = []
    for ci, (kernel, dims, meta) in enumerate(MAP_POINT_CASES):
        checked = vf.checked_catalog(kernel)
        binding = _binding(vf, kernel, dims, meta)
        grid = [int(evaluate(s, binding)) for s in checked.grid.sizes]
        total = int(np.prod(grid))
        arrays[f"c{ci}_grid"] = np.array(grid, dtype=np.int64)
        pids = np.array([decompose_pid(checked.grid, p, binding) for p in range(total)],
                        dtype=np.int64).reshape(total, len(grid))
        arrays[f"c{ci}_pids"] = pids
        params = []
        for name, imap in checked.index_maps.items():
            nest = [int(evaluate(s, binding)) for s in imap.nest_sizes]
            lane = [int(evaluate(s, binding)) for s in imap.lane_sizes]
            n_nest = int(np.prod(nest)) if nest else 1
            n_lane = int(np.prod(lane))
            offs = np.zeros((total, n_nest, n_lane), dtype=np.int64)
            mask = np.zeros((total, n_nest, n_lane), dtype=np.uint8)
            lane_grid = np.indices(lane).reshape(len(lane), -1) if lane else np.zeros((0, 1), np.int64)
            nest_grid = np.indices(nest).reshape(len(nest), -1) if nest else np.zeros((0, 1), np.int64)
            for pid in range(total):
                env = dict(binding)
                env.update({f"pid_{i}": int(v) for i, v in enumerate(pids[pid])})
                for ni in range(n_nest):
                    env.update({f"nest_{k}": int(nest_grid[k, ni]) for k in range(len(nest))})
                    env.update({f"lane_{j}": lane_grid[j].astype(np.int64) for j in range(len(lane))})
                    o = np.broadcast_to(np.asarray(evaluate(checked.index_maps[name].offset, env)), (n_lane,))
                    m = np.ones(n_lane, dtype=bool)
                    for lhs, bnd in imap.mask:
                        lv = np.broadcast_to(np.asarray(evaluate(lhs, env)), (n_lane,))
                        m &= lv < int(evaluate(bnd, env))
                    offs[pid, ni] = o
                    mask[pid, ni] = m
            arrays[f"c{ci}_{name}_offs"] = offs
            arrays[f"c{ci}_{name}_mask"] = mask
            params.append({"name": name, "nest": nest, "lane": lane})
        index.append({"kernel": kernel, "dims": dims, "meta": meta,
                      "binding": binding, "params": params})
    np.savez_compressed(out / "map_points.npz", **arrays)
    (out / "map_points.json").write_text(json.dumps(index, indent=1, sort_keys=True) + "\n")


SIM_EXTRA = [
    ("add", {"N": 37}, {"BLOCK_SIZE": 8}, 1),
    ("silu", {"N": 5}, {"BLOCK_SIZE": 8}, 1),
    ("softmax", {"R": 5, "C": 13}, {"COLS_PADDED": 16}, 1),
    ("softmax", {"R": 3, "C": 20}, {"COLS_PADDED": 8}, 4),  # chunked softmax (Appendix A.4)
    ("rms_norm", {"R": 4, "C": 13}, {"COLS_PADDED": 16}, 1),
    ("mm", {"M": 7, "N": 9, "K": 11}, {"BLOCK_SIZE_M": 4, "BLOCK_SIZE_N": 4, "BLOCK_SIZE_K": 4}, 1),
    ("bmm", {"B": 3, "M": 7, "N": 9, "K": 11}, {"BLOCK_SIZE_M": 4, "BLOCK_SIZE_N": 4, "BLOCK_SIZE_K": 4}, 1),
    ("addmm", {"M": 7, "N": 9, "K": 11}, {"BLOCK_SIZE_M": 4, "BLOCK_SIZE_N": 4, "BLOCK_SIZE_K": 4}, 1),
    ("conv2d", {"N": 2, "C": 3, "H": 6, "W": 5, "K": 4, "R": 3, "S": 2},
     {"BLOCK_SIZE_M": 4, "BLOCK_SIZE_N": 4, "BLOCK_SIZE_K": 4}, 1),
    ("add", {"N": 1}, {"BLOCK_SIZE": 1}, 0),
    ("mm", {"M": 64, "N": 48, "K": 80}, {"BLOCK_SIZE_M": 16, "BLOCK_SIZE_N": 16, "BLOCK_SIZE_K": 16}, 3),
    ("softmax", {"R": 8, "C": 100}, {"COLS_PADDED": 128}, 5),
    ("rms_norm", {"R": 8, "C": 100}, {"COLS_PADDED": 128}, 5),
]


def dump_sim_cases(vf, out):
    import numpy as np

    from tiledsl.catalog import CATALOG_NAMES

    cases = []
    for kernel in CATALOG_NAMES:
        for i, cfg in enumerate(vf.sample_configs(kernel, 20, 2024)):
            cases.append((kernel, cfg, 2024 + i))
    for kernel, dims, meta, seed in SIM_EXTRA:
        cases.append((kernel, vf.Config(kernel, dims, meta), seed))
    arrays = {}
    index = []
    for ci, (kernel, cfg, seed) in enumerate(cases):
        args = vf.make_inputs(kernel, cfg, seed)
        got = vf.simulate(kernel, args, cfg.meta)
        want = vf.run_oracle(kernel, args)
        scalars = {}
        for name, v in args.items():
            if np.ndim(v) == 0:
                scalars[name] = float(v)
            elif name != "output":
                arrays[f"c{ci}_{name}"] = v
        arrays[f"c{ci}_sim"] = got
        arrays[f"c{ci}_oracle"] = want
        index.append({"kernel": kernel, "dims": cfg.dims, "meta": cfg.meta, "seed": seed,
                      "const_rows": cfg.const_rows, "scalars": scalars,
                      "inputs": [n for n, v in args.items() if np.ndim(v) > 0 and n != "output"]})
    np.savez_compressed(out / "sim_cases.npz", **arrays)
    (out / "sim_cases.json").write_text(json.dumps(index, indent=1, sort_keys=True) + "\n")


def dump_expr_cases(out):
    sys.path.insert(0, REF_TESTS)
    from helpers import random_binding, random_expr
    from tiledsl.symexpr import evaluate, simplify, to_json

    rng = random.Random(1234)
    cases = []
    for _ in range(1000):
        e = random_expr(rng)
        b = random_binding(rng)
        cases.append({"expr": to_json(e), "simplified": to_json(simplify(e)),
                      "binding": b, "value": int(evaluate(e, b))})
    (out / "expr_cases.json").write_text(json.dumps(cases) + "\n")


def main():
    _reexec_with_hashseed()
    sys.path.insert(0, REF_SRC)
    from tiledsl import verify as vf

    dump_maps(vf, HERE)
    dump_map_points(vf, HERE)
    dump_sim_cases(vf, HERE)
    dump_expr_cases(HERE)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
