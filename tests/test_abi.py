"""The C-ABI library: loads, exports every declared entry point, and its
native map VM reproduces the reference's integer maps bit-exactly (no GPU
needed: the VM runs on the host)."""

import re
from pathlib import Path

import numpy as np
import pytest

from helpers import expr_cases, map_cases, maps
from paper_2507_11978_b200 import _lib, backend
from paper_2507_11978_b200 import catalog as C
from paper_2507_11978_b200 import symbolic as S
from paper_2507_11978_b200.bytecode import build_program, compile_expr

HEADER = Path(__file__).resolve().parent.parent / "include" / "ntb200.h"


def test_library_exports_every_declared_symbol():
    declared = set(re.findall(r"^\s*(?:int|const char\*|int64_t)\s+(ntb_\w+)\(",
                              HEADER.read_text(), re.M))
    assert declared == set(_lib.EXPORTS)
    L = _lib.lib()
    for name in declared:
        assert hasattr(L, name)
    assert L.ntb_abi_version() == 1


def test_vm_expression_eval_bit_exact():
    names = ("a", "b", "c", "d")
    for c in expr_cases():
        code = compile_expr(S.from_tree(c["expr"]), names.index)
        rc, v = _lib.expr_eval(code, [c["binding"][n] for n in names])
        assert rc == 0 and v == c["value"]


def test_vm_zero_divisor_is_eval_error():
    code = compile_expr(S.var("a") // S.var("b"), ("a", "b").index)
    rc, _ = _lib.expr_eval(code, [1, 0])
    assert rc == _lib.NTB_ERR_EVAL


def test_vm_grid_and_map_points_match_reference():
    index, arrays = map_cases()
    for ci, case in enumerate(index):
        prog = build_program(C.checked(case["kernel"]))
        slots = prog.slots(case["binding"])
        rc, grid = _lib.grid_eval(prog.blob, slots)
        assert rc == 0, _lib.last_error()
        assert list(grid) == list(arrays[f"c{ci}_grid"])
        for p in case["params"]:
            q = prog.params.index(p["name"])
            rc, offs, mask = _lib.map_enumerate(prog.blob, q, slots)
            assert rc == 0, _lib.last_error()
            np.testing.assert_array_equal(offs, arrays[f"c{ci}_{p['name']}_offs"].reshape(-1))
            np.testing.assert_array_equal(mask, arrays[f"c{ci}_{p['name']}_mask"].reshape(-1))


class _Fake:
    """Shape/stride carrier for host-side validation tests (no data)."""

    def __init__(self, shape):
        self.shape = tuple(shape)
        st, acc = [], 1
        for s in reversed(self.shape):
            st.append(acc)
            acc *= s
        self._st = tuple(reversed(st))

    def stride(self):
        return self._st


def _mm_args():
    return {"input": _Fake((4, 4)), "other": _Fake((4, 4)), "output": _Fake((4, 4))}


MM_META = {"BLOCK_SIZE_M": 2, "BLOCK_SIZE_N": 2, "BLOCK_SIZE_K": 2}


@pytest.mark.parametrize("mutate", ["missing_meta", "zero_meta", "extra_meta", "missing_arg",
                                    "extra_arg", "wrong_rank", "bad_check"])
def test_launch_validation_raises_launch_error(mutate):
    """sim.py:128-160 conditions (test_sim.py:97-140)."""
    args, meta = _mm_args(), dict(MM_META)
    if mutate == "missing_meta":
        del meta["BLOCK_SIZE_K"]
    elif mutate == "zero_meta":
        meta["BLOCK_SIZE_M"] = 0
    elif mutate == "extra_meta":
        meta["BLOCK"] = 3
    elif mutate == "missing_arg":
        del args["other"]
    elif mutate == "extra_arg":
        args["bias"] = _Fake((4,))
    elif mutate == "wrong_rank":
        args["other"] = _Fake((4,))
    elif mutate == "bad_check":
        args["output"] = _Fake((9, 4))
    with pytest.raises(backend.LaunchError):
        backend.launch(C.checked("mm"), args, meta)


def test_rms_norm_padded_width_check():
    args = {"input": _Fake((3, 20)), "weight": _Fake((20,)), "output": _Fake((3, 20))}
    with pytest.raises(backend.LaunchError, match="launch-time check failed"):
        backend.launch(C.checked("rms_norm"), args, {"COLS_PADDED": 16})


def test_non_catalog_spec_takes_the_generic_path_and_needs_cuda_tensors():
    """A spec outside the native families is code-generated (codegen.py); the
    generated path, like every other, refuses host tensors (no CPU path)."""
    from paper_2507_11978_b200.spec import KernelSpec, ParamSpec, Store, Load, typecheck, ArrangeOp
    spec = KernelSpec("copy", (ParamSpec("input", 1, "f32", "in"), ParamSpec("output", 1, "f32", "out")),
                      ("BLOCK_SIZE",),
                      {"input": (ArrangeOp("tile", shape=(S.var("BLOCK_SIZE"),)),),
                       "output": (ArrangeOp("tile", shape=(S.var("BLOCK_SIZE"),)),)},
                      (Store("output", Load("input")),))
    with pytest.raises(backend.LaunchError, match="CUDA tensor"):
        backend.launch(typecheck(spec), {"input": _Fake((8,)), "output": _Fake((8,))},
                       {"BLOCK_SIZE": 4})


def test_spec_outside_generic_subset_is_unsupported():
    """A contraction whose operand is an expression (not a loaded tile) is
    neither a native family nor generated: UnsupportedSpecError names the
    reason."""
    from paper_2507_11978_b200.spec import (ArrangeOp, BinOp, ConstF, Dot, KernelSpec, Load,
                                            ParamSpec, Store, typecheck)
    t = (ArrangeOp("tile", shape=(S.var("B"), S.var("B"))),)
    spec = KernelSpec("dot_of_expr", (ParamSpec("a", 2, "f16", "in"),
                                      ParamSpec("c", 2, "f16", "out")),
                      ("B",), {"a": t, "c": t},
                      (Store("c", Dot(BinOp("*", Load("a"), ConstF(2.0)), Load("a"))),))
    with pytest.raises(backend.UnsupportedSpecError, match="generic path"):
        backend.launch(typecheck(spec), {"a": _Fake((8, 8)), "c": _Fake((8, 8))}, {"B": 4})


def test_sdpa_rope_table_rows_checked_before_launch():
    """The query-side tables must block like the query rows (grid check,
    evaluated by the native map VM before any device work)."""
    ck = C.checked("sdpa_rope")
    b, h, s, d = 2, 3, 300, 64
    args = {"q": _Fake((b, h, s, d)), "k": _Fake((b, h, s, d)), "v": _Fake((b, h, s, d)),
            "sin_q": _Fake((100, d // 2)), "cos_q": _Fake((s, d // 2)),
            "sin_k": _Fake((s, d // 2)), "cos_k": _Fake((s, d // 2)),
            "o": _Fake((b, h, s, d))}
    with pytest.raises(backend.LaunchError, match="launch-time check failed"):
        backend.launch(ck, args, {"BLOCK_SIZE_M": 128, "BLOCK_SIZE_N": 128})


def test_sdpa_rope_is_its_own_family():
    assert backend._family_of(C.checked("sdpa_rope")) == "sdpa_rope"
    assert _lib.KERNEL_IDS["sdpa_rope"] == 11
    hdr = Path(__file__).resolve().parent.parent / "include" / "ntb200.h"
    assert "NTB_K_SDPA_ROPE = 11" in hdr.read_text()


@pytest.mark.parametrize("kernel,shapes,meta", [
    ("add", {"input": (1000,), "other": (1000,), "output": (1000,)}, {"BLOCK_SIZE": 64}),
    ("softmax", {"input": (5, 20), "output": (5, 20)}, {"COLS_PADDED": 32}),
    ("mm", {"input": (70, 40), "other": (40, 90), "output": (70, 90)},
     {"BLOCK_SIZE_M": 32, "BLOCK_SIZE_N": 16, "BLOCK_SIZE_K": 8}),
    ("bmm", {"input": (3, 20, 24), "other": (3, 24, 18), "output": (3, 20, 18)},
     {"BLOCK_SIZE_M": 8, "BLOCK_SIZE_N": 16, "BLOCK_SIZE_K": 8}),
    ("conv2d", {"input": (2, 3, 9, 7), "filter": (4, 3, 3, 2), "output": (2, 4, 7, 6)},
     {"BLOCK_SIZE_M": 16, "BLOCK_SIZE_N": 4, "BLOCK_SIZE_K": 8}),
    ("rope", {"input": (2, 5, 3, 8), "sin": (5, 4), "cos": (5, 4), "output": (2, 5, 3, 8)},
     {"HALF_D": 4}),
])
def test_write_partition_matches_the_reference_contract(kernel, shapes, meta):
    """sim.check_write_partition twin on the native map VM: every catalog
    kernel's programs write disjoint sets covering each output exactly once
    (sim.py:366-393), and launch(..., collect_writes=True) reports them."""
    ck = C.checked(kernel)
    args = {n: _Fake(s) for n, s in shapes.items()}
    backend.check_write_partition(ck, args, meta)
    w = backend.program_writes(ck, args, meta)
    out = [p.name for p in ck.spec.params if p.role == "out"][0]
    assert sum(len(x) for x in w[out]) == int(np.prod(shapes[out]))
