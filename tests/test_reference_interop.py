"""Drop-in check against the reference front end itself (build container
only; /root/reference does not exist on the GPU box, so this module skips
there).  The reference's own CheckedSpec objects must be accepted by the
B200 backend unchanged and compile to the same native map blob as this
package's front end; anything else is rejected (no CPU fallback)."""

import dataclasses
import sys
from pathlib import Path

import numpy as np
import pytest

REF = Path("/root/reference/pkg/src")
if not REF.exists():  # pragma: no cover - GPU box
    pytest.skip("reference tree not present", allow_module_level=True)
sys.path.insert(0, str(REF))

from tiledsl import verify as vf  # noqa: E402
from tiledsl.catalog import CATALOG_NAMES  # noqa: E402
from tiledsl.tileir import typecheck as ref_typecheck  # noqa: E402

from paper_2507_11978_b200 import _lib, backend  # noqa: E402
from paper_2507_11978_b200 import catalog as C  # noqa: E402
from paper_2507_11978_b200.bytecode import build_program  # noqa: E402


@pytest.mark.parametrize("kernel", CATALOG_NAMES)
def test_reference_checked_spec_is_accepted(kernel):
    ref = vf.checked_catalog(kernel)
    family, prog = backend._resolve(ref)
    assert family == kernel
    mine = build_program(C.checked(kernel))
    np.testing.assert_array_equal(prog.blob, mine.blob)
    assert prog.slot_names == mine.slot_names


def test_reference_spec_maps_through_native_vm_match_reference_sim_binding():
    from tiledsl.sim import binding_for

    cfg = vf.Config("conv2d", {"N": 2, "C": 3, "H": 6, "W": 5, "K": 4, "R": 3, "S": 2},
                    {"BLOCK_SIZE_M": 3, "BLOCK_SIZE_N": 2, "BLOCK_SIZE_K": 4})
    ref = vf.checked_catalog("conv2d")
    args = vf.to_concrete(vf.make_inputs("conv2d", cfg, 0))
    binding = binding_for(ref, args, cfg.meta)
    grid = backend.evaluate_grid(ref, binding)
    from tiledsl.symexpr import evaluate
    assert list(grid) == [int(evaluate(s, binding)) for s in ref.grid.sizes]


def test_modified_reference_spec_is_rejected():
    spec = vf.checked_catalog("add").spec
    from tiledsl.tileir import BinOp, Load, Store
    bad = dataclasses.replace(spec, application=(Store("output", BinOp("-", Load("input"),
                                                                       Load("other"))),))
    with pytest.raises(backend.UnsupportedSpecError):
        backend._resolve(ref_typecheck(bad))


class _Fake:
    def __init__(self, shape):
        self.shape = tuple(shape)
        st, acc = [], 1
        for s in reversed(self.shape):
            st.append(acc)
            acc *= s
        self._st = tuple(reversed(st))

    def stride(self):
        return self._st


def test_reference_launch_errors_are_mirrored():
    ref = vf.checked_catalog("rms_norm")
    args = {"input": _Fake((3, 20)), "weight": _Fake((20,)), "output": _Fake((3, 20))}
    with pytest.raises(backend.LaunchError, match="launch-time check failed"):
        backend.launch(ref, args, {"COLS_PADDED": 16})
    with pytest.raises(backend.LaunchError, match="missing meta-parameter"):
        backend.launch(ref, args, {})
