"""Live parity against the reference itself on the GPU box: the UNMODIFIED
reference package (installed under baseline/_ref with pip --target, the same
copy bench.py's reference arm runs; git-ignored, shipped with the snapshot)
builds its own CheckedSpecs and runs its own CPU simulator (`verify.simulate`
= `sim.launch`, verify.py:200-204); the B200 backend launches the SAME
reference CheckedSpec objects (the INTEGRATION.md drop-in usage) on the GPU,
and the outputs are compared with the reference's own tolerances
(verify.py:21-25): fp32 add bit-exact, element-wise 1e-5, reductions and
contractions 1e-4 max-abs.

The shapes are larger than the reference's desk-scale acceptance matrix
(which the committed golden fixtures already cover) and chosen so the
native fast paths run: 16-byte-aligned fp32 strides take the 3xTF32
tensor-core contractions, 4096-wide rows the streaming row kernel.  Skips
when baseline/_ref is absent (it is re-created by the pip install recorded in
DESIGN.md section 6)."""

import sys
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"
if not (REF / "tiledsl" / "sim.py").exists():  # pragma: no cover
    pytest.skip("baseline/_ref (the installed reference) not present", allow_module_level=True)
sys.path.insert(0, str(REF))

from tiledsl import verify as vf  # noqa: E402

from paper_2507_11978_b200 import backend  # noqa: E402

DEV = "cuda:0"
MM_META = {"BLOCK_SIZE_M": 64, "BLOCK_SIZE_N": 64, "BLOCK_SIZE_K": 32}

CASES = [
    ("add", {"N": 1000}, {"BLOCK_SIZE": 256}),
    ("add", {"N": 65537}, {"BLOCK_SIZE": 1024}),
    ("silu", {"N": 4099}, {"BLOCK_SIZE": 1024}),
    ("softmax", {"R": 9, "C": 33}, {"COLS_PADDED": 64}),
    ("softmax", {"R": 64, "C": 4096}, {"COLS_PADDED": 4096}),
    ("softmax", {"R": 16, "C": 1000}, {"COLS_PADDED": 256}),      # per-chunk softmax (CP < C)
    ("rms_norm", {"R": 64, "C": 4096}, {"COLS_PADDED": 4096}),
    ("rms_norm", {"R": 7, "C": 1000}, {"COLS_PADDED": 1024}),
    ("mm", {"M": 100, "N": 72, "K": 40}, MM_META),
    ("mm", {"M": 256, "N": 384, "K": 520}, MM_META),
    ("mm", {"M": 33, "N": 17, "K": 9}, MM_META),                  # unaligned: CUDA-core path
    ("addmm", {"M": 200, "N": 136, "K": 264}, MM_META),
    ("bmm", {"B": 3, "M": 64, "N": 48, "K": 40}, MM_META),
    ("bmm", {"B": 2, "M": 128, "N": 96, "K": 256}, MM_META),
    ("conv2d", {"N": 2, "C": 8, "H": 12, "W": 10, "K": 16, "R": 3, "S": 3}, MM_META),
    ("conv2d", {"N": 1, "C": 32, "H": 20, "W": 20, "K": 64, "R": 3, "S": 3}, MM_META),
    ("conv2d", {"N": 2, "C": 3, "H": 9, "W": 9, "K": 5, "R": 2, "S": 3}, MM_META),
]


@pytest.mark.parametrize("kernel,dims,meta", CASES,
                         ids=[f"{k}-" + "-".join(f"{a}{b}" for a, b in d.items()) for k, d, _ in CASES])
def test_reference_spec_on_gpu_matches_reference_sim(kernel, dims, meta):
    cfg = vf.Config(kernel, dims, meta)
    args = vf.make_inputs(kernel, cfg, seed=7)
    expected = vf.simulate(kernel, args, meta)            # the reference's own CPU path
    checked = vf.checked_catalog(kernel)                  # the reference's own front end
    targs = {k: (float(v) if np.ndim(v) == 0 else torch.from_numpy(np.ascontiguousarray(v)).to(DEV))
             for k, v in args.items()}
    backend.launch(checked, targs, meta)
    torch.cuda.synchronize()
    got = targs["output"].cpu().numpy()
    if kernel == "add":
        assert got.tobytes() == expected.tobytes()
    else:
        err = float(np.abs(got.astype(np.float64) - expected).max())
        assert err <= vf.tolerance_for(kernel), (kernel, dims, err)
