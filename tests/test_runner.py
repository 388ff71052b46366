"""The B200 artifact runner honours the reference triton_runner contract
(manifest + TWT1 tensors, exit codes 0/1/2/3; triton_runner/cli.py:9-12,
tests/test_runner.py).  Artifacts under tests/golden/runner/ were produced by
the reference CLI (tests/golden/gen_runner_artifacts.py)."""

import json
import shutil
from pathlib import Path

import numpy as np
import pytest

from paper_2507_11978_b200 import runner as R

ART = Path(__file__).resolve().parent / "golden" / "runner"
META = {
    "add": {"BLOCK_SIZE": 4},
    "mm": {"BLOCK_SIZE_M": 2, "BLOCK_SIZE_N": 2, "BLOCK_SIZE_K": 2},
    "addmm": {"BLOCK_SIZE_M": 4, "BLOCK_SIZE_N": 4, "BLOCK_SIZE_K": 8},
    "softmax": {"COLS_PADDED": 32},
    "conv2d": {"BLOCK_SIZE_M": 4, "BLOCK_SIZE_N": 4, "BLOCK_SIZE_K": 4},
}


def _argv(kernel, d=None, expect="expected.twt", meta=None):
    d = d or ART / kernel
    m = R.load_manifest(d / f"{kernel}.manifest.json")
    argv = ["run", "--manifest", str(d / f"{kernel}.manifest.json"), "--expect", str(d / expect)]
    for p in m.params:
        if p.role == "in":
            argv += ["--inputs", f"{p.name}={d / (p.name + '.twt')}"]
    for k, v in (META[kernel] if meta is None else meta).items():
        argv += ["--meta", f"{k}={v}"]
    return argv


def test_manifests_parse():
    for k in META:
        m = R.load_manifest(ART / k / f"{k}.manifest.json")
        assert m.name == k
        assert R.default_tolerance(m) == 1e-4


def test_tensor_round_trip(tmp_path):
    a = np.random.default_rng(0).uniform(-1, 1, (3, 5)).astype(np.float32)
    R.write_tensor(tmp_path / "t.twt", a)
    np.testing.assert_array_equal(R.read_tensor(tmp_path / "t.twt"), a)
    (tmp_path / "bad.twt").write_bytes(b"NOPE" + b"\0" * 16)
    with pytest.raises(R.TensorIOError):
        R.read_tensor(tmp_path / "bad.twt")
    raw = (tmp_path / "t.twt").read_bytes()
    (tmp_path / "trunc.twt").write_bytes(raw[:-4])
    with pytest.raises(R.TensorIOError):
        R.read_tensor(tmp_path / "trunc.twt")
    # the reference writer stores rank-0 scalars (addmm beta) as shape (1,);
    # build_request accepts them for rank-0 params
    assert R.read_tensor(ART / "addmm" / "beta.twt").shape == (1,)
    req = R.build_request(ART / "addmm" / "addmm.manifest.json",
                          {n: ART / "addmm" / f"{n}.twt" for n in ("input", "mat1", "mat2", "beta", "alpha")},
                          ART / "addmm" / "expected.twt", META["addmm"])
    assert req.inputs["beta"].ndim == 0


def test_manifest_errors(tmp_path):
    (tmp_path / "x.json").write_text("{")
    with pytest.raises(R.ManifestError):
        R.load_manifest(tmp_path / "x.json")
    doc = json.loads((ART / "add" / "add.manifest.json").read_text())
    doc["params"][0]["kind"] = "f64"
    (tmp_path / "y.json").write_text(json.dumps(doc))
    with pytest.raises(R.ManifestError):
        R.load_manifest(tmp_path / "y.json")
    doc = json.loads((ART / "add" / "add.manifest.json").read_text())
    doc["launcher_args"] = doc["launcher_args"][::-1]
    (tmp_path / "z.json").write_text(json.dumps(doc))
    with pytest.raises(R.ManifestError):
        R.load_manifest(tmp_path / "z.json")


@pytest.mark.parametrize("mutate", ["missing_input", "extra_input", "missing_meta",
                                    "unknown_meta", "zero_meta", "bad_pair", "no_source"])
def test_usage_errors_exit_2(mutate, tmp_path):
    argv = _argv("add")
    if mutate == "missing_input":
        i = argv.index("--inputs")
        del argv[i:i + 2]
    elif mutate == "extra_input":
        argv += ["--inputs", f"bias={ART / 'add' / 'input.twt'}"]
    elif mutate == "missing_meta":
        argv = _argv("add", meta={})
    elif mutate == "unknown_meta":
        argv += ["--meta", "FOO=3"]
    elif mutate == "zero_meta":
        argv = _argv("add", meta={"BLOCK_SIZE": 0})
    elif mutate == "bad_pair":
        argv += ["--meta", "BLOCK_SIZE"]
    elif mutate == "no_source":
        argv += ["--source", str(tmp_path / "missing.py")]
    assert R.main(argv) == R.EXIT_USAGE


def test_rank_mismatch_exit_2(tmp_path):
    d = tmp_path / "add"
    shutil.copytree(ART / "add", d)
    R.write_tensor(d / "input.twt", np.zeros((2, 5), np.float32))
    assert R.main(_argv("add", d=d)) == R.EXIT_USAGE


def test_no_gpu_exit_3():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    assert R.main(_argv("mm")) == R.EXIT_NO_ENV


@pytest.mark.gpu
@pytest.mark.parametrize("kernel", sorted(META))
def test_runner_passes_on_b200(kernel):
    assert R.main(_argv(kernel)) == R.EXIT_OK


@pytest.mark.gpu
def test_runner_detects_mismatch(tmp_path):
    d = tmp_path / "mm"
    shutil.copytree(ART / "mm", d)
    e = R.read_tensor(d / "expected.twt")
    R.write_tensor(d / "expected.twt", e + 1.0)
    assert R.main(_argv("mm", d=d)) == R.EXIT_FAIL
