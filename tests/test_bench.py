"""bench.py contract on CPU: the reference arm (tiledsl sim.launch from
baseline/_ref, or the oracle port when it is absent) prints the driver's JSON line, and the roofline / L2-rotation helpers
compute what DESIGN.md section 6 says.  The device arm needs a B200."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "3"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC
    assert line["steps"] == 1 and line["warmup"] == 3 and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == ("reference" if bench.reference_available() else "port")
    assert line["config"]["same_config"] and line["config"]["rows"] == bench.R
    assert line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_roofline_fraction():
    w = bench.Work("x", "hbm", 1, lambda n: 1e9 * n, None, None)
    r = bench._roofline(w, 1.0, {"hbm": 2000.0, "tc": 1000.0}, 123)
    assert r["achieved"] == pytest.approx(1000.0) and r["frac"] == pytest.approx(0.5)
    assert r["unit"] == "GB/s" and r["traffic"] == 123
    w = bench.Work("y", "tensor", 2, lambda n: 1e12 * n, None, None)
    r = bench._roofline(w, 2.0, {"hbm": 2000.0, "tc": 1000.0}, None)
    assert r["achieved"] == pytest.approx(1000.0) and r["frac"] == pytest.approx(1.0)
    assert r["unit"] == "TFLOP/s"


def test_rotating_sets_exceed_l2():
    # enough input/output sets that consecutive launches never hit in L2
    for b in (12_582_912, 67_108_864, 134_225_920, 2_148_532_224):
        n = bench._sets_for(b)
        assert n >= 2 and n * b >= 3 * 126e6 or n == 2


def test_peaks_and_traffic_files():
    pk = bench.peaks()
    assert pk["hbm"] > 0 and pk["tc"] > 0
    tr = bench.ncu_traffic()
    assert all(v > 0 for k, v in tr.items() if not k.startswith("_"))


def test_compare_policy():
    ok = bench.compare([1.0, 2.0], [1.0, 2.01], 1e-2, 0.0)
    assert ok["ok"] and ok["max_err"] == pytest.approx(0.01)
    bad = bench.compare([1.0, float("nan")], [1.0, 1.0], 1e-2, 1e-2)
    assert not bad["ok"]


def test_tf32x3_roofline_and_fp32_tolerance():
    # the 3xTF32 legs are judged against dense tf32 (half of bf16) / 3 MMAs
    w = bench.Work("mm_f32", "tensor", 1, lambda n: 1e12 * n, None, None,
                   peak_scale=bench.TF32X3_PEAK_SCALE)
    r = bench._roofline(w, 1.0, {"hbm": 2000.0, "tc": 1200.0}, None)
    assert r["peak"] == pytest.approx(200.0) and r["frac"] == pytest.approx(5.0)
    assert "3xTF32" in r["peak_note"]
    # the reference's 1e-4 (verify.py:24-25) at K <= 64, grown with sqrt(K)
    assert bench.F32_MM_TOL(64) == (1e-5, 1e-4)
    assert bench.F32_MM_TOL(4096)[1] == pytest.approx(8e-4)
    assert all(k in bench.KERNELS for k in ("mm_f32", "bmm_f32", "conv2d_f32"))
