"""GPU parity: the sm_100a kernels (through the C ABI) against the reference's
own outputs (tests/golden) and the CPU oracle.

Tolerances (written here, per BASELINE.json north star):
* fp32 add: bit-exact (sim == oracle == numpy bytes);
* fp32 reductions / contractions vs sim.launch: max-abs <= 1e-4 (the
  reference's own verify tolerance, verify.py:24-25), 1e-5 for silu;
* fp16/bf16: |got - ref| <= atol + rtol*|ref| with rtol = atol = 1e-2 against
  the oracle fed the SAME fp16-rounded inputs (SURVEY 8(c) policy);
* integer maps (probe): bit-exact.
"""

import numpy as np
import pytest

import oracle
from helpers import case_args, map_cases, maps, out_shape, sim_cases

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2507_11978_b200 import _lib, backend  # noqa: E402
from paper_2507_11978_b200 import catalog as C  # noqa: E402
from paper_2507_11978_b200.bytecode import build_program  # noqa: E402

DEV = "cuda:0"
F32_TOL = {"silu": 1e-5}


def _t(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV, dtype)


def _run(kernel, args, meta, dtype=torch.float32, out=None):
    ck = C.checked(kernel)
    targs = {}
    for p in ck.spec.params:
        v = args[p.name] if p.name in args else None
        if p.rank == 0:
            targs[p.name] = float(v)
        elif p.role == "out":
            targs[p.name] = out if out is not None else torch.zeros(
                out_shape(kernel, args), device=DEV, dtype=dtype)
        else:
            targs[p.name] = v if isinstance(v, torch.Tensor) else _t(v, dtype)
    backend.launch(ck, targs, meta)
    torch.cuda.synchronize()
    outs = [targs[p.name] for p in ck.spec.params if p.role == "out"]
    return outs[0]


def test_probe_reproduces_reference_maps_on_gpu():
    index, arrays = map_cases()
    for ci, case in enumerate(index):
        prog = build_program(C.checked(case["kernel"]))
        slots = prog.slots(case["binding"])
        for p in case["params"]:
            q = prog.params.index(p["name"])
            want_o = arrays[f"c{ci}_{p['name']}_offs"].reshape(-1)
            want_m = arrays[f"c{ci}_{p['name']}_mask"].reshape(-1)
            n = want_o.size
            d_off = torch.empty(n, dtype=torch.int64, device=DEV)
            d_mask = torch.empty(n, dtype=torch.uint8, device=DEV)
            cnt = np.zeros(1, dtype=np.int64)
            rc = _lib.lib().ntb_map_probe(
                _lib.i64(prog.blob), len(prog.blob), q, _lib.i64(slots), len(slots),
                d_off.data_ptr(), d_mask.data_ptr(), n, _lib.i64(cnt),
                torch.cuda.current_stream().cuda_stream)
            assert rc == 0, _lib.last_error()
            assert int(cnt[0]) == n
            np.testing.assert_array_equal(d_off.cpu().numpy(), want_o)
            np.testing.assert_array_equal(d_mask.cpu().numpy(), want_m)


@pytest.mark.parametrize("kernel", C.CATALOG_NAMES)
def test_fp32_matches_reference_simulator(kernel):
    """Acceptance matrix (test_acceptance.py:44-64) + test_sim.py cases."""
    index, arrays = sim_cases()
    n = 0
    for ci, case in enumerate(index):
        if case["kernel"] != kernel:
            continue
        args = case_args(ci, case, arrays)
        got = _run(kernel, args, case["meta"]).cpu().numpy()
        sim = arrays[f"c{ci}_sim"]
        if kernel == "add":
            assert got.tobytes() == sim.tobytes(), case
        else:
            err = float(np.max(np.abs(got.astype(np.float64) - sim))) if sim.size else 0.0
            assert err <= F32_TOL.get(kernel, 1e-4), (case["dims"], case["meta"], err)
        n += 1
    assert n >= 20


class _Paths:
    """Delta of native path launch counters across a block."""

    def __enter__(self):
        self.before = backend.path_counts()
        return self

    def __exit__(self, *exc):
        after = backend.path_counts()
        self.delta = {k: after[k] - self.before[k] for k in after}


def _close(got, ref, rtol=1e-2, atol=1e-2):
    got = got.float().cpu().numpy().astype(np.float64)
    assert np.isfinite(got).all(), f"{(~np.isfinite(got)).sum()} non-finite outputs"
    bad = ~(np.abs(got - ref) <= atol + rtol * np.abs(ref))
    assert not bad.any(), f"{bad.sum()} of {bad.size} outside tol; max err " \
                          f"{np.max(np.abs(got - ref)):.3e}"


def _r16(a, dtype):
    """Round to the device dtype and return the exact upcast (oracle input)."""
    return torch.from_numpy(a).to(dtype).float().numpy()


DTS = [torch.float16, torch.bfloat16]


@pytest.mark.parametrize("dtype", DTS)
# 8000: a partial last chunk in the streaming kernel; the last size gives
# every warp of a 148-SM grid two full chunks and a ragged third
@pytest.mark.parametrize("n", [1, 37, 4096, 8000, 1 << 20, 8 * (512 * 148 * 16 * 2 + 77)])
def test_elementwise_half(dtype, n):
    rng = np.random.default_rng(n)
    a, b = (_r16(rng.uniform(-1, 1, n).astype(np.float32), dtype) for _ in range(2))
    got = _run("add", {"input": a, "other": b}, {"BLOCK_SIZE": 1024}, dtype)
    _close(got, oracle.add(a, b), rtol=1e-2, atol=1e-3)
    got = _run("silu", {"input": a}, {"BLOCK_SIZE": 1024}, dtype)
    _close(got, oracle.silu(a), rtol=1e-2, atol=1e-3)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float16, torch.bfloat16])
def test_silu_magnitude_sweep(dtype):
    """silu pairs two elements on one reciprocal while d0*d1 < 2^126 and falls
    back to one reciprocal each beyond (k_elementwise.cu SiluOp): inputs from
    1e-3 to 1e4 in magnitude, both signs, so pairs straddle the fallback
    (x < -43), plus exact zeros and a ragged tail."""
    rng = np.random.default_rng(11)
    parts = [rng.normal(0, s, 4096) for s in (1e-3, 0.1, 1.0, 10.0, 30.0, 100.0, 1e4)]
    x = np.concatenate(parts + [np.zeros(64), np.array([-43.0, -44.0, -90.0, 88.0, -1e30, 1e30])])
    x = rng.permutation(x.astype(np.float32))
    if dtype != torch.float32:
        x = np.clip(x, -6e4, 6e4) if dtype == torch.float16 else x
        x = _r16(x, dtype)
    before = backend.path_counts()
    for n in ((x.size // 8) * 8, (x.size // 8) * 8 - 3):   # vector path, then the strided one
        got = _run("silu", {"input": x[:n]}, {"BLOCK_SIZE": 1024}, dtype)
        ref = oracle.silu(x[:n]).astype(np.float64)
        if dtype == torch.float32:
            _close(got, ref, rtol=1e-5, atol=1e-30)
        else:
            _close(got, ref, rtol=1e-2, atol=1e-3)
    d = {k: v - before.get(k, 0) for k, v in backend.path_counts().items()}
    assert d["ew_generic"] == 1 and d["ew_vec"] + d["ew_stream"] == 1, d


@pytest.mark.parametrize("n", [(1 << 24), (1 << 24) + 4 * 77])
def test_add_fp32_streaming_bit_exact(n):
    """>= 32 MB per launch takes the bulk-copy streaming kernel (ew_stream):
    still byte-identical to the oracle / sim (fp32 a + b, one rounding)."""
    rng = np.random.default_rng(n)
    a, b = (rng.uniform(-1, 1, n).astype(np.float32) for _ in range(2))
    with _Paths() as pc:
        got = _run("add", {"input": a, "other": b}, {"BLOCK_SIZE": 1024}).cpu().numpy()
    assert pc.delta["ew_stream"] == 1, pc.delta
    assert got.tobytes() == oracle.add(a, b).tobytes()


def test_add_fp32_large_bit_exact():
    rng = np.random.default_rng(7)
    n = (1 << 20) + 3
    a, b = (rng.uniform(-1, 1, n).astype(np.float32) for _ in range(2))
    got = _run("add", {"input": a, "other": b}, {"BLOCK_SIZE": 1024}).cpu().numpy()
    assert got.tobytes() == oracle.add(a, b).tobytes()


@pytest.mark.parametrize("dtype", DTS + [torch.float32])
@pytest.mark.parametrize("shape", [(7, 13), (64, 1000), (256, 4096), (3, 8192)])
def test_rowwise(dtype, shape):
    rng = np.random.default_rng(shape[1])
    x = _r16(rng.uniform(-1, 1, shape).astype(np.float32), dtype)
    w = _r16(rng.uniform(-1, 1, shape[1]).astype(np.float32), dtype)
    cp = 1 << (shape[1] - 1).bit_length()
    tol = 1e-5 if dtype == torch.float32 else 1e-2
    with _Paths() as pc:
        got = _run("softmax", {"input": x}, {"COLS_PADDED": cp}, dtype)
    _close(got, oracle.softmax(x, cp), rtol=tol, atol=tol * 1e-2)
    if shape[1] == 4096 and dtype != torch.float32:
        assert pc.delta["row_stream"] == 1
    got = _run("rms_norm", {"input": x, "weight": w}, {"COLS_PADDED": cp}, dtype)
    _close(got, oracle.rms_norm(x, w), rtol=tol, atol=tol)


@pytest.mark.parametrize("scale", [1.0, 30.0, 3000.0])
def test_rows_fp16_large_magnitudes(scale):
    """Packed-fp16 row math stays accurate for large logits / activations."""
    rng = np.random.default_rng(int(scale))
    x = _r16((rng.standard_normal((64, 4096)) * scale).astype(np.float32), torch.float16)
    w = _r16(rng.uniform(-1, 1, 4096).astype(np.float32), torch.float16)
    got = _run("softmax", {"input": x}, {"COLS_PADDED": 4096}, torch.float16)
    _close(got, oracle.softmax(x, 4096), rtol=1e-2, atol=1e-4)
    got = _run("rms_norm", {"input": x, "weight": w}, {"COLS_PADDED": 4096}, torch.float16)
    _close(got, oracle.rms_norm(x, w), rtol=1e-2, atol=1e-2)


@pytest.mark.parametrize("dtype", DTS)
@pytest.mark.parametrize("cols", [4096, 1000, 8192])
@pytest.mark.parametrize("std", [0.01, 0.05, 0.1, 0.3, 1.0, 100.0])
def test_rows_magnitude_sweep(dtype, cols, std):
    """16-bit rows are computed in fp32 (the reference simulates in f32,
    catalog.py:155-223): the only 16-bit rounding is the store,
    so the result must sit within ~one output ulp of the f32 oracle at EVERY
    activation scale, small ones included (sum of squares of N(0, 0.01^2)
    must not underflow), plus an all-zero row (softmax -> 1/C, rms -> 0).
    Tolerance: rtol = 2 ulp of the 16-bit type (fp16 2^-9, bf16 2^-6) and an
    atol at the type's subnormal spacing."""
    rng = np.random.default_rng(int(std * 1000) + cols)
    x = (rng.standard_normal((96, cols)) * std).astype(np.float32)
    x[5] = 0.0
    x = _r16(x, dtype)
    w = _r16(rng.uniform(-1, 1, cols).astype(np.float32), dtype)
    rtol = 2.0 ** -9 if dtype == torch.float16 else 2.0 ** -6
    atol = 1e-7 if dtype == torch.float16 else 1e-30
    got = _run("softmax", {"input": x}, {"COLS_PADDED": cols}, dtype)
    _close(got, oracle.softmax(x, cols).astype(np.float64), rtol=rtol, atol=atol)
    np.testing.assert_allclose(got[5].float().cpu().numpy(), 1.0 / cols, rtol=rtol)
    got = _run("rms_norm", {"input": x, "weight": w}, {"COLS_PADDED": cols}, dtype)
    _close(got, oracle.rms_norm(x, w).astype(np.float64), rtol=rtol, atol=atol)
    assert not got[5].any()


def test_softmax_chunked_matches_reference_semantics():
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, (3, 20)).astype(np.float32)
    got = _run("softmax", {"input": x}, {"COLS_PADDED": 8}).cpu().numpy()
    np.testing.assert_allclose(got, oracle.softmax(x, 8), rtol=1e-5, atol=1e-7)
    np.testing.assert_allclose(got.sum(1), 3.0, rtol=1e-5)


@pytest.mark.parametrize("dtype", DTS)
@pytest.mark.parametrize("mnk", [(128, 128, 64), (256, 512, 320), (1000, 520, 700),
                                 (4096, 4096, 4096)])
def test_mm_half(dtype, mnk):
    m, n, k = mnk
    rng = np.random.default_rng(m + n + k)
    a = _r16(rng.uniform(-1, 1, (m, k)).astype(np.float32), dtype)
    b = _r16(rng.uniform(-1, 1, (k, n)).astype(np.float32), dtype)
    meta = {"BLOCK_SIZE_M": 128, "BLOCK_SIZE_N": 128, "BLOCK_SIZE_K": 64}
    with _Paths() as pc:
        got = _run("mm", {"input": a, "other": b}, meta, dtype)
    aligned = k % 8 == 0 and n % 8 == 0
    assert pc.delta["gemm_tc" if aligned else "gemm_generic"] == 1
    rows = np.arange(m) if m <= 1024 else rng.choice(m, 256, replace=False)
    ref = oracle.mm(a[rows], b)
    _close(got[torch.as_tensor(rows, device=DEV)], ref, rtol=1e-2, atol=2e-2)


@pytest.mark.parametrize("dtype", DTS)
@pytest.mark.parametrize("kernel,shape", [("mm", (2560, 4096, 1024)), ("addmm", (2560, 4096, 1024)),
                                          ("bmm", (3, 1536, 1280, 512))])
def test_gemm_narrow_tail(dtype, kernel, shape):
    """Tile counts that leave the last wave of the 74 CTA pairs less than half
    full (160 and 90 tiles) run the tail tiles as two 256 x 128 halves (N = 128
    MMAs) on two pairs; every output element is checked, over two launches."""
    rng = np.random.default_rng(len(shape) + shape[-1])
    meta = {"BLOCK_SIZE_M": 128, "BLOCK_SIZE_N": 128, "BLOCK_SIZE_K": 64}
    if kernel == "bmm":
        bt, m, n, k = shape
        a = _r16(rng.uniform(-1, 1, (bt, m, k)).astype(np.float32), dtype)
        b = _r16(rng.uniform(-1, 1, (bt, k, n)).astype(np.float32), dtype)
        args, ref = {"input": a, "other": b}, oracle.bmm(a, b)
    else:
        m, n, k = shape
        a = _r16(rng.uniform(-1, 1, (m, k)).astype(np.float32), dtype)
        b = _r16(rng.uniform(-1, 1, (k, n)).astype(np.float32), dtype)
        if kernel == "mm":
            args, ref = {"input": a, "other": b}, oracle.mm(a, b)
        else:
            inp = _r16(rng.uniform(-1, 1, (m, n)).astype(np.float32), dtype)
            args = {"input": inp, "mat1": a, "mat2": b, "beta": 0.5, "alpha": -1.5}
            ref = oracle.addmm(inp, a, b, 0.5, -1.5)
    for _ in range(2):
        got = _run(kernel, args, meta, dtype)
        _close(got, ref, rtol=1e-2, atol=3e-2)


@pytest.mark.parametrize("dtype", DTS)
def test_mm_transposed_operands(dtype):
    rng = np.random.default_rng(3)
    m, n, k = 384, 256, 512
    a = _r16(rng.uniform(-1, 1, (k, m)).astype(np.float32), dtype)
    b = _r16(rng.uniform(-1, 1, (n, k)).astype(np.float32), dtype)
    ta, tb = _t(a, dtype).t(), _t(b, dtype).t()     # M-major A, N-major... views
    meta = {"BLOCK_SIZE_M": 64, "BLOCK_SIZE_N": 64, "BLOCK_SIZE_K": 32}
    with _Paths() as pc:
        got = _run("mm", {"input": ta, "other": tb}, meta, dtype)
    assert pc.delta["gemm_tc"] == 1
    _close(got, oracle.mm(a.T, b.T), rtol=1e-2, atol=2e-2)


@pytest.mark.parametrize("dtype", DTS)
def test_addmm_half(dtype):
    rng = np.random.default_rng(11)
    m, n, k = 512, 384, 256
    inp = _r16(rng.uniform(-1, 1, (m, n)).astype(np.float32), dtype)
    a = _r16(rng.uniform(-1, 1, (m, k)).astype(np.float32), dtype)
    b = _r16(rng.uniform(-1, 1, (k, n)).astype(np.float32), dtype)
    meta = {"BLOCK_SIZE_M": 128, "BLOCK_SIZE_N": 128, "BLOCK_SIZE_K": 64}
    got = _run("addmm", {"input": inp, "mat1": a, "mat2": b, "beta": -0.134, "alpha": -0.201},
               meta, dtype)
    _close(got, oracle.addmm(inp, a, b, -0.134, -0.201), rtol=1e-2, atol=1e-2)


@pytest.mark.parametrize("dtype", DTS)
@pytest.mark.parametrize("bmnk", [(3, 100, 72, 40), (8, 256, 256, 256), (64, 1024, 1024, 1024)])
def test_bmm_half(dtype, bmnk):
    bt, m, n, k = bmnk
    rng = np.random.default_rng(bt)
    a = _r16(rng.uniform(-1, 1, (bt, m, k)).astype(np.float32), dtype)
    b = _r16(rng.uniform(-1, 1, (bt, k, n)).astype(np.float32), dtype)
    meta = {"BLOCK_SIZE_M": 128, "BLOCK_SIZE_N": 128, "BLOCK_SIZE_K": 64}
    with _Paths() as pc:
        got = _run("bmm", {"input": a, "other": b}, meta, dtype)
    assert pc.delta["gemm_tc"] == 1
    sel = [0, bt - 1]
    _close(got[sel], oracle.bmm(a[sel], b[sel]), rtol=1e-2, atol=2e-2)


@pytest.mark.parametrize("dtype", DTS)
@pytest.mark.parametrize("shape", [(1, 2, 5, 5, 3, 3, 3), (2, 16, 12, 10, 32, 3, 3),
                                   (2, 64, 30, 30, 128, 3, 3), (4, 256, 56, 56, 256, 3, 3),
                                   (3, 100, 17, 23, 320, 5, 5), (9, 64, 40, 40, 64, 1, 1),
                                   (20, 96, 28, 28, 192, 3, 3), (8, 64, 56, 56, 64, 3, 3)])
def test_conv2d_half(dtype, shape):
    n, c, h, w, k, r, s = shape
    rng = np.random.default_rng(c)
    x = _r16(rng.uniform(-1, 1, (n, c, h, w)).astype(np.float32), dtype)
    f = _r16(rng.uniform(-1, 1, (k, c, r, s)).astype(np.float32), dtype)
    meta = {"BLOCK_SIZE_M": 128, "BLOCK_SIZE_N": 128, "BLOCK_SIZE_K": 64}
    with _Paths() as pc:
        got = _run("conv2d", {"input": x, "filter": f}, meta, dtype)
    if (h * w) % 8 == 0:
        assert pc.delta["conv_tc"] == 1
    _close(got, oracle.conv2d(x, f), rtol=1e-2, atol=3e-2)


@pytest.mark.parametrize("dtype", DTS)
@pytest.mark.parametrize("bhsd", [(1, 2, 64, 64), (2, 3, 200, 128), (1, 2, 1024, 128),
                                  (2, 2, 333, 64), (4, 40, 520, 128)])
def test_sdpa_half(dtype, bhsd):
    b, h, s, d = bhsd
    rng = np.random.default_rng(s)
    q, k, v = (_r16(rng.uniform(-1, 1, (b, h, s, d)).astype(np.float32), dtype)
               for _ in range(3))
    with _Paths() as pc:
        got = _run("sdpa", {"q": q, "k": k, "v": v, "o": None},
                   {"BLOCK_SIZE_M": 128, "BLOCK_SIZE_N": 128}, dtype,
                   out=torch.zeros((b, h, s, d), device=DEV, dtype=dtype))
    assert pc.delta["attn_tc"] == 1
    _close(got, oracle.sdpa(q, k, v), rtol=1e-2, atol=1e-2)


@pytest.mark.parametrize("d", [64, 128])
def test_sdpa_peaky_scores_rescale(d):
    """Scores spanning > 2^8 between KV tiles (the lazy O rescale path) and
    more work items than SMs (persistent CTAs carry barrier phases across
    items)."""
    rng = np.random.default_rng(11)
    b, h, s = 3, 64, 700
    q = _r16((rng.standard_normal((b, h, s, d)) * 3).astype(np.float32), torch.float16)
    k = _r16((rng.standard_normal((b, h, s, d)) * 3).astype(np.float32), torch.float16)
    v = _r16(rng.uniform(-1, 1, (b, h, s, d)).astype(np.float32), torch.float16)
    got = _run("sdpa", {"q": q, "k": k, "v": v, "o": None},
               {"BLOCK_SIZE_M": 128, "BLOCK_SIZE_N": 128}, torch.float16,
               out=torch.zeros((b, h, s, d), device=DEV, dtype=torch.float16))
    _close(got, oracle.sdpa(q, k, v), rtol=1e-2, atol=1e-2)


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("bhs", [(1, 80, 512), (2, 37, 700), (1, 1, 256), (1, 74, 256)])
def test_sdpa_tail_split(d, bhs):
    """Work-unit schedule (k_attn_sm100.cu launch_attn): full two-tile items
    round-robin, then the last round's items as single-tile units on twice as
    many CTAs (160 items on 148 SMs: 148 full + 24 single-tile units; 222
    items: 148 + 148; 1 and 74 items: single-tile units only), with peaky
    scores so the lazy O rescale runs inside single-tile units too.  Checked
    against the oracle, and relaunches are bit-identical."""
    b, h, s = bhs
    rng = np.random.default_rng(s + h + d)
    q = _r16((rng.standard_normal((b, h, s, d)) * 3).astype(np.float32), torch.float16)
    k = _r16((rng.standard_normal((b, h, s, d)) * 3).astype(np.float32), torch.float16)
    v = _r16(rng.uniform(-1, 1, (b, h, s, d)).astype(np.float32), torch.float16)
    tq, tk, tv = (_t(x, torch.float16) for x in (q, k, v))
    outs = []
    for _ in range(2):
        o = torch.zeros((b, h, s, d), device=DEV, dtype=torch.float16)
        with _Paths() as pc:
            backend.sdpa_launch(tq, tk, tv, o, 128, 128)
            torch.cuda.synchronize()
        assert pc.delta["attn_tc"] == 1
        outs.append(o)
    assert torch.equal(outs[0], outs[1])
    _close(outs[0], oracle.sdpa(q, k, v), rtol=1e-2, atol=1e-2)


@pytest.mark.parametrize("dtype", DTS)
@pytest.mark.parametrize("bshd", [(1, 256, 2, 64), (2, 300, 3, 128), (2, 1024, 4, 128),
                                  (3, 700, 40, 64), (1, 520, 64, 128)])
def test_sdpa_rope_fused(dtype, bshd):
    """sdpa(rope(q), rope(k), v) in ONE kernel (rotary embedding applied in
    shared memory between the TMA loads and the MMAs) against (1) the oracle
    fed the rotated Q/K rounded to the device dtype, as the device rounds them
    before its 16-bit products, and (2) the unfused rope_launch x2 +
    sdpa_launch pipeline.  Q/K/V are (B, S, H, D) storage viewed as
    (B, H, S, D), the paper's layout."""
    b, s, h, d = bshd
    rng = np.random.default_rng(s + d)
    base = [_r16(rng.uniform(-1, 1, (b, s, h, d)).astype(np.float32), dtype) for _ in range(3)]
    ang = rng.uniform(-3, 3, (s, d // 2))
    sn = _r16(np.sin(ang).astype(np.float32), dtype)
    cs = _r16(np.cos(ang).astype(np.float32), dtype)
    tq, tk, tv = (_t(x, dtype) for x in base)
    tsn, tcs = _t(sn, dtype), _t(cs, dtype)
    q, k, v = (t.transpose(1, 2) for t in (tq, tk, tv))
    o = torch.zeros((b, h, s, d), device=DEV, dtype=dtype)
    with _Paths() as pc:
        backend.sdpa_rope_launch(q, k, v, tsn, tcs, tsn, tcs, o, 128, 128)
        torch.cuda.synchronize()
    assert pc.delta["attn_tc"] == 1

    def rot(x):
        r = oracle.rope_bhsd(np.swapaxes(x, 1, 2), sn, cs)
        return torch.from_numpy(r.astype(np.float32)).to(dtype).float().numpy()

    ref = oracle.sdpa(rot(base[0]), rot(base[1]), np.swapaxes(base[2], 1, 2))
    _close(o, ref, rtol=1e-2, atol=1e-2)
    # unfused pipeline on the same inputs
    qr, kr = torch.empty_like(tq), torch.empty_like(tk)
    backend.rope_launch(tq, tsn, tcs, qr, d // 2)
    backend.rope_launch(tk, tsn, tcs, kr, d // 2)
    o2 = torch.zeros_like(o)
    backend.sdpa_launch(qr.transpose(1, 2), kr.transpose(1, 2), v, o2, 128, 128)
    torch.cuda.synchronize()
    assert (o.float() - o2.float()).abs().max().item() <= 2e-3


@pytest.mark.parametrize("bshd", [(3, 1024, 4, 128), (5, 1024, 8, 64)])  # 1 MB per batch
def test_sdpa_rope_chunked_workspace(bshd, monkeypatch):
    """The rotated K lives in workspace one batch chunk at a time
    (NTB_ROPE_WS_MB cap): a 1 MB cap forces one batch per chunk, and the
    output must be byte-identical to the single-chunk run (the chunking only
    changes which launch a (b, h) unit lands in)."""
    b, s, h, d = bshd
    g = torch.Generator(device=DEV).manual_seed(b * s + d)
    base = [(torch.rand((b, s, h, d), generator=g, device=DEV) * 2 - 1).half() for _ in range(3)]
    ang = torch.rand((s, d // 2), generator=g, device=DEV) * 6 - 3
    sn, cs = torch.sin(ang).half(), torch.cos(ang).half()
    q, k, v = (t.transpose(1, 2) for t in base)
    outs = []
    for cap, launches in (("4096", 1), ("1", b)):
        monkeypatch.setenv("NTB_ROPE_WS_MB", cap)
        o = torch.full((b, h, s, d), float("nan"), device=DEV, dtype=torch.float16)
        with _Paths() as pc:
            backend.sdpa_rope_launch(q, k, v, sn, cs, sn, cs, o, 128, 128)
            torch.cuda.synchronize()
        assert pc.delta["attn_tc"] == launches
        outs.append(o)
    assert torch.equal(outs[0], outs[1])


def _attn_fp32(q, k, v):
    """Exact attention in fp32 on the GPU, one batch at a time (no TF32):
    the all-heads check at the BASELINE shape."""
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        out = torch.empty(q.shape, device=DEV, dtype=torch.float32)
        for b in range(q.shape[0]):
            qb, kb, vb = (t[b].float() for t in (q, k, v))
            s_ = (qb @ kb.transpose(-1, -2)) * (1.0 / np.sqrt(q.shape[-1]))
            out[b] = torch.softmax(s_, dim=-1) @ vb
        return out
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def _attn_close_all_heads(o, ref, rtol=1e-2, atol=1e-2):
    bad = ((o.float() - ref).abs() > atol + rtol * ref.abs()).sum().item()
    assert bad == 0, f"{bad} outputs outside tol; max err {(o.float() - ref).abs().max().item():.3e}"


# deterministic head subset checked against the f64 oracle (first, last and
# a few in between)
_BASELINE_HEADS = [(0, 0), (5, 17), (13, 31), (22, 3), (31, 31)]


def test_sdpa_baseline_shape():
    """B32 H32 S4096 D128 (BASELINE configs[4]): 32 KV tiles per query block,
    many lazy-rescale events.  All heads vs exact fp32 attention on the GPU,
    a head subset vs the f64 oracle."""
    g = torch.Generator(device=DEV).manual_seed(4096)
    shp = (32, 32, 4096, 128)
    q, k, v = ((torch.rand(shp, generator=g, device=DEV) * 2 - 1).half() for _ in range(3))
    o = torch.empty(shp, device=DEV, dtype=torch.float16)
    with _Paths() as pc:
        backend.sdpa_launch(q, k, v, o, 128, 128)
        torch.cuda.synchronize()
    assert pc.delta["attn_tc"] == 1
    _attn_close_all_heads(o, _attn_fp32(q, k, v))
    for b, h in _BASELINE_HEADS:
        ref = oracle.sdpa(q[b, h].float().cpu().numpy(), k[b, h].float().cpu().numpy(),
                          v[b, h].float().cpu().numpy())
        _close(o[b, h], ref)


def test_sdpa_rope_baseline_shape():
    """sdpa(rope(q), rope(k), v) at B32 H32 S4096 D128 with (B, S, H, D)
    storage: all heads vs fp32 attention over the rotated (device-rounded)
    Q/K, a head subset vs the f64 oracle."""
    g = torch.Generator(device=DEV).manual_seed(4097)
    b_, s_, h_, d_ = 32, 4096, 32, 128
    base = [(torch.rand((b_, s_, h_, d_), generator=g, device=DEV) * 2 - 1).half() for _ in range(3)]
    ang = torch.rand((s_, d_ // 2), generator=g, device=DEV) * 6 - 3
    sn, cs = torch.sin(ang).half(), torch.cos(ang).half()
    q, k, v = (t.transpose(1, 2) for t in base)
    o = torch.empty((b_, h_, s_, d_), device=DEV, dtype=torch.float16)
    backend.sdpa_rope_launch(q, k, v, sn, cs, sn, cs, o, 128, 128)
    torch.cuda.synchronize()

    def rot(x):                                  # (B, H, S, D) fp32 rotation, then fp16
        x = x.float()
        c, s = cs.float()[None, None], sn.float()[None, None]
        x0, x1 = x[..., :d_ // 2], x[..., d_ // 2:]
        return torch.cat([x0 * c - x1 * s, x0 * s + x1 * c], -1).half()

    qr, kr = rot(q), rot(k)
    _attn_close_all_heads(o, _attn_fp32(qr, kr, v))
    del qr, kr
    snp, csp = sn.float().cpu().numpy(), cs.float().cpu().numpy()
    for b, h in _BASELINE_HEADS[:3]:
        qq, kk, vv = (t[b:b + 1, h:h + 1].float().cpu().numpy() for t in (q, k, v))
        ref = oracle.sdpa_rope(qq, kk, vv, snp, csp, snp, csp, round_to=np.float16)[0, 0]
        _close(o[b, h], ref)


def test_repeat_launch_bit_identity():
    """The reference pins reversed / repeated launches as bit-identical
    (test_acceptance.py:165-172).  The persistent / narrow-tail schedules here
    must be too: launch each twice (and once more after other work) and
    compare bytes."""
    g = torch.Generator(device=DEV).manual_seed(3)

    def U(*shape):
        return (torch.rand(shape, generator=g, device=DEV) * 2 - 1).half()

    cases = []
    a, b = U(2560, 1024), U(1024, 4096)          # mm with a narrow tail wave
    cases.append(lambda out: backend.mm_launch(a, b, out, 128, 128, 64))
    x, w = U(4, 64, 30, 30), U(256, 64, 3, 3)    # conv2d, several tiles + tail
    cases.append(lambda out: backend.conv2d_launch(x, w, out, 128, 128, 64))
    q, k, v = U(3, 64, 700, 128), U(3, 64, 700, 128), U(3, 64, 700, 128)   # > 148 items
    cases.append(lambda out: backend.sdpa_launch(q, k, v, out, 128, 128))
    shapes = [(2560, 4096), (4, 256, 28, 28), (3, 64, 700, 128)]
    firsts = []
    for fn, shp in zip(cases, shapes):
        o1, o2 = (torch.full(shp, float("nan"), device=DEV, dtype=torch.float16) for _ in range(2))
        fn(o1)
        fn(o2)
        torch.cuda.synchronize()
        assert torch.equal(o1, o2)
        firsts.append((fn, o1))
    for fn, ref in firsts:                       # again, after everything else ran
        o3 = torch.full(ref.shape, float("nan"), device=DEV, dtype=torch.float16)
        fn(o3)
        torch.cuda.synchronize()
        assert torch.equal(o3, ref)


def test_sdpa_strided_views():
    """(B, S, H, D) storage viewed as (B, H, S, D) (rope output layout)."""
    rng = np.random.default_rng(5)
    b, s, h, d = 2, 256, 4, 64
    base = [_t(rng.uniform(-1, 1, (b, s, h, d)).astype(np.float32), torch.float16)
            for _ in range(3)]
    q, k, v = (t.transpose(1, 2) for t in base)
    out = torch.zeros((b, h, s, d), device=DEV, dtype=torch.float16)
    got = _run("sdpa", {"q": q, "k": k, "v": v}, {"BLOCK_SIZE_M": 64, "BLOCK_SIZE_N": 64},
               torch.float16, out=out)
    ref = oracle.sdpa(*(t.float().cpu().numpy() for t in (q, k, v)))
    _close(got, ref, rtol=1e-2, atol=1e-2)


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("olayout", ["bshd", "offset16", "inner2"])
def test_sdpa_output_layouts(d, olayout):
    """The epilogue's store paths: O through TMA stores staged in shared
    memory (any 16-byte-aligned unit-inner-stride layout: (B, S, H, D)
    storage viewed as (B, H, S, D); a base 16 but not 32 bytes aligned) and
    the direct-store fallback (inner stride 2), with S_q not a multiple of
    the 32-row store box; multi-unit schedules (148+ units)."""
    rng = np.random.default_rng(d)
    b, h, s = 2, 80, 333
    q, k, v = (_r16(rng.uniform(-1, 1, (b, h, s, d)).astype(np.float32), torch.float16)
               for _ in range(3))
    if olayout == "bshd":
        store = torch.zeros((b, s, h, d), device=DEV, dtype=torch.float16)
        o = store.transpose(1, 2)
    elif olayout == "offset16":
        store = torch.zeros(b * h * s * d + 8, device=DEV, dtype=torch.float16)
        o = store[8:].view(b, h, s, d)
    else:
        store = torch.zeros((b, h, s, 2 * d), device=DEV, dtype=torch.float16)
        o = store[..., ::2]
    with _Paths() as pc:
        backend.sdpa_launch(*(_t(x, torch.float16) for x in (q, k, v)), o, 128, 128)
        torch.cuda.synchronize()
    assert pc.delta["attn_tc"] == 1
    _close(o, oracle.sdpa(q, k, v), rtol=1e-2, atol=1e-2)
    if olayout == "inner2":   # the interleaved columns were not touched
        assert torch.count_nonzero(store[..., 1::2]).item() == 0


@pytest.mark.parametrize("dtype", DTS + [torch.float32])
@pytest.mark.parametrize("shape", [(1, 4, 2, 16), (2, 64, 8, 128), (2, 128, 32, 64)])
def test_rope(dtype, shape):
    b, s, h, d = shape
    rng = np.random.default_rng(d)
    x = _r16(rng.uniform(-1, 1, shape).astype(np.float32), dtype)
    ang = rng.uniform(-3, 3, (s, d // 2))
    sn, cs = (_r16(np.sin(ang).astype(np.float32), dtype), _r16(np.cos(ang).astype(np.float32), dtype))
    out = torch.zeros(shape, device=DEV, dtype=dtype)
    got = _run("rope", {"input": x, "sin": sn, "cos": cs}, {"HALF_D": d // 2}, dtype, out=out)
    tol = 1e-5 if dtype == torch.float32 else 1e-2
    _close(got, oracle.rope(x, sn, cs), rtol=tol, atol=tol)


@pytest.mark.parametrize("dtype", DTS)
@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, False), (True, True)])
def test_mm_all_operand_majors(dtype, a_mn, b_mn):
    """K-major / MN-major A and B (every UMMA descriptor combination)."""
    rng = np.random.default_rng(17)
    m, n, k = 320, 288, 192
    a = _r16(rng.uniform(-1, 1, (m, k)).astype(np.float32), dtype)
    b = _r16(rng.uniform(-1, 1, (k, n)).astype(np.float32), dtype)
    ta = _t(a.T.copy(), dtype).t() if a_mn else _t(a, dtype)
    tb = _t(b, dtype) if b_mn else _t(b.T.copy(), dtype).t()
    with _Paths() as pc:
        got = _run("mm", {"input": ta, "other": tb}, {"BLOCK_SIZE_M": 16, "BLOCK_SIZE_N": 16,
                                                      "BLOCK_SIZE_K": 16}, dtype)
    assert pc.delta["gemm_tc"] == 1
    _close(got, oracle.mm(a, b), rtol=1e-2, atol=2e-2)


def test_mm_unaligned_takes_generic_gpu_path():
    rng = np.random.default_rng(2)
    a = rng.uniform(-1, 1, (33, 13)).astype(np.float16).astype(np.float32)
    b = rng.uniform(-1, 1, (13, 7)).astype(np.float16).astype(np.float32)
    with _Paths() as pc:
        got = _run("mm", {"input": a, "other": b}, {"BLOCK_SIZE_M": 16, "BLOCK_SIZE_N": 16,
                                                    "BLOCK_SIZE_K": 16}, torch.float16)
    assert pc.delta["gemm_generic"] == 1
    _close(got, oracle.mm(a, b), rtol=1e-2, atol=1e-2)


def test_launch_counter_proves_native_path():
    before = backend.launch_count()
    _run("add", {"input": np.ones(10, np.float32), "other": np.ones(10, np.float32)},
         {"BLOCK_SIZE": 4})
    assert backend.launch_count() == before + 1


def test_cpu_tensors_are_rejected():
    a = torch.ones(8)
    with pytest.raises(backend.LaunchError, match="CUDA tensor"):
        backend.add_launch(a, a, torch.empty(8), 4)


@pytest.mark.parametrize("case", ["add", "silu", "softmax", "rms_norm", "mm_m0", "bmm_b0",
                                  "conv_n0", "sdpa_b0", "rope_s0"])
def test_empty_grid_is_a_launch_error_like_the_reference(case):
    """An empty grid raises LaunchError("grid dimension evaluated to 0"),
    exactly as sim.launch does (sim.py:180-182)."""
    f16 = torch.float16
    z = lambda *s, dt=f16: torch.zeros(s, device=DEV, dtype=dt)  # noqa: E731
    calls = {
        "add": lambda: backend.add_launch(z(0, dt=torch.float32), z(0, dt=torch.float32),
                                          z(0, dt=torch.float32), 1024),
        "silu": lambda: backend.silu_launch(z(0), z(0), 1024),
        "softmax": lambda: backend.softmax_launch(z(0, 64), z(0, 64), 64),
        "rms_norm": lambda: backend.rms_norm_launch(z(0, 64), z(64), z(0, 64), 64),
        "mm_m0": lambda: backend.mm_launch(z(0, 64), z(64, 32), z(0, 32), 64, 64, 32),
        "bmm_b0": lambda: backend.bmm_launch(z(0, 64, 64), z(0, 64, 64), z(0, 64, 64), 64, 64, 32),
        "conv_n0": lambda: backend.conv2d_launch(z(0, 8, 10, 10), z(16, 8, 3, 3), z(0, 16, 8, 8),
                                                 64, 64, 32),
        "sdpa_b0": lambda: backend.sdpa_launch(z(0, 2, 64, 64), z(0, 2, 64, 64), z(0, 2, 64, 64),
                                               z(0, 2, 64, 64), 128, 128),
        "rope_s0": lambda: backend.rope_launch(z(2, 0, 4, 64), z(0, 32), z(0, 32), z(2, 0, 4, 64),
                                               32),
    }
    with pytest.raises(backend.LaunchError, match="grid dimension evaluated to 0"):
        calls[case]()


@pytest.mark.parametrize("kernel", ["mm", "addmm", "bmm"])
def test_zero_length_contraction_stores_the_epilogue(kernel):
    """K = 0: the reference's K loop runs zero times, so mm stores zeros and
    addmm stores beta * input (sim.py:269-363)."""
    f16 = torch.float16
    meta = (64, 64, 32)
    if kernel == "bmm":
        out = torch.full((2, 48, 40), 7.0, device=DEV, dtype=f16)
        backend.bmm_launch(torch.zeros((2, 48, 0), device=DEV, dtype=f16),
                           torch.zeros((2, 0, 40), device=DEV, dtype=f16), out, *meta)
        ref = torch.zeros_like(out)
    elif kernel == "mm":
        out = torch.full((48, 40), 7.0, device=DEV, dtype=f16)
        backend.mm_launch(torch.zeros((48, 0), device=DEV, dtype=f16),
                          torch.zeros((0, 40), device=DEV, dtype=f16), out, *meta)
        ref = torch.zeros_like(out)
    else:
        inp = torch.randn((48, 40), device=DEV).to(f16)
        out = torch.full((48, 40), 7.0, device=DEV, dtype=f16)
        backend.addmm_launch(inp, torch.zeros((48, 0), device=DEV, dtype=f16),
                             torch.zeros((0, 40), device=DEV, dtype=f16), 0.5, -2.0, out, *meta)
        ref = (inp.float() * 0.5).to(f16)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_add_beyond_int32_elements():
    """2^31 + 4104 elements (past the reference's int32 Triton offsets,
    SURVEY 8(a) A7): the kernels index in int64; checked at the far end."""
    n = (1 << 31) + 4104
    a = torch.ones(n, device=DEV, dtype=torch.float16)
    b = torch.empty(n, device=DEV, dtype=torch.float16)
    b[-8192:] = torch.arange(8192, device=DEV, dtype=torch.float16) * 0.25
    b[:-8192] = 0.5
    out = torch.empty_like(a)
    backend.add_launch(a, b, out, 1024)
    torch.cuda.synchronize()
    assert torch.equal(out[-8192:], (a[-8192:].float() + b[-8192:].float()).half())
    assert float(out[: 1 << 20].float().mean()) == 1.5
    del a, b, out
    torch.cuda.empty_cache()


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("sq,sk", [(300, 700), (1000, 64), (129, 1), (256, 2000)])
def test_sdpa_cross_attention_lengths(sq, sk, d):
    """S_q != S_k (cross attention): partial query tiles, partial and single-key
    KV tiles, more KV tiles than query tiles and the reverse; D = 64 runs the
    separate-P-buffer schedule (S_{j+1} issued before P.V_j)."""
    rng = np.random.default_rng(sq * 7 + sk + d)
    b, h = 2, 5
    q = _r16(rng.uniform(-1, 1, (b, h, sq, d)).astype(np.float32), torch.float16)
    k = _r16(rng.uniform(-1, 1, (b, h, sk, d)).astype(np.float32), torch.float16)
    v = _r16(rng.uniform(-1, 1, (b, h, sk, d)).astype(np.float32), torch.float16)
    with _Paths() as pc:
        got = _run("sdpa", {"q": q, "k": k, "v": v, "o": None},
                   {"BLOCK_SIZE_M": 128, "BLOCK_SIZE_N": 128}, torch.float16,
                   out=torch.zeros((b, h, sq, d), device=DEV, dtype=torch.float16))
    assert pc.delta["attn_tc"] == 1
    _close(got, oracle.sdpa(q, k, v), rtol=1e-2, atol=1e-2)


def test_launch_accepts_the_simulator_knobs():
    """launch(..., pid_order="reverse", collect_writes=True) like sim.launch:
    same output for either order, writes reported per program."""
    rng = np.random.default_rng(9)
    a = _t(rng.uniform(-1, 1, 3000).astype(np.float32))
    b = _t(rng.uniform(-1, 1, 3000).astype(np.float32))
    outs = []
    for order in ("forward", "reverse"):
        out = torch.zeros(3000, device=DEV)
        res = backend.launch(C.checked("add"), {"input": a, "other": b, "output": out},
                             {"BLOCK_SIZE": 1024}, pid_order=order, collect_writes=True)
        torch.cuda.synchronize()
        outs.append(out.cpu())
        assert res.total == 3 and [len(w) for w in res.writes["output"]] == [1024, 1024, 952]
    assert torch.equal(outs[0], outs[1])
    with pytest.raises(backend.LaunchError, match="unknown pid order"):
        backend.launch(C.checked("add"), {"input": a, "other": b, "output": out},
                       {"BLOCK_SIZE": 1024}, pid_order="random")


@pytest.mark.parametrize("kernel", ["add", "softmax", "mm", "conv2d"])
def test_verify_simulate_twin(kernel):
    """backend.simulate(kernel, args, meta) == the reference's
    verify.simulate outputs committed in tests/golden (same inputs)."""
    index, arrays = sim_cases()
    done = 0
    for ci, case in enumerate(index):
        if case["kernel"] != kernel or done >= 3:
            continue
        args = case_args(ci, case, arrays)
        outs = [p.name for p in C.checked(kernel).spec.params if p.role == "out"]
        args[outs[0]] = np.zeros(out_shape(kernel, args), dtype=np.float32)
        got = backend.simulate(kernel, args, case["meta"], pid_order="reverse")
        sim = arrays[f"c{ci}_sim"]
        tol = 0.0 if kernel == "add" else 1e-4
        assert float(np.max(np.abs(got.astype(np.float64) - sim), initial=0.0)) <= tol
        done += 1
    assert done == 3


def test_pdl_dependent_chains():
    """Kernels launched with programmatic dependent launch prefetch their
    first inputs into L2 BEFORE griddepcontrol.wait.  Chains in which every
    kernel reads the previous kernel's output, queued back to back on one
    stream (and captured in a CUDA graph), must give bit-identical results
    to the same chain with a device synchronisation after every launch
    (L2 is the coherence point; nothing reaches registers or shared memory
    before the wait).  Outputs are pre-filled with NaN so stale reads show."""
    torch.manual_seed(0)
    f16 = torch.float16
    a = torch.rand(1 << 20, device=DEV)
    bufs = [a] + [torch.empty_like(a) for _ in range(6)]
    x = (torch.rand((4096, 4096), device=DEV) * 2 - 1).to(f16)
    w = (torch.rand(4096, device=DEV) + 0.5).to(f16)
    rows = [x] + [torch.empty_like(x) for _ in range(4)]
    m0 = (torch.rand((512, 512), device=DEV) * 2 - 1).to(f16)
    e = (torch.eye(512, device=DEV) * 0.5).to(f16)
    mats = [m0] + [torch.empty_like(m0) for _ in range(3)]
    # attention: each output is the next launch's query (the persistent
    # attention kernel is PDL-launched too)
    qa = [(torch.rand((1, 2, 640, 128), device=DEV) * 2 - 1).to(f16)]
    qa += [torch.empty_like(qa[0]) for _ in range(3)]
    ka, va = ((torch.rand((1, 2, 640, 128), device=DEV) * 2 - 1).to(f16) for _ in range(2))
    outs = bufs[1:] + rows[1:] + mats[1:] + qa[1:]

    def run(sync):
        def s():
            if sync:
                torch.cuda.synchronize()
        for i in range(6):
            backend.add_launch(bufs[i], bufs[i], bufs[i + 1], 1024)
            s()
        for i in range(4):
            if i % 2 == 0:
                backend.softmax_launch(rows[i], rows[i + 1], 4096)
            else:
                backend.rms_norm_launch(rows[i], w, rows[i + 1], 4096)
            s()
        for i in range(3):
            backend.mm_launch(mats[i], e, mats[i + 1], 128, 128, 64)
            s()
        for i in range(3):
            backend.sdpa_launch(qa[i], ka, va, qa[i + 1], 128, 128)
            s()

    def nan_fill():
        for t in outs:
            t.fill_(float("nan"))

    nan_fill()
    run(sync=True)
    torch.cuda.synchronize()
    expect = [t.clone() for t in outs]
    assert torch.equal(bufs[6], a * 64)
    r = m0
    for _ in range(3):   # one fp16 rounding per step (subnormals round each time)
        r = (r.float() * 0.5).to(f16)
    assert torch.equal(mats[3], r)
    assert bool(torch.isfinite(rows[4]).all())
    for mode in ("stream", "graph"):
        nan_fill()
        if mode == "stream":
            run(sync=False)
        else:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                run(sync=False)
            nan_fill()
            g.replay()
        torch.cuda.synchronize()
        for i, (got, ref) in enumerate(zip(outs, expect)):
            assert torch.equal(got, ref), (mode, i)


def test_workspace_is_per_stream():
    """Library scratch (conv's repacked filter + image, sdpa_rope's rotated
    K) is per stream: the same ops queued concurrently on two streams give
    the results of running them one at a time; and they can be captured in
    a CUDA graph after a warm-up."""
    f16 = torch.float16
    g = torch.Generator(device=DEV).manual_seed(7)

    def U(*shape):
        return (torch.rand(shape, generator=g, device=DEV) * 2 - 1).to(f16)

    def rope_case():
        b, s, h, d = 2, 512, 4, 128
        q, k, v = U(b, s, h, d), U(b, s, h, d), U(b, s, h, d)
        ang = torch.rand((s, d // 2), generator=g, device=DEV) * 6 - 3
        sn, cs = torch.sin(ang).to(f16), torch.cos(ang).to(f16)
        o = torch.empty((b, h, s, d), device=DEV, dtype=f16)
        return (q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2), sn, cs, sn, cs, o)

    def conv_case():
        x, w = U(2, 64, 20, 20), U(128, 64, 3, 3)
        return (x, w, torch.empty((2, 128, 18, 18), device=DEV, dtype=f16))

    cases = [(rope_case(), lambda a: backend.sdpa_rope_launch(*a, 128, 128)),
             (rope_case(), lambda a: backend.sdpa_rope_launch(*a, 128, 128)),
             (conv_case(), lambda a: backend.conv2d_launch(*a, 128, 128, 64)),
             (conv_case(), lambda a: backend.conv2d_launch(*a, 128, 128, 64))]
    expect = []
    for args, fn in cases:                       # one at a time
        fn(args)
        torch.cuda.synchronize()
        expect.append(args[-1].clone())
    streams = [torch.cuda.Stream() for _ in range(2)]
    for _ in range(3):
        for args, _fn in cases:
            args[-1].fill_(float("nan"))
        torch.cuda.synchronize()
        for i, (args, fn) in enumerate(cases):   # interleaved on two streams
            with torch.cuda.stream(streams[i % 2]):
                fn(args)
        torch.cuda.synchronize()
        for (args, _fn), ref in zip(cases, expect):
            assert torch.equal(args[-1], ref)
    # CUDA-graph capture on a fresh stream (no buffer yet: the capture
    # allocates its own, pinned), then an eager call on the SAME stream that
    # grows the workspace: the graph's buffer must stay alive (retired, not
    # freed) and the replay must still be exact (ntb_abi.cu).
    cap = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=cap):
        for args, fn in cases:
            fn(args)
    xb, wb = U(2, 256, 20, 20), U(256, 256, 3, 3)
    yb = torch.empty((2, 256, 18, 18), device=DEV, dtype=f16)
    with torch.cuda.stream(cap):
        backend.conv2d_launch(xb, wb, yb, 128, 128, 64)
    torch.cuda.synchronize()
    for _ in range(2):
        for args, _fn in cases:
            args[-1].fill_(float("nan"))
        graph.replay()
        torch.cuda.synchronize()
        for (args, _fn), ref in zip(cases, expect):
            assert torch.equal(args[-1], ref)
    ref = torch.nn.functional.conv2d(xb.float(), wb.float())
    assert (yb.float() - ref).abs().max().item() < 0.5
