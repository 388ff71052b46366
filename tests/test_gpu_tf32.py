"""GPU parity of the fp32 contractions (mm / addmm / bmm / conv2d) on the
tensor cores (3xTF32, csrc/k_gemm_tf32_sm100.cu) against the CPU oracle (f64
dot rounded to f32, the reference's own Dot semantics, sim.py:317-320).

Tolerance (written here): |got - ref| <= 1e-4 * sqrt(K / 64) + 1e-5 * |ref|
- the reference's fp32 contraction tolerance (1e-4 max-abs, verify.py:24-25)
at its own K sizes, grown with sqrt(K) for the fp32 accumulation of longer
sums.  One-pass TF32 (10-bit mantissa) misses it by ~30x at K = 700, so the
test also shows that the lo terms are applied.
"""

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2507_11978_b200 import backend  # noqa: E402
from paper_2507_11978_b200 import catalog as C  # noqa: E402

DEV = "cuda:0"
META = {"BLOCK_SIZE_M": 128, "BLOCK_SIZE_N": 128, "BLOCK_SIZE_K": 64}


def _run(kernel, args, out_shape):
    ck = C.checked(kernel)
    targs = {}
    for p in ck.spec.params:
        v = args.get(p.name)
        if p.rank == 0:
            targs[p.name] = float(v)
        elif p.role == "out":
            targs[p.name] = torch.zeros(out_shape, device=DEV, dtype=torch.float32)
        else:
            targs[p.name] = v if isinstance(v, torch.Tensor) else torch.from_numpy(
                np.ascontiguousarray(v)).to(DEV)
    before = backend.path_counts()
    backend.launch(ck, targs, META)
    torch.cuda.synchronize()
    after = backend.path_counts()
    out = [targs[p.name] for p in ck.spec.params if p.role == "out"][0]
    return out, {k: after[k] - before[k] for k in after}


def _tol(k):
    return 1e-4 * max(1.0, np.sqrt(k / 64.0)), 1e-5


def _check(got, ref, k):
    atol, rtol = _tol(k)
    got = got.cpu().numpy().astype(np.float64)
    err = np.abs(got - ref)
    bad = err > atol + rtol * np.abs(ref)
    assert not bad.any(), f"{bad.sum()} of {bad.size} outside tol; max err {err.max():.3e}"
    return err.max()


def _u(rng, shape):
    return rng.uniform(-1, 1, shape).astype(np.float32)


@pytest.mark.parametrize("mnk", [(128, 128, 64), (256, 512, 320), (1000, 520, 700),
                                 (300, 36, 4100), (4096, 4096, 4096)])
def test_mm_f32_tensor_cores(mnk):
    m, n, k = mnk
    rng = np.random.default_rng(m * 7 + n + k)
    a, b = _u(rng, (m, k)), _u(rng, (k, n))
    got, d = _run("mm", {"input": a, "other": b}, (m, n))
    assert d["gemm_tf32"] == 1 and d["gemm_generic"] == 0
    rows = np.arange(m) if m <= 1024 else np.sort(rng.choice(m, 192, replace=False))
    ref = oracle.mm(a[rows], b).astype(np.float64)
    err = _check(got[torch.as_tensor(rows, device=DEV)], ref, k)
    if k == 700:
        # one-pass TF32 would be ~2^-11 relative per product: the split matters
        tr = lambda x: (x.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)  # noqa: E731
        one_pass = np.abs(tr(a).astype(np.float64) @ tr(b).astype(np.float64) - ref).max()
        assert err * 10 < one_pass, (err, one_pass)


@pytest.mark.parametrize("a_t,b_t", [(False, False), (True, False), (False, True), (True, True)])
def test_mm_f32_all_operand_majors(a_t, b_t):
    rng = np.random.default_rng(5)
    m, n, k = 384, 320, 264
    a, b = _u(rng, (m, k)), _u(rng, (k, n))
    ta = torch.from_numpy(a.T.copy()).to(DEV).t() if a_t else torch.from_numpy(a).to(DEV)
    tb = torch.from_numpy(b.T.copy()).to(DEV).t() if b_t else torch.from_numpy(b).to(DEV)
    got, d = _run("mm", {"input": ta, "other": tb}, (m, n))
    assert d["gemm_tf32"] == 1
    _check(got, oracle.mm(a, b).astype(np.float64), k)


def test_addmm_f32_tensor_cores():
    rng = np.random.default_rng(11)
    m, n, k = 520, 384, 1000
    inp, a, b = _u(rng, (m, n)), _u(rng, (m, k)), _u(rng, (k, n))
    got, d = _run("addmm", {"input": inp, "mat1": a, "mat2": b, "beta": -0.134, "alpha": -0.201},
                  (m, n))
    assert d["gemm_tf32"] == 1
    _check(got, oracle.addmm(inp, a, b, -0.134, -0.201).astype(np.float64), k)


@pytest.mark.parametrize("bmnk", [(3, 100, 72, 40), (8, 256, 256, 256), (64, 1024, 1024, 1024)])
def test_bmm_f32_tensor_cores(bmnk):
    bt, m, n, k = bmnk
    rng = np.random.default_rng(bt + k)
    a, b = _u(rng, (bt, m, k)), _u(rng, (bt, k, n))
    got, d = _run("bmm", {"input": a, "other": b}, (bt, m, n))
    assert d["gemm_tf32"] == 1
    sel = [0, bt // 2, bt - 1]
    _check(got[sel], oracle.bmm(a[sel], b[sel]).astype(np.float64), k)


def test_f32_repeat_launch_bit_identity():
    """Same inputs, launched twice (and reversed pid order requested): the
    bytes must match (test_acceptance.py:165-172 analogue)."""
    rng = np.random.default_rng(2)
    a, b = _u(rng, (1536, 768)), _u(rng, (768, 1280))
    ck = C.checked("mm")
    ta, tb = torch.from_numpy(a).to(DEV), torch.from_numpy(b).to(DEV)
    outs = []
    for order in ("forward", "reverse"):
        o = torch.empty((1536, 1280), device=DEV)
        backend.launch(ck, {"input": ta, "other": tb, "output": o}, META, pid_order=order)
        outs.append(o)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])


def test_f32_magnitudes():
    """Large / tiny magnitudes: the split is scale-free (exact in fp32)."""
    rng = np.random.default_rng(9)
    for scale in (1e-20, 1e-3, 1e3, 1e15):
        a, b = _u(rng, (256, 256)) * np.float32(scale), _u(rng, (256, 256))
        got, d = _run("mm", {"input": a, "other": b}, (256, 256))
        ref = oracle.mm(a, b).astype(np.float64)
        err = np.abs(got.cpu().numpy() - ref).max()
        assert err <= 2e-6 * np.abs(ref).max(), (scale, err, np.abs(ref).max())


@pytest.mark.parametrize("shape", [(1, 2, 5, 5, 3, 3, 3), (2, 16, 12, 10, 32, 3, 3),
                                   (2, 64, 30, 30, 128, 3, 3), (3, 100, 17, 23, 320, 5, 5),
                                   (9, 64, 40, 40, 64, 1, 1), (4, 256, 56, 56, 256, 3, 3)])
def test_conv2d_f32_tensor_cores(shape):
    n, c, h, w, k, r, s = shape
    rng = np.random.default_rng(n * 31 + c + k)
    x, f = _u(rng, (n, c, h, w)), _u(rng, (k, c, r, s))
    got, d = _run("conv2d", {"input": x, "filter": f}, (n, k, h - r + 1, w - s + 1))
    assert d["conv_tf32"] == 1 and d["conv_generic"] == 0
    sel = [0, n - 1]
    ref = oracle.conv2d(x[sel], f).astype(np.float64)
    _check(got[sel], ref, c * r * s)


def test_conv2d_f32_channels_last():
    rng = np.random.default_rng(4)
    n, c, h, w, k = 2, 64, 20, 18, 96
    x, f = _u(rng, (n, c, h, w)), _u(rng, (k, c, 3, 3))
    xt = torch.from_numpy(x).to(DEV).contiguous(memory_format=torch.channels_last)
    got, d = _run("conv2d", {"input": xt, "filter": f}, (n, k, h - 2, w - 2))
    assert d["conv_tf32"] == 1
    _check(got, oracle.conv2d(x, f).astype(np.float64), c * 9)


@pytest.mark.parametrize("kernel,shape", [("mm", (2560, 4096, 1024)), ("addmm", (2560, 4096, 512)),
                                          ("bmm", (3, 1536, 1280, 512)),
                                          ("conv2d", (7, 64, 56, 56, 256, 3, 3))])
def test_f32_narrow_tail(kernel, shape):
    """Tile counts that leave the last wave of the 74 CTA pairs less than half
    full (160, 90, 84 tiles) run the tail tiles as two 256 x 128 units; every
    output element is checked."""
    rng = np.random.default_rng(sum(shape))
    if kernel == "conv2d":
        n, c, h, w, k, r, s = shape
        x, f = _u(rng, (n, c, h, w)), _u(rng, (k, c, r, s))
        got, d = _run("conv2d", {"input": x, "filter": f}, (n, k, h - r + 1, w - s + 1))
        assert d["conv_tf32"] == 1
        _check(got, oracle.conv2d(x, f).astype(np.float64), c * r * s)
        return
    if kernel == "bmm":
        bt, m, n, k = shape
        a, b = _u(rng, (bt, m, k)), _u(rng, (bt, k, n))
        got, d = _run("bmm", {"input": a, "other": b}, (bt, m, n))
        ref = oracle.bmm(a, b)
    else:
        m, n, k = shape
        a, b = _u(rng, (m, k)), _u(rng, (k, n))
        if kernel == "mm":
            got, d = _run("mm", {"input": a, "other": b}, (m, n))
            ref = oracle.mm(a, b)
        else:
            inp = _u(rng, (m, n))
            got, d = _run("addmm", {"input": inp, "mat1": a, "mat2": b, "beta": 0.5, "alpha": -1.5},
                          (m, n))
            ref = oracle.addmm(inp, a, b, 0.5, -1.5)
    assert d["gemm_tf32"] == 1
    _check(got, ref.astype(np.float64), k)
