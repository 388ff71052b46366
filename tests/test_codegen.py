"""Generic path: specs that match no native kernel
family are printed as CUDA C++ (codegen.py) and NVRTC-compiled for sm_100a by
the C ABI (ntb_jit_compile).  CPU tests: the generated source compiles for
sm_100a with NVRTC; GPU tests: results against numpy."""

import numpy as np
import pytest

from paper_2507_11978_b200 import backend, codegen
from paper_2507_11978_b200.make import Symbol, Tensor, language as ntl, make

BLOCK = Symbol("BLOCK", constexpr=True)


def fma_kernel():
    def arrangement(x, y, z, out, BLOCK=BLOCK):
        return x.tile((BLOCK,)), y.tile((BLOCK,)), z.tile((BLOCK,)), out.tile((BLOCK,))

    def application(x, y, z, out):
        out = x * y + z  # noqa: F841

    return make(arrangement, application, (Tensor(1), Tensor(1), Tensor(1), Tensor(1)))


def gelu_kernel():
    def arrangement(x, out, BLOCK=BLOCK):
        return x.tile((BLOCK,)), out.tile((BLOCK,))

    def application(x, out):
        out = x * ntl.sigmoid(1.702 * x)  # noqa: F841

    return make(arrangement, application, (Tensor(1), Tensor(1)))


def temp_softmax_kernel():
    def arrangement(x, out, BLOCK=BLOCK):
        return x.tile((1, BLOCK)), out.tile((1, BLOCK))

    def application(x, out):
        z = x * 0.5
        e = ntl.exp(z - ntl.max(z))
        out = e / ntl.sum(e)  # noqa: F841

    return make(arrangement, application, (Tensor(2, other=float("-inf")), Tensor(2)))


def l2norm_kernel():
    def arrangement(x, out, BLOCK=BLOCK):
        return x.tile((1, BLOCK)), out.tile((1, BLOCK))

    def application(x, out):
        out = x / ntl.sqrt(ntl.sum(x * x) + 1e-6)  # noqa: F841

    return make(arrangement, application, (Tensor(2), Tensor(2)))


BM = Symbol("BM", constexpr=True)
BN = Symbol("BN", constexpr=True)
BK = Symbol("BK", constexpr=True)


def mm_relu_kernel():
    """The paper's matmul arrangement with a fused ReLU epilogue: a
    contraction no native family implements."""
    def arrangement(input, other, output, BM=BM, BN=BN, BK=BK):
        output_tiled = output.tile((BM, BN))
        input_tiled = input.tile((BM, BK)).tile((1, -1)).expand((-1, output_tiled.shape[1]))
        input_tiled.dtype = input_tiled.dtype.squeeze(0)
        other_tiled = other.tile((BK, BN)).tile((-1, 1)).expand((output_tiled.shape[0], -1))
        other_tiled.dtype = other_tiled.dtype.squeeze(1)
        return input_tiled, other_tiled, output_tiled

    def application(input, other, output):
        accumulator = ntl.zeros(output.shape, dtype=ntl.float32)
        for k in range(input.shape[0]):
            accumulator += ntl.dot(input[k], other[k])
        output = ntl.maximum(accumulator, 0.0)  # noqa: F841

    return make(arrangement, application, (Tensor(2), Tensor(2), Tensor(2)))


def rowsum_kernel():
    """Row sums of a (BM, BN) tile stored as a (BM,) tile: a reduction along
    one axis of a tile larger than the stored one."""
    def arrangement(x, out, BM=BM, BN=BN):
        return x.tile((BM, BN)).squeeze(1), out.tile((BM,))

    def application(x, out):
        out = ntl.sum(x, axis=1)  # noqa: F841

    return make(arrangement, application, (Tensor(2), Tensor(1)))


def colnorm_kernel():
    """x - max(x, axis=0): column maxima broadcast back over the rows."""
    def arrangement(x, out, BM=BM, BN=BN):
        return x.tile((BM, BN)), out.tile((BM, BN))

    def application(x, out):
        out = ntl.exp(x - ntl.max(x, axis=0))  # noqa: F841

    return make(arrangement, application, (Tensor(2, other=float("-inf")), Tensor(2)))


def rowcenter_kernel():
    """a - sum(a, axis=1) on a square tile: the (B,) row sums broadcast
    right-aligned, i.e. along the LAST axis (the reference's numpy rules,
    tileir.py:290-306) - out[i][j] = a[i][j] - sum_k a[j][k]."""
    B = Symbol("B", constexpr=True)

    def arrangement(a, c, B=B):
        return a.tile((B, B)), c.tile((B, B))

    def application(a, c):
        c = a - ntl.sum(a, axis=1)  # noqa: F841

    return make(arrangement, application, (Tensor(2), Tensor(2)))


def mm_scaled_kernel():
    """A local declared inside the K loop (fresh binding per iteration)."""
    def arrangement(input, other, output, BM=BM, BN=BN, BK=BK):
        output_tiled = output.tile((BM, BN))
        input_tiled = input.tile((BM, BK)).tile((1, -1)).expand((-1, output_tiled.shape[1]))
        input_tiled.dtype = input_tiled.dtype.squeeze(0)
        other_tiled = other.tile((BK, BN)).tile((-1, 1)).expand((output_tiled.shape[0], -1))
        other_tiled.dtype = other_tiled.dtype.squeeze(1)
        return input_tiled, other_tiled, output_tiled

    def application(input, other, output):
        accumulator = ntl.zeros(output.shape, dtype=ntl.float32)
        for k in range(input.shape[0]):
            part = ntl.dot(input[k], other[k])
            accumulator += part * 0.5
        output = accumulator  # noqa: F841

    return make(arrangement, application, (Tensor(2), Tensor(2), Tensor(2)))


def _binding(k, shapes, meta):
    b = dict(meta)
    for p, shp in zip(k.checked.spec.params, shapes):
        st, acc = [], 1
        for s in reversed(shp):
            st.append(acc)
            acc *= s
        for i, (s, t) in enumerate(zip(shp, reversed(st))):
            b[f"{p.name}_size_{i}"] = s
            b[f"{p.name}_stride_{i}"] = t
    return b


CASES = [
    (fma_kernel, [(5000,)] * 4, {"BLOCK": 1024}),
    (gelu_kernel, [(777,)] * 2, {"BLOCK": 256}),
    (temp_softmax_kernel, [(33, 1000)] * 2, {"BLOCK": 1024}),
    (l2norm_kernel, [(7, 4096)] * 2, {"BLOCK": 4096}),
    (mm_relu_kernel, [(200, 96), (96, 130), (200, 130)], {"BM": 32, "BN": 32, "BK": 32}),
    (mm_scaled_kernel, [(200, 96), (96, 130), (200, 130)], {"BM": 32, "BN": 32, "BK": 32}),
    (rowsum_kernel, [(100, 300), (100,)], {"BM": 16, "BN": 512}),
    (colnorm_kernel, [(100, 300)] * 2, {"BM": 64, "BN": 32}),
    (rowcenter_kernel, [(40, 40)] * 2, {"B": 16}),
]


@pytest.mark.parametrize("build,shapes,meta", CASES)
def test_generated_source_compiles_for_sm100a(build, shapes, meta):
    nvrtc = pytest.importorskip("cuda.bindings.nvrtc")
    k = build()
    with pytest.raises(backend.UnsupportedSpecError):
        backend._family_of(k.checked)          # not a native family
    for dt in (0, 1, 2):
        g = codegen.generate(k.checked, _binding(k, shapes, meta), dt)
        err, prog = nvrtc.nvrtcCreateProgram(g.source.encode(), b"gen.cu", 0, [], [])
        assert err == nvrtc.nvrtcResult.NVRTC_SUCCESS
        opts = [b"--gpu-architecture=sm_100a", b"-std=c++17", b"-default-device",
                b"--include-path=/usr/local/cuda/include"]
        err, = nvrtc.nvrtcCompileProgram(prog, len(opts), opts)
        if err != nvrtc.nvrtcResult.NVRTC_SUCCESS:
            _, n = nvrtc.nvrtcGetProgramLogSize(prog)
            log = b" " * n
            nvrtc.nvrtcGetProgramLog(prog, log)
            pytest.fail(log.decode())


def test_generated_maps_follow_the_lowered_index_maps():
    g = codegen.generate(fma_kernel().checked, _binding(fma_kernel(), [(5000,)] * 4,
                                                         {"BLOCK": 1024}), 0)
    # offset = (pid_0 * BLOCK + lane_0) * stride, mask against the size slot
    assert "((pid_0 * ((i64)1024LL)) + Larr0[e]) * S.v[1]" in g.source
    assert g.block == 256 and "constexpr int E = 4;" in g.source


def _run(k, arrays, meta, dtype):
    import torch

    ts = [torch.from_numpy(a).cuda().to(dtype) for a in arrays]
    out = torch.empty_like(ts[0])
    before = backend.path_counts()["jit"]
    k(*ts, out, **meta)
    torch.cuda.synchronize()
    assert backend.path_counts()["jit"] == before + 1
    return [t.float().cpu().numpy() for t in ts], out.float().cpu().numpy()


@pytest.mark.gpu
def test_generic_elementwise_on_b200():
    import torch

    rng = np.random.default_rng(1)
    xs = [rng.uniform(-1, 1, 5000).astype(np.float32) for _ in range(3)]
    ins, out = _run(fma_kernel(), xs, {"BLOCK": 1024}, torch.float32)
    # fp32 x*y+z on both sides; the device may contract to one fma
    np.testing.assert_allclose(out, ins[0] * ins[1] + ins[2], rtol=1e-6, atol=1e-7)
    for dt in (torch.float16, torch.bfloat16):
        x = rng.uniform(-3, 3, 777).astype(np.float32)
        (xin,), out = _run(gelu_kernel(), [x], {"BLOCK": 256}, dt)
        ref = xin / (1 + np.exp(-1.702 * xin))
        np.testing.assert_allclose(out, ref, rtol=1e-2, atol=1e-2)


@pytest.mark.gpu
def test_generic_row_reductions_on_b200():
    import torch

    rng = np.random.default_rng(2)
    x = rng.uniform(-4, 4, (33, 1000)).astype(np.float32)
    (xin,), out = _run(temp_softmax_kernel(), [x], {"BLOCK": 1024}, torch.float32)
    z = xin * 0.5
    ref = np.exp(z - z.max(1, keepdims=True))
    ref /= ref.sum(1, keepdims=True)
    np.testing.assert_allclose(out, ref, rtol=1e-5, atol=1e-6)
    x = rng.uniform(-1, 1, (7, 4096)).astype(np.float32)
    (xin,), out = _run(l2norm_kernel(), [x], {"BLOCK": 4096}, torch.float16)
    ref = xin / np.sqrt((xin.astype(np.float64) ** 2).sum(1, keepdims=True) + 1e-6)
    np.testing.assert_allclose(out, ref, rtol=1e-2, atol=1e-3)


@pytest.mark.gpu
def test_generic_contraction_on_b200():
    import torch

    rng = np.random.default_rng(3)
    a = rng.uniform(-1, 1, (200, 96)).astype(np.float32)
    b = rng.uniform(-1, 1, (96, 130)).astype(np.float32)
    for dt in (torch.float32, torch.float16):
        ta, tb = torch.from_numpy(a).cuda().to(dt), torch.from_numpy(b).cuda().to(dt)
        out = torch.empty((200, 130), device="cuda", dtype=dt)
        before = backend.path_counts()["jit"]
        mm_relu_kernel()(ta, tb, out, BM=32, BN=32, BK=32)
        torch.cuda.synchronize()
        assert backend.path_counts()["jit"] == before + 1
        ref = np.maximum(ta.float().cpu().numpy() @ tb.float().cpu().numpy(), 0)
        tol = 1e-4 if dt == torch.float32 else 1e-2
        np.testing.assert_allclose(out.float().cpu().numpy(), ref, rtol=tol, atol=tol)


@pytest.mark.gpu
def test_generic_axis_reductions_on_b200():
    """Reductions along one axis of a loaded tile (results in shared memory,
    broadcast with the reference's rules) against numpy on the same
    fp16-rounded inputs."""
    import torch

    rng = np.random.default_rng(4)
    x = rng.uniform(-1, 1, (100, 300)).astype(np.float32)
    for dt, tol in ((torch.float32, 1e-5), (torch.float16, 1e-2)):
        tx = torch.from_numpy(x).cuda().to(dt)
        out = torch.empty(100, device="cuda", dtype=dt)
        before = backend.path_counts()["jit"]
        rowsum_kernel()(tx, out, BM=16, BN=512)
        torch.cuda.synchronize()
        assert backend.path_counts()["jit"] == before + 1
        ref = tx.float().cpu().numpy().sum(1)
        np.testing.assert_allclose(out.float().cpu().numpy(), ref, rtol=tol, atol=tol)
        (xin,), got = _run(colnorm_kernel(), [x], {"BM": 64, "BN": 32}, dt)
        # per program: the column maximum over that program's 64 rows
        ref = np.empty_like(xin)
        for r0 in range(0, 100, 64):
            blk = xin[r0:r0 + 64]
            ref[r0:r0 + 64] = np.exp(blk - blk.max(0, keepdims=True))
        np.testing.assert_allclose(got, ref, rtol=tol, atol=tol)
    a = rng.uniform(-1, 1, (40, 40)).astype(np.float32)
    (ain,), got = _run(rowcenter_kernel(), [a], {"B": 16}, torch.float32)
    ref = np.empty_like(ain)
    for i0 in range(0, 40, 16):
        for j0 in range(0, 40, 16):
            t = np.zeros((16, 16), np.float32)
            blk = ain[i0:i0 + 16, j0:j0 + 16]
            t[:blk.shape[0], :blk.shape[1]] = blk          # masked loads read 0
            r = t - t.sum(1)                                # (16,) broadcast over rows
            ref[i0:i0 + 16, j0:j0 + 16] = r[:blk.shape[0], :blk.shape[1]]
    np.testing.assert_allclose(got, ref, rtol=1e-5, atol=1e-5)


@pytest.mark.gpu
def test_generic_loop_local_on_b200():
    import torch

    rng = np.random.default_rng(5)
    a = rng.uniform(-1, 1, (200, 96)).astype(np.float32)
    b = rng.uniform(-1, 1, (96, 130)).astype(np.float32)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    out = torch.empty((200, 130), device="cuda")
    mm_scaled_kernel()(ta, tb, out, BM=32, BN=32, BK=32)
    torch.cuda.synchronize()
    np.testing.assert_allclose(out.cpu().numpy(), 0.5 * (a @ b), rtol=1e-4, atol=1e-4)


@pytest.mark.gpu
def test_generic_path_matches_reference_sim():
    """Pinned: specs written in the reference's own IR and run through the
    reference's sim.launch (fixtures from tests/golden/gen_generic.py) against
    this package's make() kernels on the generic path, fp32, within the
    reference's 1e-4 reduction tolerance (verify.py:25): element-wise (fma,
    GELU approximation), whole-tile reductions (temperature softmax, l2-norm)
    and axis reductions (row sums stored as a vector, exp(x - max(x, 0)),
    a - sum(a, 1) broadcast along the last axis)."""
    import torch
    from pathlib import Path

    g = np.load(Path(__file__).resolve().parent / "golden" / "generic_cases.npz")
    cases = [("fma", fma_kernel, ("x", "y", "z"), "out", {"BLOCK": 1024}),
             ("gelu", gelu_kernel, ("x",), "out", {"BLOCK": 256}),
             ("temp_softmax", temp_softmax_kernel, ("x",), "out", {"BLOCK": 1024}),
             ("l2norm", l2norm_kernel, ("x",), "out", {"BLOCK": 4096}),
             ("rowsum", rowsum_kernel, ("x",), "out", {"BM": 16, "BN": 512}),
             ("colexp", colnorm_kernel, ("x",), "out", {"BM": 64, "BN": 32}),
             ("rowcenter", rowcenter_kernel, ("a",), "c", {"B": 16})]
    for name, build, pins, pout, meta in cases:
        xs = [torch.from_numpy(g[f"{name}.in.{k}"]).cuda() for k in pins]
        ref = g[f"{name}.out.{pout}"]
        out = torch.zeros(ref.shape, device="cuda")
        before = backend.path_counts()["jit"]
        build()(*xs, out, **meta)
        torch.cuda.synchronize()
        assert backend.path_counts()["jit"] == before + 1, name
        np.testing.assert_allclose(out.cpu().numpy(), ref, rtol=1e-4, atol=1e-5, err_msg=name)
