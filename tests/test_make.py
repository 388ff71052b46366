"""The paper's front door: make(arrangement, application, tensors) written
exactly as in the paper compiles to specs the
B200 backend recognises structurally."""

import pytest

from paper_2507_11978_b200 import backend
from paper_2507_11978_b200.make import Symbol, Tensor, language as ntl, make
from paper_2507_11978_b200.spec import SpecError

BLOCK_SIZE = Symbol("BLOCK_SIZE", constexpr=True)
BLOCK_SIZE_M = Symbol("BLOCK_SIZE_M", constexpr=True)
BLOCK_SIZE_N = Symbol("BLOCK_SIZE_N", constexpr=True)
BLOCK_SIZE_K = Symbol("BLOCK_SIZE_K", constexpr=True)


def add_kernel():
    def arrangement(input, other, output, BLOCK_SIZE=BLOCK_SIZE):
        return input.tile((BLOCK_SIZE,)), other.tile((BLOCK_SIZE,)), output.tile((BLOCK_SIZE,))

    def application(input, other, output):
        output = input + other  # noqa: F841

    return make(arrangement, application, (Tensor(1), Tensor(1), Tensor(1)))


def mm_kernel():
    def arrangement(input, other, output, BLOCK_SIZE_M=BLOCK_SIZE_M,
                    BLOCK_SIZE_N=BLOCK_SIZE_N, BLOCK_SIZE_K=BLOCK_SIZE_K):
        output_tiled = output.tile((BLOCK_SIZE_M, BLOCK_SIZE_N))
        input_tiled = (input.tile((BLOCK_SIZE_M, BLOCK_SIZE_K)).tile((1, -1))
                       .expand((-1, output_tiled.shape[1])))
        input_tiled.dtype = input_tiled.dtype.squeeze(0)
        other_tiled = (other.tile((BLOCK_SIZE_K, BLOCK_SIZE_N)).tile((-1, 1))
                       .expand((output_tiled.shape[0], -1)))
        other_tiled.dtype = other_tiled.dtype.squeeze(1)
        return input_tiled, other_tiled, output_tiled

    def application(input, other, output):
        accumulator = ntl.zeros(output.shape, dtype=ntl.float32)
        for k in range(input.shape[0]):
            accumulator += ntl.dot(input[k], other[k])
        output = accumulator  # noqa: F841

    return make(arrangement, application, (Tensor(2), Tensor(2), Tensor(2)))


def softmax_kernel():
    def arrangement(input, output, BLOCK_SIZE=BLOCK_SIZE):
        return input.tile((1, BLOCK_SIZE)), output.tile((1, BLOCK_SIZE))

    def application(input, output):
        input_loaded = input
        row_minus_max = input_loaded - ntl.max(input_loaded)
        numerator = ntl.exp(row_minus_max)
        denominator = ntl.sum(numerator)
        output = numerator / denominator  # noqa: F841

    return make(arrangement, application, (Tensor(2, other=float("-inf")), Tensor(2)))


@pytest.mark.parametrize("build,family", [(add_kernel, "add"), (mm_kernel, "mm"),
                                          (softmax_kernel, "softmax")])
def test_paper_kernels_map_to_native_families(build, family):
    k = build()
    assert backend._family_of(k.checked) == family


def test_renamed_parameters_still_match():
    def arrangement(x, y, z, B=Symbol("B", constexpr=True)):
        return x.tile((B,)), y.tile((B,)), z.tile((B,))

    def application(x, y, z):
        z = x + y  # noqa: F841

    k = make(arrangement, application, (Tensor(1), Tensor(1), Tensor(1)), name="my_add")
    assert backend._family_of(k.checked) == "add"


def test_non_native_application_is_rejected():
    def arrangement(input, other, output, BLOCK_SIZE=BLOCK_SIZE):
        return input.tile((BLOCK_SIZE,)), other.tile((BLOCK_SIZE,)), output.tile((BLOCK_SIZE,))

    def application(input, other, output):
        output = input * other  # noqa: F841

    k = make(arrangement, application, (Tensor(1), Tensor(1), Tensor(1)))
    with pytest.raises(backend.UnsupportedSpecError):
        backend._family_of(k.checked)


def test_unsupported_python_is_a_spec_error():
    def arrangement(input, output, BLOCK_SIZE=BLOCK_SIZE):
        return input.tile((BLOCK_SIZE,)), output.tile((BLOCK_SIZE,))

    def application(input, output):
        while True:
            pass

    with pytest.raises(SpecError):
        make(arrangement, application, (Tensor(1), Tensor(1)))


@pytest.mark.gpu
def test_make_kernels_run_on_b200():
    import numpy as np
    import torch

    import oracle

    rng = np.random.default_rng(0)
    a = rng.uniform(-1, 1, 5000).astype(np.float32)
    b = rng.uniform(-1, 1, 5000).astype(np.float32)
    out = torch.empty(5000, device="cuda")
    add_kernel()(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), out, BLOCK_SIZE=1024)
    assert out.cpu().numpy().tobytes() == oracle.add(a, b).tobytes()
    A = torch.randn(256, 192, device="cuda", dtype=torch.float16)
    B = torch.randn(192, 320, device="cuda", dtype=torch.float16)
    C = torch.empty(256, 320, device="cuda", dtype=torch.float16)
    mm_kernel()(A, B, C, BLOCK_SIZE_M=64, BLOCK_SIZE_N=64, BLOCK_SIZE_K=32)
    torch.testing.assert_close(C.float(), A.float() @ B.float(), rtol=1e-2, atol=5e-2)
    X = torch.randn(64, 1000, device="cuda", dtype=torch.float16)
    Y = torch.empty_like(X)
    softmax_kernel()(X, Y, BLOCK_SIZE=1024)
    torch.testing.assert_close(Y.float(), torch.softmax(X.float(), 1), rtol=1e-2, atol=1e-4)


def test_snapshot_of_a_running_value_is_not_the_live_value():
    """A Let that snapshots a mutable local before the loop (m0 = m) and is
    read inside the loop must NOT be inlined into the live m: the variant
    computes something else than attention and must not resolve to the
    native sdpa family (backend._inline_lets)."""
    import dataclasses

    from paper_2507_11978_b200 import catalog as C
    from paper_2507_11978_b200.spec import BinOp, ForRange, Let, Local, typecheck

    spec = C.catalog("sdpa")
    assert backend._family_of(typecheck(spec)) == "sdpa"
    app = list(spec.application)
    loop_at = next(i for i, st in enumerate(app) if isinstance(st, ForRange))
    loop = app[loop_at]

    def freeze(node):
        # m_new = max(m0, rowmax(s)) instead of max(m, rowmax(s))
        if isinstance(node, Let) and node.name == "m_new":
            assert isinstance(node.expr, BinOp) and node.expr.a == Local("m")
            return dataclasses.replace(node, expr=dataclasses.replace(node.expr, a=Local("m0")))
        return node

    frozen = dataclasses.replace(loop, body=tuple(freeze(st) for st in loop.body))
    app[loop_at:loop_at + 1] = [Let("m0", Local("m")), frozen]
    variant = dataclasses.replace(spec, application=tuple(app))
    with pytest.raises(backend.UnsupportedSpecError):
        backend._family_of(typecheck(variant))
