"""Pin the CPU oracle (oracle/) against the reference's own outputs."""

import numpy as np
import pytest

import oracle
from helpers import case_args, expr_cases, map_cases, maps, run_oracle, sim_cases

TOL = {"add": 0.0, "silu": 1e-6, "softmax": 1e-6, "rms_norm": 1e-5, "mm": 1e-5,
       "bmm": 1e-5, "addmm": 1e-5, "conv2d": 1e-5}


def test_expr_eval_matches_reference_values():
    for c in expr_cases():
        assert oracle.expr_eval(c["expr"], c["binding"]) == c["value"]


def test_sim_cases_cover_every_catalog_kernel():
    index, _ = sim_cases()
    assert {c["kernel"] for c in index} == set(TOL)
    assert len(index) >= 160


@pytest.mark.parametrize("kernel", sorted(TOL))
def test_oracle_matches_reference_simulator(kernel):
    index, arrays = sim_cases()
    n = 0
    for ci, case in enumerate(index):
        if case["kernel"] != kernel:
            continue
        args = case_args(ci, case, arrays)
        got = run_oracle(kernel, args, case["meta"])
        sim = arrays[f"c{ci}_sim"]
        assert got.shape == sim.shape
        if kernel == "add":
            # fp32 add: bit-exact against sim.launch
            assert got.tobytes() == sim.tobytes()
        else:
            err = np.max(np.abs(got.astype(np.float64) - sim)) if sim.size else 0.0
            assert err <= TOL[kernel] * max(1.0, float(np.max(np.abs(sim))) if sim.size else 1.0), \
                (kernel, case["dims"], err)
        n += 1
    assert n >= 20


def test_oracle_map_points_match_reference():
    index, arrays = map_cases()
    m = maps()
    for ci, case in enumerate(index):
        k = m[case["kernel"]]
        for p in case["params"]:
            mp = k["maps"][p["name"]]
            offs, mask = oracle.map_points(
                k["grid"]["sizes"], k["grid"]["pid_components"], mp["nest_sizes"],
                mp["lane_sizes"], mp["offset"], mp["mask"], case["binding"])
            want_o = arrays[f"c{ci}_{p['name']}_offs"].reshape(-1)
            want_m = arrays[f"c{ci}_{p['name']}_mask"].reshape(-1)
            np.testing.assert_array_equal(offs, want_o)
            np.testing.assert_array_equal(mask, want_m)


def test_conv2d_three_way():
    """direct conv == im2col @ filter (test_acceptance.py:132-149 analogue)."""
    rng = np.random.default_rng(2)
    x = rng.uniform(-1, 1, (1, 2, 5, 5)).astype(np.float32)
    w = rng.uniform(-1, 1, (3, 2, 3, 3)).astype(np.float32)
    direct = np.zeros((1, 3, 3, 3))
    for k in range(3):
        for p in range(3):
            for q in range(3):
                direct[0, k, p, q] = np.sum(x[0, :, p:p + 3, q:q + 3].astype(np.float64) * w[k])
    np.testing.assert_allclose(oracle.conv2d(x, w), direct, atol=1e-6)


def test_builder_sdpa_rope_restatements():
    rng = np.random.default_rng(0)
    q, k, v = (rng.standard_normal((2, 3, 5, 8)) for _ in range(3))
    o = oracle.sdpa(q, k, v)
    # direct per-row loop restatement
    for b in range(2):
        for h in range(3):
            for i in range(5):
                s = q[b, h, i] @ k[b, h].T / np.sqrt(8)
                p = np.exp(s - s.max())
                p /= p.sum()
                np.testing.assert_allclose(o[b, h, i], p @ v[b, h], rtol=1e-5, atol=1e-6)
    x = rng.standard_normal((2, 4, 3, 8))
    ang = rng.standard_normal((4, 4))
    y = oracle.rope(x, np.sin(ang), np.cos(ang))
    # rotation preserves the norm of each (x_i, x_{i+half}) pair
    np.testing.assert_allclose(np.sum(y.astype(np.float64) ** 2, -1), np.sum(x ** 2, -1),
                               rtol=1e-5)


def test_builder_oracles_against_torch():
    """The builder-written sdpa / rope / sdpa_rope oracles against independent
    torch implementations (f64 on the CPU): torch's scaled_dot_product_attention
    and a complex-number rotary embedding (rotation of (x_i + j x_{i+D/2}) by
    the angle whose cos / sin are the tables)."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(1)
    q, k, v = (rng.standard_normal((2, 3, 37, 16)) for _ in range(3))
    ref = torch.nn.functional.scaled_dot_product_attention(
        torch.from_numpy(q), torch.from_numpy(k), torch.from_numpy(v)).numpy()
    np.testing.assert_allclose(oracle.sdpa(q, k, v), ref, rtol=1e-5, atol=1e-6)
    ang = rng.uniform(-3, 3, (37, 8))
    sin, cos = np.sin(ang), np.cos(ang)

    def rope_complex(x_bshd):
        z = torch.complex(torch.from_numpy(x_bshd[..., :8]), torch.from_numpy(x_bshd[..., 8:]))
        z = z * torch.polar(torch.ones(37, 8, dtype=torch.float64),
                            torch.from_numpy(ang))[None, :, None, :]
        return torch.cat([z.real, z.imag], -1).numpy()

    x = rng.standard_normal((2, 37, 3, 16))
    np.testing.assert_allclose(oracle.rope(x, sin, cos), rope_complex(x), rtol=1e-5, atol=1e-6)
    qb, kb = np.swapaxes(rope_complex(np.swapaxes(q, 1, 2)), 1, 2), \
        np.swapaxes(rope_complex(np.swapaxes(k, 1, 2)), 1, 2)
    ref = torch.nn.functional.scaled_dot_product_attention(
        torch.from_numpy(qb), torch.from_numpy(kb), torch.from_numpy(v)).numpy()
    np.testing.assert_allclose(oracle.sdpa_rope(q, k, v, sin, cos, sin, cos), ref,
                               rtol=1e-5, atol=1e-6)
