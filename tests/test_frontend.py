"""The B200 front end reproduces the reference's arrangement semantics:
symbolic evaluation, simplification, meta-ops, grid inference and the
lowered index maps (tree-for-tree against tests/golden/maps.json)."""

import numpy as np
import pytest

from helpers import expr_cases, maps
from paper_2507_11978_b200 import catalog as C
from paper_2507_11978_b200 import symbolic as S
from paper_2507_11978_b200.arrange import ArrangeError, infer_grid, lower
from paper_2507_11978_b200.spec import ir_tree
from paper_2507_11978_b200.tensor import FULL, TensorError, new_param, param_with_shape


def test_evaluate_matches_reference_on_random_expressions():
    for c in expr_cases():
        e = S.from_tree(c["expr"])
        assert S.evaluate(e, c["binding"]) == c["value"]
        assert S.to_tree(S.simplify(e)) == c["simplified"]
        assert S.evaluate(S.simplify(e), c["binding"]) == c["value"]


def test_floor_semantics_and_zero_divisor():
    a, b = S.var("a"), S.var("b")
    assert S.evaluate(a // b, {"a": -7, "b": 2}) == -4
    assert S.evaluate(a % b, {"a": -7, "b": 2}) == 1
    assert S.evaluate(S.ceil_div(a, b), {"a": 7, "b": 2}) == 4
    assert S.evaluate(S.ceil_div(a, b), {"a": -7, "b": 2}) == -3
    with pytest.raises(S.EvalError):
        S.evaluate(a // b, {"a": 1, "b": 0})
    with pytest.raises(S.EvalError):
        S.evaluate(a, {})
    # array bindings (symexpr.py:157-160)
    v = S.evaluate(a * 2 + 1, {"a": np.arange(4)})
    np.testing.assert_array_equal(v, [1, 3, 5, 7])


def test_render_precedence():
    a, b, c = S.var("a"), S.var("b"), S.var("c")
    assert S.text(a - (b - c)) == "a - (b - c)"
    assert S.text((a - b) - c) == "a - b - c"
    assert S.text(a * (b % c)) == "a * (b % c)"
    assert S.text(-(a + b)) == "-(a + b)"


def test_tile_counts():
    t = param_with_shape("x", (4, 4)).tile((2, 2))
    assert [s.value for s in t.level_shape(0)] == [2, 2]
    assert [s.value for s in t.level_shape(1)] == [2, 2]
    t = param_with_shape("x", (5,)).tile((2,))
    assert t.level_shape(0)[0].value == 3
    t = param_with_shape("x", (5,)).tile((3,), strides=(1,))
    assert t.level_shape(0)[0].value == 3          # sliding window count
    with pytest.raises(TensorError):
        param_with_shape("x", (5,)).tile((3,), strides=(0,))


def test_expand_squeeze_rules():
    t = param_with_shape("x", (4, 4)).tile((1, FULL))
    assert [s.value for s in t.level_shape(0)] == [4, 1]
    assert t.expand((-1, 7)).level_shape(0)[1].value == 7
    with pytest.raises(TensorError):
        t.expand((7, -1))
    with pytest.raises(TensorError):
        t.squeeze(0)
    u = new_param("y", 1).tile((S.var("B"),))
    sq = u.squeeze(0)                       # symbolic -> deferred launch check
    assert len(sq.checks) == 1


def test_grid_validation_errors():
    a = param_with_shape("a", (4,)).tile((2,))
    b = param_with_shape("b", (6,)).tile((2,))
    with pytest.raises(ArrangeError):
        infer_grid([("a", a), ("b", b)])
    with pytest.raises(ArrangeError):
        infer_grid([("a", param_with_shape("a", (4,)))])
    c = new_param("c", 1).tile((S.var("B"),))
    d = new_param("d", 1).tile((S.var("B"),))
    g = infer_grid([("c", c), ("d", d)])
    assert len(g.checks) == 1


@pytest.mark.parametrize("kernel", C.CATALOG_NAMES)
def test_maps_identical_to_reference(kernel):
    ref = maps()[kernel]
    ck = C.checked(kernel)
    assert [S.to_tree(s) for s in ck.grid.sizes] == ref["grid"]["sizes"]
    assert S.to_tree(ck.grid.total) == ref["grid"]["total"]
    assert [[S.to_tree(a), S.to_tree(b)] for a, b in ck.grid.checks] == ref["grid"]["checks"]
    assert [S.to_tree(c) for c in ck.grid.pid_components(S.var("pid"))] == \
        ref["grid"]["pid_components"]
    assert [S.text(c, cdiv="tl.cdiv") for c in ck.grid.pid_components(S.var("pid"))] == \
        ref["grid"]["pid_components_text"]
    for name, m in ck.index_maps.items():
        r = ref["maps"][name]
        assert S.to_tree(m.offset) == r["offset"]
        assert S.text(m.offset) == r["offset_text"]
        assert [[S.to_tree(a), S.to_tree(b)] for a, b in m.mask] == r["mask"]
        assert [[S.text(a), S.text(b)] for a, b in m.mask] == r["mask_text"]
        assert [S.to_tree(s) for s in m.lane_sizes] == r["lane_sizes"]
        assert [S.to_tree(s) for s in m.nest_sizes] == r["nest_sizes"]
        assert [S.to_tree(s) for s in m.source_index] == r["source_index"]
    assert ir_tree(ck.spec.application) == ref["application"]
    assert [[p.name, p.rank, p.role] for p in ck.spec.params] == \
        [[p[0], p[1], p[3]] for p in ref["params"]]


def test_builder_defined_specs_typecheck():
    sd = C.checked("sdpa")
    assert [S.text(s) for s in sd.grid.sizes] == ["q_size_0", "q_size_1",
                                                  "cdiv(q_size_2, BLOCK_SIZE_M)"]
    assert [S.text(s) for s in sd.index_maps["k"].nest_sizes] == ["cdiv(k_size_2, BLOCK_SIZE_N)"]
    rp = C.checked("rope")
    assert [S.text(s) for s in rp.grid.sizes] == ["input_size_1", "input_size_0 * input_size_2"]
    fr = C.checked("sdpa_rope")
    assert [S.text(s) for s in fr.grid.sizes] == ["q_size_0 * q_size_1",
                                                  "cdiv(q_size_2, BLOCK_SIZE_M)"]
    # query-side tables follow the program (outer) level, key-side tables
    # the K/V nest
    assert fr.index_maps["sin_q"].nest_sizes == ()
    assert [S.text(s) for s in fr.index_maps["cos_k"].nest_sizes] == \
        ["cdiv(cos_k_size_0, BLOCK_SIZE_N)"]
    checks = [(S.text(a), S.text(b)) for a, b in fr.grid.checks]
    assert ("cdiv(q_size_2, BLOCK_SIZE_M)", "cdiv(sin_q_size_0, BLOCK_SIZE_M)") in checks
    assert [S.text(s) for s in rp.index_maps["input"].nest_sizes] == ["cdiv(input_size_3, HALF_D)"]


@pytest.mark.parametrize("kernel", C.CATALOG_NAMES)
def test_maps_canonically_equal_to_reference(kernel):
    """The backend fingerprints maps by canonical form (symbolic.canonical),
    so a spec built in any association/commutation order matches; the
    reference's own trees must have the same canonical forms as ours."""
    ref = maps()[kernel]
    ck = C.checked(kernel)
    canon = S.canonical
    assert [canon(s) for s in ck.grid.sizes] == [canon(S.from_tree(t)) for t in ref["grid"]["sizes"]]
    for name, m in ck.index_maps.items():
        r = ref["maps"][name]
        assert canon(m.offset) == canon(S.from_tree(r["offset"]))
        assert [canon(a) for a, _ in m.mask] == [canon(S.from_tree(a)) for a, _ in r["mask"]]


def test_canonical_form_identities():
    a, b, c = S.var("a"), S.var("b"), S.var("c")
    assert S.canonical(a * (b * c)) == S.canonical((c * a) * b)
    assert S.canonical((a * b + a * c) // a) == S.canonical(b + c)
    assert S.canonical((a * 6 + 3 * b) % 3) == S.canonical(S.lit(0))
    assert S.canonical((a // b) // c) == S.canonical(a // (c * b))
    assert S.canonical(S.emin(a, b)) == S.canonical(S.emin(b, a))
    assert S.canonical(a // b) != S.canonical(a % b)
    assert S.canonical(a - a + b * 0) == S.canonical(S.lit(0))


def test_decompose_pid_matches_reference_points():
    from paper_2507_11978_b200.arrange import decompose_pid
    from helpers import map_cases

    index, arrays = map_cases()
    for ci, case in enumerate(index):
        ck = C.checked(case["kernel"])
        pids = arrays[f"c{ci}_pids"]
        for p in range(pids.shape[0]):
            assert decompose_pid(ck.grid, p, case["binding"]) == tuple(int(v) for v in pids[p])
    with pytest.raises(ArrangeError):
        decompose_pid(ck.grid, pids.shape[0], case["binding"])


def test_flatten_of_flattened_dims_decodes_one_level_deep():
    """flatten(flatten(x)) == flatten over all dims at once (same maps)."""
    t = param_with_shape("x", (3, 4, 5))
    once = t.flatten(0, 3).tile((7,))
    twice = t.flatten(0, 2).flatten(0, 2).tile((7,))
    a, b = lower([("x", once)]), lower([("x", twice)])
    assert a[0].offset == b[0].offset and a[0].mask == b[0].mask


def test_inner_views_compose_with_outer_rewrites():
    """with_inner keeps the substitutions of both views (mm's
    `input_tiled.dtype = input_tiled.dtype.squeeze(0)` pattern)."""
    x = param_with_shape("x", (8, 6)).tile((4, 3)).tile((1, -1))
    y = x.with_inner(x.inner().squeeze(0))
    m = lower([("x", y)])[0]
    assert len(m.nest_sizes) == 1 and len(m.lane_sizes) == 2
    env = {"x_stride_0": 6, "x_stride_1": 1, "pid_0": 1, "pid_1": 0, "nest_0": 1,
           "lane_0": 2, "lane_1": 1}
    # row 4*1 + 2, column 3*1 + 1
    assert S.evaluate(m.offset, env) == 6 * 6 + 4
