"""Pin the CPU oracle (oracle/fm_oracle.py) against the reference's own
outputs recorded in tests/golden/ (tests/golden/make_golden.py) and the
reference tests' known answers.  CPU only."""

import math

import numpy as np
import pytest

from conftest import GOLDEN, case_env, case_expected
from oracle import fm_oracle as orc
from paper_2604_22242_b200.exprtree import ElemType
from treeio import from_json


def test_rng_streams_bit_exact():
    g = np.load(GOLDEN / "rng.npz")
    for seed in (0, 1, 42, 43, 44, 2**63 + 5):
        assert np.array_equal(orc.raw_words(seed, 64), g[f"raw_{seed}"])
        assert np.array_equal(orc.uniform_fill(seed, 4096, "f32"), g[f"u_f32_{seed}"])
        assert np.array_equal(orc.uniform_fill(seed, 4096, "f64"), g[f"u_f64_{seed}"])
        assert np.array_equal(orc.uniform_int_fill(seed, 4096, "u32", 10), g[f"i_u32_{seed}"])


def test_rng_offset_is_a_slice_of_the_stream():
    full = orc.uniform_fill(42, 1000, "f32")
    assert np.array_equal(orc.uniform_fill(42, 300, "f32", offset=500), full[500:800])


def test_rng_known_answer_formula():
    # test_matrix.py:40-50: element k of seed s from the published formula
    seed, n = 42, 4
    a = orc.randu(n, n, seed)
    for (r, c) in [(0, 0), (3, 2), (1, 3)]:
        k = r + c * n
        with np.errstate(over="ignore"):
            word = orc.mix64(np.array([np.uint64(seed) + np.uint64(k + 1) * orc.GOLDEN]))[0]
        assert a[r, c] == np.float32((int(word) >> 40) * 2.0 ** -24)


def _cases(golden_cases, prefix):
    cases, arrays = golden_cases
    return [(c, arrays) for c in cases if c["name"].startswith(prefix)]


@pytest.mark.parametrize("prefix", ["suite_", "c1_", "c3_", "c4_", "tree_", "view_", "gemm_"])
def test_materialize_numpy_mode_equals_reference_oracle(golden_cases, prefix):
    """In numpy mode the restatement reproduces the reference oracle bit for bit."""
    checked = 0
    for case, arrays in _cases(golden_cases, prefix):
        if "oracle" not in case["expected"]:
            continue
        node = from_json(case["tree"])
        got = orc.materialize(node, case_env(case, arrays), transcendental="numpy")
        exp = case_expected(case, arrays, "oracle")
        assert got.dtype == exp.dtype, case["name"]
        assert orc.max_ulp(got, exp) == 0, case["name"]
        checked += 1
    assert checked > 0


@pytest.mark.parametrize("prefix", ["suite_", "c1_", "c3_", "tree_f32", "tree_f64", "view_"])
def test_materialize_cr_mode_close_to_reference_backends(golden_cases, prefix):
    """Correctly-rounded transcendentals stay within the reference's own
    tolerances of its ref (interpreter) and cjit (glibc) backends."""
    for case, arrays in _cases(golden_cases, prefix):
        node = from_json(case["tree"])
        got = orc.materialize(node, case_env(case, arrays))
        tol = 1e-12 if node.etype is ElemType.f64 else 1e-5
        for label in ("ref", "cjit"):
            if label in case["expected"]:
                exp = case_expected(case, arrays, label)
                assert orc.allclose_mixed(got, exp), (case["name"], label)
                if "exp" not in str(case["tree"]) and "log" not in str(case["tree"]) \
                        and "tanh" not in str(case["tree"]):
                    # no transcendental: every route is bit-identical
                    assert orc.max_ulp(got, exp) == 0, (case["name"], label)
                else:
                    assert orc.compare(got, exp) <= tol or orc.allclose_mixed(got, exp), case["name"]


@pytest.mark.parametrize("prefix", ["tree_i32", "tree_u32"])
def test_integer_trees_exact(golden_cases, prefix):
    for case, arrays in _cases(golden_cases, prefix):
        node = from_json(case["tree"])
        got = orc.materialize(node, case_env(case, arrays))
        for label in ("oracle", "ref", "cjit"):
            assert np.array_equal(got, case_expected(case, arrays, label)), (case["name"], label)


def test_accu_matches_reference_backends(golden_cases):
    for case, arrays in _cases(golden_cases, "c2_"):
        node = from_json(case["tree"])
        vals = orc.materialize(node, case_env(case, arrays))
        total = orc.accu(vals, node.etype)
        for label in ("accu_ref", "accu_cjit"):
            assert total == pytest.approx(case_expected(case, arrays, label), rel=1e-12)


def test_accu_known_answers(golden_cases):
    cases, arrays = golden_cases
    by = {c["name"]: c for c in cases}
    c = by["accu_small"]
    assert orc.accu(case_env(c, arrays)[int(next(iter(c["env"])))], ElemType.f32) == 10.0
    c = by["accu_u32_wrap"]
    v = case_env(c, arrays)[int(next(iter(c["env"])))]
    assert orc.accu(v, ElemType.u32) == case_expected(c, arrays, "accu_ref") == 0


def test_gemm_f64_accumulation_bit_exact(golden_cases):
    for case, arrays in _cases(golden_cases, "gemm_"):
        node = from_json(case["tree"])
        got = orc.materialize(node, case_env(case, arrays))
        assert np.array_equal(got, case_expected(case, arrays, "ref")), case["name"]


def test_reduce_dim_semantics():
    x = np.array([[1.0, 5.0, np.nan], [3.0, 5.0, 2.0], [3.0, -1.0, 9.0]], np.float64)
    k = orc.ReduceKind
    assert orc.reduce_dim(k.index_max, 0, x, ElemType.f64).tolist() == [[1, 0, 0]]
    assert np.isnan(orc.reduce_dim(k.max, 0, x, ElemType.f64)[0, 2])
    assert orc.reduce_dim(k.index_min, 1, x, ElemType.f64).ravel().tolist() == [2, 2, 1]
    assert orc.reduce_dim(k.sum, 1, x[:, :2], ElemType.f64).ravel().tolist() == [6.0, 8.0, 2.0]
    assert orc.reduce_dim(k.mean, 0, x[:, :2], ElemType.f64).ravel().tolist() == [7 / 3, 3.0]


def test_bf16_rounding():
    x = np.array([1.0, 1.00390625, 1.005859375, 1.0078125, -3.0e38, np.inf], np.float32)
    r = orc.bf16_round(x)
    assert r[0] == 1.0 and r[1] == 1.0          # tie to even
    assert r[2] == np.float32(1.0078125)         # above half -> up
    assert np.isinf(orc.bf16_round(np.array([3.4e38], np.float32))[0])
    d = np.array([1.0 + 2.0 ** -8 + 2.0 ** -40], np.float64)   # just above the tie
    assert orc.bf16_from_f64(d)[0] == np.float32(1.0078125)
    assert orc.bf16_round(d.astype(np.float32))[0] == 1.0         # double rounding would tie-to-even


def test_ulp_metric():
    a = np.array([1.0, 2.0], np.float32)
    b = np.nextafter(a, np.float32(3))
    assert orc.max_ulp(a, b) == 1
    assert orc.max_ulp(np.float32([0.0]), np.float32([-0.0])) == 0
    assert math.isinf(orc.compare(np.array([np.nan]), np.array([1.0])))


# --- north-star ops pinned through the reference ---------------------------
def _pin_cases(golden_cases, prefix):
    cases, arrays = golden_cases
    return [(c, arrays) for c in cases if c["name"].startswith(prefix)]


def test_dim_sums_pinned_to_reference_submat_accu(golden_cases):
    """sum / mean along dim 0 and dim 1 equal the reference's own
    accu(V.submat(...)) of each column / row (matrix.py:258, 481-496); max /
    min / index_* follow numpy on the values the reference computed."""
    from conftest import case_env
    from treeio import from_json
    cases = _pin_cases(golden_cases, "pin_c4_")
    assert len(cases) == 3
    for c, arrays in cases:
        node = from_json(c["tree"])
        v = orc.materialize(node, case_env(c, arrays))
        ety = node.etype
        assert np.array_equal(v, arrays[c["expected"]["cjit"]])          # exact elementwise
        colsum = arrays[c["expected"]["colsum_ref"]]
        rowsum = arrays[c["expected"]["rowsum_ref"]]
        K = orc.ReduceKind
        mag0 = np.abs(v.astype(np.float64)).sum(axis=0)
        mag1 = np.abs(v.astype(np.float64)).sum(axis=1)
        s0 = orc.reduce_dim(K.sum, 0, v, ety).ravel().astype(np.float64)
        s1 = orc.reduce_dim(K.sum, 1, v, ety).ravel().astype(np.float64)
        tol = 1e-13 if ety is orc.ElemType.f64 else 2 ** -24
        if ety is orc.ElemType.f64:
            assert np.all(np.abs(s0 - colsum) <= tol * mag0)
            assert np.all(np.abs(s1 - rowsum) <= tol * mag1)
        else:                       # f32 output: the f64 sum rounded once
            assert np.array_equal(s0.astype(np.float32), colsum.astype(np.float32))
            assert np.array_equal(s1.astype(np.float32), rowsum.astype(np.float32))
        m0 = orc.reduce_dim(K.mean, 0, v, ety).ravel().astype(np.float64)
        assert np.all(np.abs(m0 - colsum / v.shape[0]) <= max(tol, 2 ** -24) * mag0 / v.shape[0])


def test_norm_and_dot_pinned_to_reference_accu(golden_cases):
    from conftest import case_env
    for c, arrays in _pin_cases(golden_cases, "pin_norm_dot_"):
        env = case_env(c, arrays)
        x, y = (env[k] for k in sorted(env))
        ety = orc.ElemType.f32 if x.dtype == np.float32 else orc.ElemType.f64
        normsq = c["expected"]["normsq_ref"]["scalar"]
        dot = c["expected"]["dot_ref"]["scalar"]
        assert abs(orc.accu((x - y) * (x - y), ety) - normsq) <= 1e-12 * normsq
        assert abs(orc.accu(x * y, ety) - dot) <= 1e-12 * dot
