"""CPU: pin the oracle (oracle/ak_oracle.c) against the reference.

Two independent anchors:
  * tests/golden/reference_golden.npz -- outputs of the reference itself, recorded by
    tests/golden/make_golden.py from oracle/_ref (reference sources compiled in place);
  * the live reference library oracle/_ref/libakref.so when it is present.
Plus the reference's own known-answer tests (tests/test_primitives.cpp, SPEC.md examples).
"""
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "reference_golden.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def test_golden_sort_family(orc, gold):
    for s in ("int32", "uint32", "int64", "uint64", "float32", "float64"):
        x = gold[f"sort_{s}_in"]
        assert np.array_equal(orc.merge_sort(x).view(np.uint8), gold[f"sort_{s}_asc"].view(np.uint8))
        assert np.array_equal(orc.merge_sort(x, True).view(np.uint8), gold[f"sort_{s}_desc"].view(np.uint8))
        assert np.array_equal(orc.sortperm(x), gold[f"sortperm_{s}_u64"])
        assert np.array_equal(orc.sortperm(x, True).astype(np.int32), gold[f"sortperm_{s}_i32_desc"])
        assert np.array_equal(orc.sortperm(x), gold[f"sortperm_lowmem_{s}_u64"])
        k, v = orc.merge_sort_by_key(x, gold[f"bykey_{s}_payload_in"])
        assert np.array_equal(k.view(np.uint8), gold[f"bykey_{s}_keys"].view(np.uint8))
        assert np.array_equal(v, gold[f"bykey_{s}_payload"])
    assert orc.sortperm(gold["signed_zero_in"]).tolist() == gold["signed_zero_sortperm"].tolist() == [5, 0, 1, 3, 4, 2]


def test_golden_reduce_scan_search(orc, gold):
    x = gold["reduce_i64_in"]
    assert orc.reduce(x, "sum") == gold["reduce_i64_sum"][0]
    assert orc.reduce(x, "min") == gold["reduce_i64_min"][0]
    assert orc.reduce(x, "max") == gold["reduce_i64_max"][0]
    assert np.array_equal(orc.scan(x, True), gold["scan_i64_incl"])
    assert np.array_equal(orc.scan(x, False), gold["scan_i64_excl"])
    assert np.array_equal(orc.scan(gold["scan_i32_init100_in"], True, 100), gold["scan_i32_init100"])
    xf = gold["reduce_f32_in"]
    # at 2e4 elements the reference's f32 fold is still accurate: both within 1e-5
    assert abs(orc.reduce(xf) - float(gold["reduce_f32_sum_ref"][0])) <= 1e-5 * abs(orc.reduce(xf))
    assert np.array_equal(orc.searchsorted(gold["search_hay"], gold["search_needles"], "first"), gold["search_first"])
    assert np.array_equal(orc.searchsorted(gold["search_hay"], gold["search_needles"], "last"), gold["search_last"])


@pytest.mark.parametrize("name", ["sih_uniform_p4", "sih_uniform_p8", "sih_zipf_p4", "sih_equal_p4",
                                  "sih_u64_p3", "sih_f64_p4"])
def test_golden_sihsort(orc, gold, name):
    P = int(gold[f"{name}_P"][0])
    ins = [gold[f"{name}_in{r}"] for r in range(P)]
    outs, stats, _ = orc.sihsort(ins)
    for r in range(P):
        assert np.array_equal(outs[r], gold[f"{name}_out{r}"])
        s = stats[r]
        row = [s["rounds_used"], s["converged"], s["max_deviation"], s["redistribution_sends"],
               s["redistribution_bytes"], s["collective_ops"], s["output_count"]]
        assert np.array_equal(np.array(row, dtype=np.float64), gold[f"{name}_stats"][r])


def test_spec_known_answers(orc):
    assert orc.merge_sort(np.array([3, 2, 1], dtype=np.int64)).tolist() == [1, 2, 3]
    assert orc.sortperm(np.array([30, 10, 20], dtype=np.int64)).tolist() == [1, 2, 0]  # :214
    assert orc.sortperm(np.full(5, 3, dtype=np.int64)).tolist() == [0, 1, 2, 3, 4]  # :216
    k, v = orc.merge_sort_by_key(np.array([1, 1], dtype=np.int64), np.array([10, 20]))  # :206
    assert v.tolist() == [10, 20]
    assert orc.sample_positions(10, 3).tolist() == [0, 5, 9]  # sample [1..10], k=3 -> [1, 6, 10] (:288)
    assert orc.sample_positions(10, 1).tolist() == [5]  # k=1 -> median position -> 6 (:289)
    outs, stats, _ = orc.sihsort([np.array([r], dtype=np.int64) for r in range(4)])  # :280
    assert [o.tolist() for o in outs] == [[0], [1], [2], [3]]
    outs, stats, _ = orc.sihsort([np.full(1000, 5, dtype=np.int64) for _ in range(4)])  # :316
    assert [len(o) for o in outs] == [4000, 0, 0, 0]
    assert stats[0]["rounds_used"] == 4 and stats[0]["converged"] == 0
    outs, stats, spl = orc.sihsort([np.array([1, 2, 9], dtype=np.int64), np.array([3, 8, 10], dtype=np.int64)])
    assert sorted(np.concatenate(outs).tolist()) == [1, 2, 3, 8, 9, 10]
    assert np.concatenate(outs).tolist() == [1, 2, 3, 8, 9, 10]


def test_primitives_known_answers(orc):  # reference tests/test_primitives.cpp:36-175
    assert orc.reduce(np.arange(1, 101, dtype=np.int64)) == 5050
    assert orc.scan(np.ones(4, dtype=np.int32)).tolist() == [1, 2, 3, 4]
    assert orc.scan(np.array([1, 2, 3], dtype=np.int32), False).tolist() == [0, 1, 3]
    hay = np.array([1, 2, 4, 4, 7], dtype=np.int32)
    nd = np.array([4, 0, 9], dtype=np.int32)
    assert orc.searchsorted(hay, nd, "first").tolist() == [2, 0, 5]
    assert orc.searchsorted(hay, nd, "last").tolist() == [4, 0, 5]


needs_ref = pytest.mark.skipif("not __import__('oracle').ref_available()")


@needs_ref
@pytest.mark.parametrize("dt", [np.int32, np.uint32, np.int64, np.uint64, np.float32, np.float64])
@pytest.mark.parametrize("n", [0, 1, 2, 17, 5000])
def test_oracle_vs_live_reference_sort(orc, dt, n):
    rng = np.random.default_rng(n)
    dt = np.dtype(dt)
    if dt.kind == "f":
        x = rng.uniform(-1e6, 1e6, n).astype(dt)
    else:
        x = rng.integers(0, 50, n).astype(dt)  # many ties
    for desc in (False, True):
        assert np.array_equal(orc.merge_sort(x, desc), orc.ref_merge_sort(x, 4, desc))
        assert np.array_equal(orc.sortperm(x, desc), orc.ref_sortperm(x, np.uint64, 3, False, desc))
        assert np.array_equal(orc.sortperm(x, desc), orc.ref_sortperm(x, np.uint64, 2, True, desc))


@needs_ref
@pytest.mark.parametrize("P", [1, 2, 3, 4, 8, 16])
@pytest.mark.parametrize("kind", ["uniform", "zipf", "equal", "sorted", "reversed"])
def test_oracle_vs_live_reference_sihsort(orc, P, kind):
    rng = np.random.default_rng(P)
    n = 3000
    if kind == "uniform":
        ins = [rng.integers(-2**63, 2**63 - 1, n, dtype=np.int64) for _ in range(P)]
    elif kind == "zipf":
        ins = [np.minimum(rng.zipf(1.1, n), 10**6).astype(np.int64) for _ in range(P)]
    elif kind == "equal":
        ins = [np.full(n, 9, dtype=np.int64) for _ in range(P)]
    elif kind == "sorted":
        ins = [np.arange(r * n, (r + 1) * n, dtype=np.int64) for r in range(P)]
    else:
        ins = [np.arange((P - r) * n, (P - r - 1) * n, -1, dtype=np.int64) for r in range(P)]
    a, sa, _ = orc.sihsort(ins)
    b, sb = orc.ref_sihsort(ins, threads_per_rank=1)
    for r in range(P):
        assert np.array_equal(a[r], b[r])
    assert sa == sb


@needs_ref
def test_oracle_vs_live_reference_configs(orc):
    ins = [np.random.default_rng(r).integers(-50, 50, 2000).astype(np.int64) for r in range(4)]
    for cfg in (orc.SihConfig(7, 3, 0, 0.25), orc.SihConfig(0, 0, 1, 0.01), orc.SihConfig(1, 1, 4, 0.5)):
        a, sa, _ = orc.sihsort(ins, cfg)
        b, sb = orc.ref_sihsort(ins, cfg, 1)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))
        assert sa == sb
