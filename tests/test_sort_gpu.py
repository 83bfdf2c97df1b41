"""GPU parity: sort family (merge_sort / by_key / sortperm / sortperm_lowmem) vs the oracle.

Oracle = oracle/ak_oracle.c, the C restatement of sort.hpp:75-290 (pinned to the
reference in tests/test_oracle.py). Integer and float keys: bit-exact.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

DTYPES = [np.int32, np.uint32, np.int64, np.uint64, np.float32, np.float64]
SIZES = [0, 1, 2, 31, 1000, 6143, 6144, 6145, 100_003]


def keys_for(rng, dt, n, kind="uniform"):
    dt = np.dtype(dt)
    if kind == "uniform":
        if dt.kind == "f":
            x = rng.uniform(-1e6, 1e6, n).astype(dt)
            if n > 10:
                x[rng.integers(0, n, n // 10)] = 0.0
                x[rng.integers(0, n, n // 10)] = -0.0
            return x
        info = np.iinfo(dt)
        return rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)
    if kind == "few":
        return rng.integers(0, 5, n).astype(dt)
    if kind == "equal":
        return np.full(n, 7, dtype=dt)
    if kind == "sorted":
        return np.sort(keys_for(rng, dt, n))
    if kind == "reversed":
        return np.sort(keys_for(rng, dt, n))[::-1].copy()
    raise ValueError(kind)


def tdev(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("n", SIZES)
def test_merge_sort_matches_oracle(ak, orc, ex, dev, dt, n):
    rng = np.random.default_rng(n * 7 + np.dtype(dt).itemsize)
    x = keys_for(rng, dt, n)
    for desc in (False, True):
        d = tdev(x, dev)
        ak.merge_sort(d, ex=ex, cmp="greater" if desc else None)
        got = d.cpu().numpy()
        want = orc.merge_sort(x, descending=desc)
        assert np.array_equal(got.view(np.uint8), want.view(np.uint8))  # bit-exact, incl. -0.0


@pytest.mark.parametrize("kind", ["few", "equal", "sorted", "reversed"])
@pytest.mark.parametrize("dt", [np.int64, np.float32])
def test_merge_sort_distributions(ak, orc, ex, dev, kind, dt):
    x = keys_for(np.random.default_rng(3), dt, 50_001, kind)
    d = tdev(x, dev)
    ak.merge_sort(d, ex=ex)
    assert np.array_equal(d.cpu().numpy(), orc.merge_sort(x))


def test_merge_sort_config1_1e6_int64(ak, orc, ex, dev):
    # BASELINE config 1: merge_sort of 1M uniform-random Int64 keys (reference bench keys)
    x = ak.bench_keys(42, 0, 1_000_000, np.int64)
    d = tdev(x, dev)
    ak.merge_sort(d, ex=ex)
    assert np.array_equal(d.cpu().numpy(), orc.merge_sort(x))
    assert np.array_equal(d.cpu().numpy(), orc.ref_merge_sort(x, threads=4)) if orc.ref_available() else True


def test_spec_known_answers(ak, ex, dev):
    d = tdev(np.array([3, 2, 1], dtype=np.int64), dev)
    ak.merge_sort(d, ex=ex)
    assert d.cpu().tolist() == [1, 2, 3]
    p = ak.sortperm(tdev(np.array([30, 10, 20], dtype=np.int64), dev), ex=ex)
    assert p.cpu().tolist() == [1, 2, 0]
    p = ak.sortperm_lowmem(tdev(np.array([30, 10, 20], dtype=np.int64), dev), ex=ex)
    assert p.cpu().tolist() == [1, 2, 0]
    p = ak.sortperm(tdev(np.full(5, 9, dtype=np.int64), dev), ex=ex)
    assert p.cpu().tolist() == [0, 1, 2, 3, 4]
    k = tdev(np.array([1, 1], dtype=np.int64), dev)
    v = tdev(np.array([10, 20], dtype=np.int32), dev)
    ak.merge_sort_by_key(k, v, ex=ex)
    assert v.cpu().tolist() == [10, 20]
    k = tdev(np.array([2, 1], dtype=np.int64), dev)
    v = tdev(np.array([20, 10], dtype=np.int64), dev)
    ak.merge_sort_by_key(k, v, ex=ex)
    assert k.cpu().tolist() == [1, 2] and v.cpu().tolist() == [10, 20]


def test_signed_zero_stability(ak, orc, ex, dev):
    # std::less treats -0.0 == +0.0; stable order kept
    x = np.array([0.0, -0.0, 1, -0.0, 0.0, -1], dtype=np.float32)
    for lowmem in (False, True):
        f = ak.sortperm_lowmem if lowmem else ak.sortperm
        p = f(tdev(x, dev), ex=ex)
        assert p.cpu().tolist() == [5, 0, 1, 3, 4, 2]
    if orc.ref_available():
        assert orc.ref_sortperm(x).tolist() == [5, 0, 1, 3, 4, 2]


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("idx", [torch.int32, torch.int64])
@pytest.mark.parametrize("n", [0, 1, 5, 6145, 70_001])
def test_sortperm_matches_oracle(ak, orc, ex, dev, dt, idx, n):
    rng = np.random.default_rng(11 + n)
    x = keys_for(rng, dt, n, "few" if n % 2 else "uniform")
    for desc in (False, True):
        want = orc.sortperm(x, descending=desc)
        cmp = "greater" if desc else None
        p = ak.sortperm(tdev(x, dev), ex=ex, cmp=cmp, index_dtype=idx)
        assert np.array_equal(p.cpu().numpy().astype(np.uint64), want)
        q = ak.sortperm_lowmem(tdev(x, dev), ex=ex, cmp=cmp, index_dtype=idx)
        assert np.array_equal(q.cpu().numpy().astype(np.uint64), want)


@pytest.mark.parametrize("kt", [np.float32, np.int64, np.float64, np.uint32])
@pytest.mark.parametrize("vt", [np.int32, np.int64, np.float32])
def test_by_key_matches_oracle(ak, orc, ex, dev, kt, vt):
    rng = np.random.default_rng(5)
    n = 40_000
    k = keys_for(rng, kt, n, "few")
    v = np.arange(n).astype(vt)
    want_k, want_v = orc.merge_sort_by_key(k, v)
    dk, dv = tdev(k, dev), tdev(v, dev)
    ak.merge_sort_by_key(dk, dv, ex=ex)
    assert np.array_equal(dk.cpu().numpy(), want_k)
    assert np.array_equal(dv.cpu().numpy(), want_v)


def test_argument_errors(ak, ex, dev):
    d = torch.zeros(10, dtype=torch.int64, device=dev)
    with pytest.raises(ak.InvalidArgument):  # sort.hpp:182-184
        ak.merge_sort(d, torch.zeros(9, dtype=torch.int64, device=dev), ex=ex)
    with pytest.raises(ak.InvalidArgument):  # sort.hpp:214-216
        ak.merge_sort_by_key(d, torch.zeros(9, dtype=torch.int32, device=dev), ex=ex)
    with pytest.raises(ak.InvalidArgument):  # sort.hpp:242-244
        ak.sortperm(d, out=torch.zeros(9, dtype=torch.int64, device=dev), ex=ex)
    with pytest.raises(ak.InvalidArgument):  # sort.hpp:270-272
        ak.sortperm_lowmem(d, out=torch.zeros(11, dtype=torch.int64, device=dev), ex=ex)
    with pytest.raises(ak.InvalidArgument):
        ak.merge_sort(d, ex=ex, cmp=lambda a, b: a < b)  # no custom comparators on the cuda kind


def test_config2_sortperm_1e8_f32_properties(ak, ex, dev):
    """BASELINE config 2 at full size (1e8 f32 -> int32): permutation, sortedness, stability."""
    n = 100_000_000
    x = ak.bench_keys(42, 0, n, np.float32)
    dx = tdev(x, dev)
    p = ak.sortperm(dx, ex=ex, index_dtype=torch.int32).long()
    assert torch.equal(torch.bincount(p, minlength=n), torch.ones(n, dtype=torch.int64, device=dev))
    s = dx[p]
    assert bool((s[1:] >= s[:-1]).all())
    tie = s[1:] == s[:-1]
    assert bool((p[1:][tie] > p[:-1][tie]).all())  # stable: equal keys keep ascending indices
    # by_key with int32 iota payload must give the same permutation
    k = dx.clone()
    v = torch.arange(n, dtype=torch.int32, device=dev)
    ak.merge_sort_by_key(k, v, ex=ex)
    assert torch.equal(v.long(), p)
    assert torch.equal(k, s)


@pytest.mark.parametrize("dt", [np.float32, np.int32, np.uint32])
@pytest.mark.parametrize("idx", [torch.int32, torch.int64])
def test_sortperm_composite_path_matches_oracle(ak, orc, ex, dev, dt, idx):
    """n >= 2^20 32-bit integer keys take the composite (key, index) 64-bit sort
    (sortperm_fast.cu); float keys the onesweep. Bit-exact vs the oracle, ties and
    -0.0/+0.0 included, both directions."""
    n = 1_500_001
    rng = np.random.default_rng(20)
    if dt == np.float32:
        x = rng.uniform(-1e6, 1e6, n).astype(np.float32)
        x[rng.integers(0, n, 20_000)] = 0.0
        x[rng.integers(0, n, 20_000)] = -0.0
        x[rng.integers(0, n, 50_000)] = x[7]
    else:
        info = np.iinfo(dt)
        x = rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)
        x[rng.integers(0, n, 100_000)] = x[3]
    for desc in (False, True):
        want = orc.sortperm(x, descending=desc)
        p = ak.sortperm(tdev(x, dev), ex=ex, cmp="greater" if desc else None, index_dtype=idx)
        assert np.array_equal(p.cpu().numpy().astype(np.uint64), want)


@pytest.mark.parametrize("desc", [False, True])
def test_sortperm_composite_msd_sizes_int32(ak, ex, dev, desc):
    """n >= 2^24 int32 sortperm: the composite 64-bit keys take the MSD partition passes too."""
    n = (1 << 24) + 3
    rng = np.random.default_rng(2424)
    x = rng.integers(-(1 << 31), 1 << 31, n, dtype=np.int64).astype(np.int32)
    x[rng.integers(0, n, 1 << 20)] = x[11]  # ties
    want = np.argsort(-x.astype(np.int64) if desc else x, kind="stable")
    p = ak.sortperm(torch.from_numpy(x).to(dev), ex=ex, cmp="greater" if desc else None, index_dtype=torch.int32)
    assert np.array_equal(p.cpu().numpy(), want)


@pytest.mark.parametrize("n", [1_000_000, (1 << 23) + 5])
def test_merge_sort_host_pageable_and_pinned(ak, ex, n):
    """merge_sort_host on host arrays: a pageable numpy array (>= 32 MB is page-locked for the
    call and released after it), an array that is already pinned (left alone), and the same
    pageable array twice (a second registration of the same range must work)."""
    x = ak.bench_keys(42, 1, n, np.int64)
    want = np.sort(x)
    for _ in range(2):
        y = x.copy()
        ak.merge_sort_host(y, ex)
        assert np.array_equal(y, want)
    pinned = torch.empty(n, dtype=torch.int64, pin_memory=True)
    pinned.numpy()[:] = x
    ak.merge_sort_host(pinned.numpy(), ex)
    assert np.array_equal(pinned.numpy(), want)


def test_sihsort_host_large_pageable(ak, ex):
    """sihsort_host with pageable input and output arrays over 32 MB (both page-locked for the
    call): equals the sorted input."""
    n = (1 << 22) + 3
    x = ak.bench_keys(7, 0, n, np.int64)
    out, st = ak.sihsort_host(x, None, None, ex)
    assert np.array_equal(out, np.sort(x))
