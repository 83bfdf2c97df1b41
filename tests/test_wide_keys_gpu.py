"""GPU parity of the int16 and int128 sort keys (dtype.hpp:14-21; csrc/wide_keys.cu):
merge_sort, merge_sort_by_key, sortperm and sortperm_lowmem against Python's stable sort
(sorted() is stable, and reverse=True keeps equal keys in input order -- std::greater)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def stable_perm(vals, desc):
    return sorted(range(len(vals)), key=lambda i: vals[i], reverse=desc)


def i128_tensor(vals, dev):
    lo = [v & ((1 << 64) - 1) for v in vals]
    hi = [(v >> 64) for v in vals]
    a = np.empty((len(vals), 2), dtype=np.uint64)
    a[:, 0] = lo
    a[:, 1] = np.array(hi, dtype=np.int64).view(np.uint64)
    return torch.from_numpy(a.view(np.int64)).to(dev)


def i128_values(t):
    a = t.cpu().numpy().view(np.uint64)
    return [int(lo) | (int(np.int64(np.uint64(hi))) << 64) for lo, hi in a]


def i128_keys(rng, n):
    pool = [int(rng.integers(-(1 << 62), 1 << 62)) * (1 << 64) + int(rng.integers(0, 1 << 63)) * 2 for _ in range(n // 3)]
    vals = [int(rng.integers(-(1 << 62), 1 << 62)) << int(rng.integers(0, 64)) for _ in range(n - len(pool))] + pool
    vals[::7] = [vals[1]] * len(vals[::7])  # ties
    if n > 6:
        vals[5] = -(1 << 127)
        vals[6] = (1 << 127) - 1
    rng.shuffle(vals)
    return vals


@pytest.mark.parametrize("n", [1, 2, 1000, 70_001])
@pytest.mark.parametrize("desc", [False, True])
def test_int16_sort_family(ak, ex, dev, n, desc):
    rng = np.random.default_rng(n)
    x = rng.integers(-32768, 32768, n).astype(np.int16)
    x[::5] = 7
    cmp = "greater" if desc else None
    want = stable_perm(x.tolist(), desc)
    d = torch.from_numpy(x.copy()).to(dev)
    ak.merge_sort(d, ex=ex, cmp=cmp)
    assert d.cpu().numpy().tolist() == [int(x[i]) for i in want]
    for idx in (torch.int32, torch.int64):
        p = ak.sortperm(torch.from_numpy(x).to(dev), ex=ex, cmp=cmp, index_dtype=idx)
        assert p.cpu().numpy().tolist() == want
        q = ak.sortperm_lowmem(torch.from_numpy(x).to(dev), ex=ex, cmp=cmp, index_dtype=idx)
        assert q.cpu().numpy().tolist() == want
    k = torch.from_numpy(x.copy()).to(dev)
    v = torch.arange(n, dtype=torch.int32, device=dev)
    ak.merge_sort_by_key(k, v, ex=ex, cmp=cmp)
    assert v.cpu().numpy().tolist() == want


@pytest.mark.parametrize("n", [2, 999, 30_011])
@pytest.mark.parametrize("desc", [False, True])
def test_int128_sort_family(ak, ex, dev, n, desc):
    rng = np.random.default_rng(128 + n)
    vals = i128_keys(rng, n)
    cmp = "greater" if desc else None
    want = stable_perm(vals, desc)
    d = i128_tensor(vals, dev)
    ak.merge_sort(d, ex=ex, cmp=cmp)
    assert i128_values(d) == [vals[i] for i in want]
    for idx in (torch.int32, torch.int64):
        p = ak.sortperm(i128_tensor(vals, dev), ex=ex, cmp=cmp, index_dtype=idx)
        assert p.cpu().numpy().tolist() == want
        q = ak.sortperm_lowmem(i128_tensor(vals, dev), ex=ex, cmp=cmp, index_dtype=idx)
        assert q.cpu().numpy().tolist() == want
    k = i128_tensor(vals, dev)
    v = torch.arange(n, dtype=torch.int64, device=dev)
    ak.merge_sort_by_key(k, v, ex=ex, cmp=cmp)
    assert v.cpu().numpy().tolist() == want
    assert i128_values(k) == [vals[i] for i in want]
