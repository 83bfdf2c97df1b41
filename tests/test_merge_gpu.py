"""GPU parity: stable P-way merge (K8, search_merge.cu merge_runs) -- the second local
sort of SIHSort (sihsort.hpp:555) done as one merge of the P received runs.

Oracle: the stable sort of the runs' concatenation (oracle.merge_sort, pinned to the
reference). Float runs carry -0.0 / +0.0, which compare equal: their output order shows
that ties keep run order (stability), bit for bit.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def runs_for(rng, P, sizes, dt, kind="uniform"):
    out = []
    for r in range(P):
        n = sizes[r]
        if kind == "uniform":
            if np.dtype(dt).kind == "f":
                x = rng.uniform(-1e3, 1e3, n).astype(dt)
                x[rng.integers(0, max(n, 1), n // 7)] = 0.0 if r % 2 else -0.0
            else:
                info = np.iinfo(dt)
                x = rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)
        elif kind == "dups":
            x = rng.integers(0, 3, n).astype(dt)
        else:
            x = np.full(n, 5, dtype=dt)
        out.append(np.sort(x, kind="stable"))
    return out


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8, 16])
@pytest.mark.parametrize("dt", [np.int64, np.uint64, np.float32, np.float64, np.int32])
def test_merge_runs_matches_stable_sort(ak, orc, ex, dev, P, dt):
    rng = np.random.default_rng(P * 31 + np.dtype(dt).itemsize)
    sizes = [int(s) for s in rng.integers(0, 60_000, P)]
    sizes[0] = 0 if P > 2 else sizes[0]  # an empty run among the others
    runs = runs_for(rng, P, sizes, dt)
    got = ak.merge_runs([torch.from_numpy(r).to(dev) for r in runs], ex=ex).cpu().numpy()
    want = orc.merge_sort(np.concatenate(runs)) if sum(sizes) else np.zeros(0, dt)
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8))


@pytest.mark.parametrize("kind", ["dups", "equal"])
def test_merge_runs_duplicates_fallback(ak, ex, dev, kind):
    # massive ties exceed a tile: the oversized-tile path (stable radix of the segment)
    rng = np.random.default_rng(1)
    runs = runs_for(rng, 8, [200_000] * 8, np.int64, kind)
    got = ak.merge_runs([torch.from_numpy(r).to(dev) for r in runs], ex=ex).cpu().numpy()
    assert np.array_equal(got, np.sort(np.concatenate(runs)))


def test_merge_runs_large_8way(ak, ex, dev):
    P, n = 8, 1 << 23
    runs = [torch.sort(torch.randint(-2**62, 2**62, (n,), device=dev))[0] for _ in range(P)]
    got = ak.merge_runs(runs, ex=ex)
    want = torch.sort(torch.cat(runs))[0]
    assert torch.equal(got, want)


def test_merge_runs_descending(ak, ex, dev):
    rng = np.random.default_rng(9)
    runs = [np.sort(rng.integers(-1000, 1000, 30_000))[::-1].copy() for _ in range(5)]
    got = ak.merge_runs([torch.from_numpy(r).to(dev) for r in runs], ex=ex, cmp="greater").cpu().numpy()
    assert np.array_equal(got, np.sort(np.concatenate(runs))[::-1])


@pytest.mark.parametrize("P", [6, 8, 16])
@pytest.mark.parametrize("kind", ["uniform", "ties", "narrow"])
def test_merge_runs_value_tiles_int64(ak, ex, dev, P, kind):
    """P >= 6 int64 runs >= 2^22 keys take the one-pass value-tile merge (radix_sort.cu,
    merge_runs_counting); ties and narrow ranges exercise the clustered-tile fallback."""
    n = (1 << 22) + 12345
    g = torch.Generator(device=dev).manual_seed(P)
    if kind == "uniform":
        x = torch.randint(-(1 << 62), 1 << 62, (n,), device=dev, generator=g)
    elif kind == "ties":
        x = torch.randint(0, 5000, (n,), device=dev, generator=g) * 1000003
    else:
        x = torch.randint(-300, 300, (n,), device=dev, generator=g) + (1 << 40)
    cuts = sorted(torch.randint(0, n, (P - 1,), generator=torch.Generator().manual_seed(P)).tolist())
    bounds = [0] + cuts + [n]
    runs = [torch.sort(x[bounds[r]:bounds[r + 1]])[0] for r in range(P)]
    out = torch.empty(n, dtype=torch.int64, device=dev)
    ak.merge_runs(runs, out=out, scratch=torch.empty_like(out), ex=ex)
    assert torch.equal(out, torch.sort(x)[0])
    for r in runs:  # descending
        r.copy_(torch.flip(r, [0]))
    ak.merge_runs(runs, out=out, scratch=torch.empty_like(out), ex=ex, cmp="greater")
    assert torch.equal(out, torch.sort(x, descending=True)[0])
