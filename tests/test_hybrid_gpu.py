"""GPU parity of the hybrid 64-bit keys sort (radix_sort.cu: hybrid_sort_keys).

The hybrid picks (m global top-digit passes, bucket/step range mode, 8/12/16-item local
CTAs) from n, and falls back to the segment LSD for ranges that do not fit on chip. These
sizes and distributions drive every branch: single-CTA (n <= 6144), m = 1 bucket mode,
m = 2 step mode, m = 2 bucket mode with 8- and 12-item CTAs, narrow bucket digits, and
oversized ranges (few distinct top bits, heavy duplicates, clusters). Keys-only integer
sorts have a unique answer, so numpy's sort is an exact oracle at sizes the C oracle would
take minutes on; the C oracle is used where it is fast.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SIZES = [6144, 6145, 50_000, 1 << 20, (1 << 22) + 3, 3 << 23, 1 << 27]


def dist(rng, n, kind, dt=np.int64):
    info = np.iinfo(dt)
    if kind == "uniform":
        return rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)
    if kind == "low40":  # top 24 bits constant: one giant bucket -> oversized-range fallback
        return rng.integers(0, 1 << 40, n, dtype=np.int64).astype(dt)
    if kind == "dups":  # heavy duplicates spread over the key space
        pool = rng.integers(info.min, info.max, 97, dtype=dt, endpoint=True)
        return pool[rng.integers(0, 97, n)]
    if kind == "cluster":  # half the keys in one bucket, half uniform
        x = rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)
        x[: n // 2] = (x[: n // 2] & 0xFFFF) + (0x1234 << 40)
        rng.shuffle(x)
        return x
    if kind == "midconst":  # bits 16..47 constant: every bucket is one long run of equal high bits
        x = rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)
        return (x & ~np.int64(0xFFFFFFFF0000)) | np.int64(0x5A5A5A5A0000)
    if kind == "runs40":  # high 32 bits from a pool of n/40 values: runs of ~40 for the insertion fix-up
        pool = rng.integers(-(1 << 31), 1 << 31, max(1, n // 40), dtype=np.int64)
        hi = pool[rng.integers(0, pool.size, n)] << 32
        return hi | rng.integers(0, 1 << 32, n, dtype=np.int64)
    if kind == "sorted":
        return np.sort(rng.integers(info.min, info.max, n, dtype=dt, endpoint=True))
    if kind == "reversed":
        return np.sort(rng.integers(info.min, info.max, n, dtype=dt, endpoint=True))[::-1].copy()
    raise ValueError(kind)


@pytest.mark.parametrize("n", SIZES)
def test_hybrid_uniform_sizes(ak, ex, dev, n):
    x = ak.bench_keys(42, 3, n, np.int64)
    d = torch.from_numpy(x).to(dev)
    s = torch.empty_like(d)
    ak.merge_sort(d, s, ex)
    assert np.array_equal(d.cpu().numpy(), np.sort(x))


@pytest.mark.parametrize("kind", ["low40", "dups", "cluster", "midconst", "runs40", "sorted", "reversed"])
@pytest.mark.parametrize("n", [50_000, 1 << 20, 3 << 22])
def test_hybrid_distributions(ak, ex, dev, kind, n):
    x = dist(np.random.default_rng(n + len(kind)), n, kind)
    d = torch.from_numpy(x).to(dev)
    ak.merge_sort(d, ex=ex)
    assert np.array_equal(d.cpu().numpy(), np.sort(x))


@pytest.mark.parametrize("n", [6145, 1 << 20, 3 << 22])
def test_hybrid_descending_uint64(ak, ex, dev, n):
    x = dist(np.random.default_rng(n), n, "uniform", np.uint64)
    d = torch.from_numpy(x.view(np.int64)).to(dev)
    ak.merge_sort(d.view(torch.uint64), ex=ex, cmp="greater")
    assert np.array_equal(d.cpu().numpy().view(np.uint64), np.sort(x)[::-1])


def test_hybrid_out_of_place_copy(ak, orc, ex, dev):
    # merge_sort_copy: input untouched, output sorted (kin != kout path of the hybrid)
    x = ak.bench_keys(7, 0, 300_001, np.int64)
    d = torch.from_numpy(x).to(dev)
    y = ak.merge_sort_copy(d, ex=ex)
    assert np.array_equal(d.cpu().numpy(), x)
    assert np.array_equal(y.cpu().numpy(), orc.merge_sort(x))


def test_hybrid_f64_keys_bit_exact(ak, orc, ex, dev):
    # 64-bit float keys go through the hybrid too: -0.0 == +0.0 keeps input order
    rng = np.random.default_rng(5)
    x = rng.uniform(-1e6, 1e6, 200_000)
    x[rng.integers(0, x.size, 5000)] = 0.0
    x[rng.integers(0, x.size, 5000)] = -0.0
    d = torch.from_numpy(x).to(dev)
    ak.merge_sort(d, ex=ex)
    assert np.array_equal(d.cpu().numpy().view(np.uint64), orc.merge_sort(x).view(np.uint64))


def _fingerprint(t):
    # order-independent multiset fingerprint (int64 wrap-around arithmetic on the device)
    return (t.numel(), int(t.sum()), int((t * t).sum()), int(((t >> 17) * t).sum()), int((t ^ (t >> 29)).sum()))


@pytest.mark.parametrize("n", [(1 << 29) + 12345])
def test_hybrid_three_level_msd(ak, ex, dev, n):
    # n >= 2^29 takes three unstable MSD partition levels (24-bit cursors) before the local
    # stage; checked by on-device sortedness + multiset fingerprint (a host sort of 4 GB
    # would dominate the suite)
    g = torch.Generator(device=dev).manual_seed(29)
    x = torch.randint(-(1 << 62), 1 << 62, (n,), device=dev, dtype=torch.int64, generator=g) * 2 + 1
    fp = _fingerprint(x)
    s = torch.empty_like(x)
    ak.merge_sort(x, s, ex)
    del s
    assert bool((x[1:] >= x[:-1]).all())
    assert _fingerprint(x) == fp


@pytest.mark.parametrize("kind", ["uniform", "low40", "dups", "cluster", "midconst", "sorted"])
@pytest.mark.parametrize("desc", [False, True])
def test_msd_path_distributions(ak, ex, dev, kind, desc):
    # n >= 2^24: the unstable MSD partition passes (msd_pass.cu) before the local stage,
    # both directions, skewed inputs (exact-largest-bucket range sizing, oversized ranges)
    n = (1 << 24) + 77
    x = dist(np.random.default_rng(24 + len(kind)), n, kind)
    d = torch.from_numpy(x).to(dev)
    ak.merge_sort(d, ex=ex, cmp="greater" if desc else None)
    want = np.sort(x)
    assert np.array_equal(d.cpu().numpy(), want[::-1] if desc else want)


def test_msd_path_uint64_out_of_place(ak, ex, dev):
    n = (1 << 24) + 5
    x = dist(np.random.default_rng(7), n, "uniform", np.uint64)
    d = torch.from_numpy(x.view(np.int64)).to(dev).view(torch.uint64)
    y = ak.merge_sort_copy(d, ex=ex, cmp="greater")
    assert np.array_equal(d.cpu().numpy().view(np.uint64), x)
    assert np.array_equal(y.cpu().numpy().view(np.uint64), np.sort(x)[::-1])


@pytest.mark.parametrize("n", [50_000, 1_000_000, 1 << 20, 2_000_000])
def test_small_sort_graph_replays(ak, ex, dev, n):
    """Small keys-only sorts (n <= 2^20) are replayed as a CUDA graph once the same buffers come
    back: every replay recomputes the plan from the new data (uniform, skewed, narrow, all-equal
    inputs alternate through the same buffers) and equals np.sort. 2e6 keys take the
    device-planned two-level path with the same alternation (plans rejected for skewed data)."""
    rng = np.random.default_rng(n)
    w = torch.empty(n, dtype=torch.int64, device=dev)
    s = torch.empty_like(w)
    kinds = ["uniform", "low40", "uniform", "dups", "cluster", "uniform", "equal", "uniform"]
    for i, kind in enumerate(kinds):
        x = ak.bench_keys(42, i, n, np.int64) if kind == "uniform" else (
            np.full(n, 7, dtype=np.int64) if kind == "equal" else dist(rng, n, kind))
        w.copy_(torch.from_numpy(x))
        ak.merge_sort(w, s, ex)
        assert np.array_equal(w.cpu().numpy(), np.sort(x)), f"call {i} ({kind})"


@pytest.mark.parametrize("n,kind", [((1 << 29) + 12345, "uniform"), ((1 << 29) + 7, "dups"), (1 << 30, "uniform")])
def test_hybrid_big_range_stage(ak, ex, dev, n, kind):
    """n >= 2^29: partitions by the top 8 and 16 bits, then the big-range counting stage
    (local_big_kernel: ranges of up to 18432 keys = aligned groups of 16-bit buckets, two
    per range at 2^29, one at 2^30). Checked by sortedness + order-independent
    multiset fingerprint (a full host sort of 8 GiB is too slow)."""
    g = torch.Generator(device=dev)
    g.manual_seed(n)
    if kind == "uniform":
        x = torch.randint(-(1 << 62), 1 << 62, (n,), dtype=torch.int64, device=dev, generator=g) * 2 + 1
    else:  # 2^20 distinct values spread over the whole range: heavy duplicates in every bucket
        x = torch.randint(0, 1 << 20, (n,), dtype=torch.int64, device=dev, generator=g) * (1 << 43) - (1 << 62)
    fp_in = _fp(x)
    s = torch.empty_like(x)
    ak.merge_sort(x, s, ex)
    assert bool((x[1:] >= x[:-1]).all())
    assert _fp(x) == fp_in


def _fp(t):
    z = t * -7046029254386353131
    z = z ^ ((z >> 29) & ((1 << 35) - 1))
    return int(t.numel()), int(z.sum()), int((z * (2 * t + 1)).sum())


def _top13(rng, n, low):
    """Top 13 bits uniform (16-bit MSD buckets of ~n / 8192 keys: over the 4608-key stage from
    n ~ 2^26 on, so the big-range stage runs well below 2^29), the low 51 bits from `low`."""
    hi = rng.integers(0, 1 << 13, n, dtype=np.int64) << 51
    return hi | low


@pytest.mark.parametrize("kind", ["uniform", "dups", "const", "narrow", "oversized"])
@pytest.mark.parametrize("desc", [False, True])
def test_big_range_stage_skew(ak, ex, dev, kind, desc):
    """local_big_kernel at 2^26 (ranges = aligned pairs of ~8K-key 16-bit buckets) under skew: uniform, dups (bins over 48 keys: the
    segment fallback), const (every 16-bit bucket one value), narrow (60 % of each bucket in
    a 2^30-wide sliver), oversized (one top-13 value holds 40000 keys: a bucket over 18432
    keys, so the plan falls back to a third MSD level and the 4608-key stage)."""
    n = (1 << 26) + 2 * len(kind) + 1
    rng = np.random.default_rng(len(kind) + 100 * desc)
    if kind == "uniform":
        x = _top13(rng, n, rng.integers(0, 1 << 51, n, dtype=np.int64))
    elif kind == "dups":
        x = _top13(rng, n, rng.integers(0, 3, n, dtype=np.int64) << 20)
    elif kind == "const":
        x = _top13(rng, n, np.int64(0))
    elif kind == "narrow":  # 60 % of every bucket within 2^30 of its start
        low = rng.integers(0, 1 << 51, n, dtype=np.int64)
        sel = rng.random(n) < 0.6
        low[sel] = rng.integers(0, 1 << 30, int(sel.sum()), dtype=np.int64)
        x = _top13(rng, n, low)
    else:  # one top-13 value holds 40000 keys
        x = _top13(rng, n, rng.integers(0, 1 << 51, n, dtype=np.int64))
        x[rng.integers(0, n, 40000)] = (np.int64(77) << 51) | rng.integers(0, 1 << 40, 40000, dtype=np.int64)
    d = torch.from_numpy(x).to(dev)
    ak.merge_sort(d, ex=ex, cmp="greater" if desc else None)
    want = np.sort(x)
    assert np.array_equal(d.cpu().numpy(), want[::-1] if desc else want)


@pytest.mark.parametrize("kind", ["uniform", "oversized"])
def test_big_range_stage_bucket_mode(ak, ex, dev, kind):
    """~16K-key 16-bit buckets (n = 2^27, top 13 bits uniform): local_big_kernel with one
    bucket per range (OR-reduced varying bits), uint64 keys; oversized: one bucket holds
    30000 extra keys (over 18432: the segment fallback). Checked on the device."""
    n = 1 << 27
    g = torch.Generator(device=dev)
    g.manual_seed(27 + len(kind))
    x = (torch.randint(0, 1 << 13, (n,), dtype=torch.int64, device=dev, generator=g) << 51) | torch.randint(
        0, 1 << 51, (n,), dtype=torch.int64, device=dev, generator=g)
    if kind == "oversized":
        x[:30000] = (5 << 51) + torch.arange(30000, device=dev) * 977
    fp_in = _fp(x)
    u = x.view(torch.uint64)
    ak.merge_sort(u, ex=ex)
    y = x ^ (-(1 << 63))  # uint64 order as int64 order
    assert bool((y[1:] >= y[:-1]).all())
    assert _fp(x) == fp_in


@pytest.mark.parametrize("n,desc,unsigned", [
    ((1 << 28) + (1 << 23) - 7, False, False),   # just under the big-range threshold: 4608-key stage or host plan
    ((1 << 28) + (1 << 23) + 9, True, False),    # just over: big-range stage, descending
    ((1 << 29) + 3, True, True),                 # 2^29 uint64 descending: pairs of buckets per range
])
def test_plan_boundaries(ak, ex, dev, n, desc, unsigned):
    """Sizes at the device plan's stage boundaries, both directions, signed and unsigned keys;
    checked on the device (order + multiset fingerprint)."""
    g = torch.Generator(device=dev)
    g.manual_seed(n)
    x = torch.randint(-(1 << 62), 1 << 62, (n,), dtype=torch.int64, device=dev, generator=g) * 2 + 1
    fp_in = _fp(x)
    s = torch.empty_like(x)
    if unsigned:
        ak.merge_sort(x.view(torch.uint64), s.view(torch.uint64), ex, cmp="greater" if desc else None)
        y = x ^ (-(1 << 63))
    else:
        ak.merge_sort(x, s, ex, cmp="greater" if desc else None)
        y = x
    del s
    ok = bool((y[1:] <= y[:-1]).all()) if desc else bool((y[1:] >= y[:-1]).all())
    assert ok
    assert _fp(x) == fp_in
