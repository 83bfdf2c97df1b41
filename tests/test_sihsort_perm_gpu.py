"""GPU tests of the distributed sortperm (sihsort_perm: SIHSort of (key, global index) pairs).

The reference's sihsort is keys-only (sihsort.hpp:472-501); this extension (SURVEY §8(f)
rank 4) is checked against its definition: the ranks' outputs concatenated must be the
globally STABLE sort of all ranks' keys (numpy's stable argsort of the concatenated input)
and the permutation itself; every rank must receive exactly the slice the keys-only sihsort
gives it (same splitters: the protocol runs on the keys), and the stats must equal the
keys-only stats except for the index bytes added to redistribution_bytes.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def inputs(kind, P, n, dt, seed):
    rng = np.random.default_rng(seed)
    dt = np.dtype(dt)
    out = []
    for r in range(P):
        m = n if kind != "ragged" else (0 if r == 1 else n + 37 * r)
        if kind == "dups":
            out.append(rng.integers(0, 50, m).astype(dt))
        elif kind == "equal":
            out.append(np.full(m, 7, dtype=dt))
        elif dt.kind == "f":
            x = rng.uniform(-1e6, 1e6, m).astype(dt)
            x[rng.integers(0, max(m, 1), m // 50)] = 0.0
            x[rng.integers(0, max(m, 1), m // 50)] = -0.0  # equal to +0.0: ties by global index
            out.append(x)
        else:
            info = np.iinfo(dt)
            out.append(rng.integers(info.min, info.max, m, dtype=dt, endpoint=True))
    return out


def check(ak, dev, ins, cfg=None):
    P = len(ins)
    keys, idx, stats = ak.sihsort_perm_loopback([torch.from_numpy(a).to(dev) for a in ins], cfg)
    ref_outs, ref_stats = ak.sihsort_loopback([torch.from_numpy(a).to(dev) for a in ins], cfg)
    allk = np.concatenate(ins)
    perm = np.argsort(allk, kind="stable")
    got_idx = np.concatenate([t.cpu().numpy() for t in idx])
    got_keys = np.concatenate([t.cpu().numpy() for t in keys])
    assert np.array_equal(got_idx, perm), "global permutation"
    assert np.array_equal(got_keys.view(np.uint8), allk[perm].view(np.uint8)), "sorted keys (bit-exact)"
    isz = 8
    for r in range(P):
        assert keys[r].numel() == ref_outs[r].numel(), f"rank {r} slice size"
        assert np.array_equal(keys[r].cpu().numpy(), ref_outs[r].cpu().numpy()), f"rank {r} keys"
        a, b = stats[r].as_dict(), ref_stats[r].as_dict()
        extra = a.pop("redistribution_bytes") - b.pop("redistribution_bytes")
        assert a == b, f"rank {r} stats"
        assert extra % isz == 0 and extra >= 0
    return keys, idx, stats


@pytest.mark.parametrize("P", [1, 2, 3, 4])
@pytest.mark.parametrize("dt", [np.float32, np.int64])
def test_perm_uniform(ak, dev, P, dt):
    check(ak, dev, inputs("uniform", P, 20_000, dt, P))


@pytest.mark.parametrize("kind", ["dups", "equal", "ragged"])
@pytest.mark.parametrize("dt", [np.int32, np.uint64, np.float64])
def test_perm_ties_and_ragged(ak, dev, kind, dt):
    check(ak, dev, inputs(kind, 3, 5_000, dt, 11))


def test_perm_large_p8(ak, dev):
    # 8 ranks x 2^20 float32 keys with heavy ties: the by-key radix sorts run their full
    # multi-pass paths and the second local sort merges 8 runs
    check(ak, dev, inputs("dups", 8, 1 << 20, np.float32, 3))


def test_perm_index_bytes_accounting(ak, dev):
    ins = inputs("uniform", 4, 10_000, np.int64, 5)
    keys, idx, stats = ak.sihsort_perm_loopback([torch.from_numpy(a).to(dev) for a in ins])
    _, ref_stats = ak.sihsort_loopback([torch.from_numpy(a).to(dev) for a in ins])
    offs = np.cumsum([0] + [a.size for a in ins])
    for r in range(4):
        assert stats[r].redistribution_bytes >= ref_stats[r].redistribution_bytes
    # every index a rank received from another rank (global index outside the receiver's own
    # range) was sent once: the added bytes are 8 per such index
    total_extra = sum(stats[r].redistribution_bytes - ref_stats[r].redistribution_bytes for r in range(4))
    total_foreign = sum(int(((idx[r].cpu().numpy() < offs[r]) | (idx[r].cpu().numpy() >= offs[r + 1])).sum())
                        for r in range(4))
    assert total_extra == 8 * total_foreign


def test_perm_single_rank_api(ak, ex, dev):
    x = inputs("dups", 1, 100_001, np.float32, 9)[0]
    k, i, st = ak.sihsort_perm(torch.from_numpy(x).to(dev), ex=ex)
    perm = np.argsort(x, kind="stable")
    assert np.array_equal(i.cpu().numpy(), perm)
    assert np.array_equal(k.cpu().numpy(), x[perm])
    assert st.converged == 1
