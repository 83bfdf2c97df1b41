"""GPU parity: any_pred / all_pred (predicates.hpp:16-78, test_primitives.cpp:206-263) and the
multi-rank reduce / scan over a communicator on P logical ranks of
the single-GPU loopback world, one host thread per rank.
"""
import threading

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("algo", ["early_exit", "via_mapreduce"])
def test_predicates_trivial_and_empty(ak, ex, dev, algo):
    z = torch.zeros(100, dtype=torch.int32, device=dev)
    o = torch.ones(100, dtype=torch.int32, device=dev)
    e = torch.zeros(0, dtype=torch.int32, device=dev)
    assert not ak.any_pred(z, ">", 0, ex, algo)
    assert ak.all_pred(o, "==", 1, ex, algo)
    assert not ak.any_pred(e, ">", 0, ex, algo)
    assert ak.all_pred(e, ">", 0, ex, algo)


def test_predicates_sparse_bytes(ak, ex, dev):
    rng = np.random.default_rng(14)
    for n in (1, 15, 100_000, 3_000_001):
        b = (rng.integers(0, 4096, n) == 0).astype(np.uint8)
        d = torch.from_numpy(b).to(dev)
        assert ak.any_pred(d, "!=", 0, ex) == bool(b.any())
        assert ak.all_pred(d, "==", 0, ex) == (not b.any())
    one = torch.zeros(1 << 22, dtype=torch.uint8, device=dev)
    one[-1] = 1  # the only true element is the very last one (tail of the vector loop)
    assert ak.any_pred(one, "==", 1, ex) and ak.any_pred(one[1:], "==", 1, ex)  # misaligned view too


@pytest.mark.parametrize("dt", [np.int8, np.int16, np.int32, np.uint32, np.int64, np.uint64, np.float32, np.float64])
def test_predicates_match_numpy_and_duality(ak, ex, dev, dt):
    rng = np.random.default_rng(15)
    for inst in range(40):
        n = int(rng.integers(0, 5000))
        x = rng.integers(0, 100, n).astype(dt)
        cut = dt(rng.integers(0, 100))
        d = torch.from_numpy(x).to(dev)
        for op, f in (("<", np.less), ("<=", np.less_equal), (">", np.greater), (">=", np.greater_equal),
                      ("==", np.equal), ("!=", np.not_equal)):
            want = f(x, cut)
            assert ak.any_pred(d, op, cut, ex) == bool(want.any())
            assert ak.all_pred(d, op, cut, ex, "via_mapreduce") == bool(want.all())
        assert ak.all_pred(d, "<", cut, ex) == (not ak.any_pred(d, ">=", cut, ex))


def run_ranks(P, body):
    world = ak_mod().LoopbackWorld(P)
    comms = [world.comm(r) for r in range(P)]
    exs = [ak_mod().ExecBackend(0) for _ in range(P)]
    out, err = [None] * P, []

    def go(r):
        try:
            out[r] = body(r, comms[r], exs[r])
        except Exception as e:  # noqa: BLE001
            err.append(e)
            world.abort()

    th = [threading.Thread(target=go, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    torch.cuda.synchronize()
    return out


def ak_mod():
    import paper_2507_16710_b200 as ak
    return ak


@pytest.mark.parametrize("P", [1, 3, 4])
@pytest.mark.parametrize("dt", [torch.int64, torch.int32, torch.float64])
def test_reduce_all_and_accumulate_all(ak, dev, P, dt):
    g = torch.Generator(device="cpu").manual_seed(P)
    parts = [torch.randint(-10000, 10001, (int(n),), generator=g).to(dt).to(dev)
             for n in torch.randint(0, 20000, (P,), generator=g)]
    cat = torch.cat(parts)
    res = run_ranks(P, lambda r, comm, e: (ak.reduce_all("sum", parts[r], comm, ex=e),
                                           ak.reduce_all("max", parts[r], comm, ex=e),
                                           ak.accumulate_all("sum", parts[r], comm, ex=e),
                                           ak.accumulate_all("sum", parts[r], comm, inclusive=False, init=5, ex=e)))
    want_sum = cat.double().sum().item()
    want_inc = torch.cumsum(cat.double(), 0)
    want_exc = torch.cat([torch.zeros(1, dtype=torch.float64, device=dev), want_inc[:-1]]) + 5
    for r in range(P):
        assert res[r][0] == want_sum
        if cat.numel():
            assert res[r][1] == cat.max().item()
    got_inc = torch.cat([res[r][2] for r in range(P)]).double()
    got_exc = torch.cat([res[r][3] for r in range(P)]).double()
    assert torch.equal(got_inc, want_inc) and torch.equal(got_exc, want_exc)
