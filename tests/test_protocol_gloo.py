"""CPU, world_size 2 over torch.distributed gloo: the multi-rank SIHSort host protocol.

The product protocol (paper_2507_16710_b200/csrc/sih_protocol.hpp -- config check,
global summaries, distributed histogram, splitter selection and refinement,
P x P count exchange, capacity agreement, redistribution bookkeeping) is compiled
with a host rank policy (tests/cpp/proto_host.cpp, test-only) and driven through
the callback transport by two real processes whose collectives are gloo
all_gather / all_reduce / isend+irecv. Outputs and sih_stats must equal the
oracle's (== the reference sihsort, tests/test_oracle.py) exactly.
"""
import ctypes as C
import os
import socket
import subprocess
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "proto_host.cpp")
INC = os.path.join(ROOT, "paper_2507_16710_b200", "csrc")
LIB = os.path.join(ROOT, "build", "libproto_host.so")

AG = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p)
AR = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64)
EX = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                 C.c_uint64)


class Cfg(C.Structure):
    _fields_ = [("sample_per_rank", C.c_uint64), ("bins", C.c_uint64), ("max_refine_rounds", C.c_uint64),
                ("imbalance_tol", C.c_double)]


class Stats(C.Structure):
    _fields_ = [("rounds_used", C.c_uint64), ("converged", C.c_uint64), ("max_deviation", C.c_double),
                ("redistribution_sends", C.c_uint64), ("redistribution_bytes", C.c_uint64),
                ("collective_ops", C.c_uint64), ("output_count", C.c_uint64)]


def bind(lib):
    fn = lib.proto_sihsort_i64
    fn.restype = C.c_int
    fn.argtypes = [C.c_int, C.c_int, C.c_void_p, AG, AR, EX, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64,
                   C.POINTER(C.c_uint64), C.POINTER(Cfg), C.POINTER(Stats)]
    lib.proto_last_error.restype = C.c_char_p
    return fn


def build_lib():
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(SRC), os.path.getmtime(
            os.path.join(INC, "sih_protocol.hpp"))):
        subprocess.run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-I", INC, SRC, "-o", LIB], check=True)
    return LIB


def inputs(case, world):
    rng = np.random.default_rng(7)
    n = 4000
    if case == "uniform":
        return [rng.integers(-2**63, 2**63 - 1, n, dtype=np.int64) for _ in range(world)]
    if case == "zipf":
        return [np.minimum(rng.zipf(1.1, n), 10**6).astype(np.int64) for _ in range(world)]
    if case == "equal":
        return [np.full(n, 3, dtype=np.int64) for _ in range(world)]
    if case == "ragged":
        return [np.empty(0, dtype=np.int64)] + [rng.integers(-50, 50, 777).astype(np.int64)
                                                for _ in range(world - 1)]
    raise ValueError(case)


def worker(rank, world, port, case, cfg_rows, outdir):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = C.CDLL(LIB)

    def ag(user, inp, nbytes, out):
        buf = torch.from_numpy(np.frombuffer((C.c_char * nbytes).from_address(inp), dtype=np.uint8).copy())
        outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(outs, buf)
        cat = torch.cat(outs).numpy()
        C.memmove(out, cat.ctypes.data, nbytes * world)
        return 0

    def ar(user, ptr, n):
        arr = np.frombuffer((C.c_char * (8 * n)).from_address(ptr), dtype=np.int64).copy()
        t = torch.from_numpy(arr)
        dist.all_reduce(t)
        C.memmove(ptr, t.numpy().ctypes.data, 8 * n)
        return 0

    def ex(user, sb, so, sc, rb, ro, rc, eb):
        so_ = np.ctypeslib.as_array((C.c_uint64 * world).from_address(so))
        sc_ = np.ctypeslib.as_array((C.c_uint64 * world).from_address(sc))
        ro_ = np.ctypeslib.as_array((C.c_uint64 * world).from_address(ro))
        rc_ = np.ctypeslib.as_array((C.c_uint64 * world).from_address(rc))
        reqs, bufs = [], []
        for q in range(world):
            if q == rank:
                continue
            if sc_[q]:
                nb = int(sc_[q]) * eb
                src = np.frombuffer((C.c_char * nb).from_address(sb + int(so_[q]) * eb), dtype=np.uint8).copy()
                reqs.append(dist.isend(torch.from_numpy(src), q))
            if rc_[q]:
                r = torch.empty(int(rc_[q]) * eb, dtype=torch.uint8)
                bufs.append((q, r))
                reqs.append(dist.irecv(r, q))
        for r in reqs:
            r.wait()
        for q, r in bufs:
            C.memmove(rb + int(ro_[q]) * eb, r.numpy().ctypes.data, r.numel())
        return 0

    cb = (AG(ag), AR(ar), EX(ex))
    fn = bind(lib)
    x = inputs(case, world)[rank]
    cap = sum(a.size for a in inputs(case, world)) + 16 if case != "capacity" else 10
    out = np.empty(max(cap, 1), dtype=np.int64)
    oc = C.c_uint64(0)
    st = Stats()
    cfg = Cfg(*cfg_rows[rank])
    rc = fn(rank, world, None, cb[0], cb[1], cb[2], C.c_void_p(x.ctypes.data), x.size,
            C.c_void_p(out.ctypes.data), out.size, C.byref(oc), C.byref(cfg), C.byref(st))
    lib.proto_last_error.restype = C.c_char_p
    if rc not in (0, 2, 6):
        print("proto error:", lib.proto_last_error(), flush=True)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), rc=rc, out=out[: oc.value] if rc == 0 else out[:0],
             stats=np.array([getattr(st, f) for f, _ in Stats._fields_], dtype=np.float64))
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_world(case, cfg_rows, world=2):
    import torch.multiprocessing as mp

    build_lib()
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(worker, args=(world, free_port(), case, cfg_rows, d), nprocs=world, join=True,
                           start_method="spawn")
        return [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(world)]


DEFAULT = (0, 0, 4, 0.25)


@pytest.mark.parametrize("case", ["uniform", "zipf", "equal", "ragged"])
def test_protocol_two_ranks_matches_oracle(orc, case):
    res = run_world(case, [DEFAULT, DEFAULT])
    want, wstats, _ = orc.sihsort(inputs(case, 2))
    for r in range(2):
        assert int(res[r]["rc"]) == 0
        assert np.array_equal(res[r]["out"], want[r])
        s = wstats[r]
        row = [s["rounds_used"], s["converged"], s["max_deviation"], s["redistribution_sends"],
               s["redistribution_bytes"], s["collective_ops"], s["output_count"]]
        assert np.array_equal(res[r]["stats"], np.array(row, dtype=np.float64))


def test_protocol_config_mismatch_is_protocol_error():
    # sihsort.hpp:240-256: every rank throws protocol_error
    res = run_world("uniform", [DEFAULT, (0, 0, 3, 0.25)])
    assert [int(r["rc"]) for r in res] == [2, 2]


def test_protocol_capacity_agreement():
    # all ranks detect an undersized output together (no rank hangs in the exchange)
    res = run_world_capacity()
    assert [int(r["rc"]) for r in res] == [6, 6]


def run_world_capacity():
    import torch.multiprocessing as mp

    build_lib()
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(capacity_worker, args=(2, free_port(), d), nprocs=2, join=True, start_method="spawn")
        return [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(2)]


def capacity_worker(rank, world, port, outdir):
    # all-equal keys route everything to rank 0 whose capacity (n) is too small
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    lib = C.CDLL(LIB)

    def ag(user, inp, nbytes, out):
        buf = torch.from_numpy(np.frombuffer((C.c_char * nbytes).from_address(inp), dtype=np.uint8).copy())
        outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(outs, buf)
        cat = torch.cat(outs).numpy()  # keep alive across the memmove
        C.memmove(out, cat.ctypes.data, nbytes * world)
        return 0

    def ar(user, ptr, n):
        t = torch.from_numpy(np.frombuffer((C.c_char * (8 * n)).from_address(ptr), dtype=np.int64).copy())
        dist.all_reduce(t)
        C.memmove(ptr, t.numpy().ctypes.data, 8 * n)
        return 0

    def ex(*a):
        return 1  # must never be reached

    cb = (AG(ag), AR(ar), EX(ex))
    x = np.full(1000, 4, dtype=np.int64)
    out = np.empty(1000, dtype=np.int64)
    oc = C.c_uint64(0)
    st = Stats()
    cfg = Cfg(*DEFAULT)
    rc = bind(lib)(rank, world, None, cb[0], cb[1], cb[2], C.c_void_p(x.ctypes.data), x.size,
                               C.c_void_p(out.ctypes.data), out.size, C.byref(oc), C.byref(cfg), C.byref(st))
    np.savez(os.path.join(outdir, f"r{rank}.npz"), rc=rc, required=oc.value)
    dist.destroy_process_group()
