"""Multi-process SIHSort on real communicators (one process per rank), compared per rank with
the reference itself (oracle/_ref: sihsort over sim::world, sihsort.hpp:508-569).

* IpcComm (peer-store exchange through CUDA IPC mappings, control over gloo) runs with 2-3
  processes on ONE GPU: the exchange kernel only stores into the peers' receive buffers and
  every wait is a host barrier, so no kernel waits on another process. On a multi-GPU box the
  same code maps peer HBM over NVLink.
* NcclComm needs one GPU per rank (NCCL refuses two ranks on one device): skipped below P GPUs.
* torchrun bench.py at N = 2 likewise needs 2 GPUs.
"""
import json
import os
import socket
import subprocess
import sys
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def gpu_count():
    import torch
    return torch.cuda.device_count()


def worker(rank, world, port, transport, n, dtype, outdir, same_gpu, op="sort"):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import oracle
    import paper_2507_16710_b200 as ak

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = 0 if same_gpu else rank
    torch.cuda.set_device(dev)
    ex = ak.ExecBackend(dev)
    if transport == "ipc":
        comm = ak.IpcComm(dev)
    else:
        obj = [ak.NcclComm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = ak.NcclComm(obj[0], world, rank, dev)
    dt = np.dtype(dtype)
    x = oracle.ref_bench_keys(42, rank, n + 17 * rank, dt)  # ragged sizes
    d = torch.from_numpy(x.view(np.int64) if dt == np.uint64 else x).to(f"cuda:{dev}")
    if dt == np.uint64:
        d = d.view(torch.uint64)
    if op == "perm":  # distributed sortperm: keys + global indices over the same transport
        k, i, st = ak.sihsort_perm(d, comm, None, ex)
        np.savez(os.path.join(outdir, f"r{rank}.npz"), keys=k.cpu().numpy(), idx=i.cpu().numpy())
        comm.close()
        dist.barrier()
        dist.destroy_process_group()
        return
    outs = []
    for _ in range(2):  # twice: the second call reuses the cached peer mappings
        out, st = ak.sihsort(d, comm, None, ex)
        outs.append(out.cpu().numpy().copy())
    np.savez(os.path.join(outdir, f"r{rank}.npz"), out=outs[-1], first=outs[0],
             stats=np.array([getattr(st, f) for f, _ in ak.SihStats._fields_], dtype=np.float64),
             sent=np.array([comm.bytes_sent()], dtype=np.uint64))
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


def run_world(transport, world, n, dtype, same_gpu, op="sort"):
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(worker, args=(world, free_port(), transport, n, dtype, d, same_gpu, op), nprocs=world,
                           join=True, start_method="spawn")
        return [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(world)]


def check_vs_reference(orc, res, world, n, dtype):
    dt = np.dtype(dtype)
    ins = [orc.ref_bench_keys(42, r, n + 17 * r, dt) for r in range(world)]
    want, wstats = orc.ref_sihsort(ins, threads_per_rank=max(1, (os.cpu_count() or 1) // world))
    names = [f for f, _ in orc.SihStats._fields_]
    for r in range(world):
        got = res[r]["out"].view(dt)
        assert np.array_equal(got, want[r]), f"rank {r} output"
        assert np.array_equal(res[r]["first"].view(dt), want[r]), f"rank {r} first call"
        st = dict(zip(names, res[r]["stats"].tolist()))
        for k in names:
            assert st[k] == pytest.approx(wstats[r][k]), f"rank {r} stat {k}"
    sent = sum(int(r_["sent"][0]) for r_ in res)
    assert sent > 0 or world == 1


@pytest.mark.parametrize("world,n,dtype", [(2, 1 << 20, np.int64), (3, 300_000, np.uint64), (2, 1 << 22, np.uint64)])
def test_ipc_exchange_processes_on_one_gpu(orc, world, n, dtype):
    if not orc.ref_available():
        pytest.skip("oracle/_ref not built")
    res = run_world("ipc", world, n, dtype, same_gpu=True)
    check_vs_reference(orc, res, world, n, dtype)


def test_ipc_distributed_sortperm_processes_on_one_gpu(orc):
    """sihsort_perm over IpcComm with 3 processes: keys AND global indices travel through the
    peer-store exchange; the concatenated outputs are the stable global order."""
    world, n = 3, 200_000
    res = run_world("ipc", world, n, np.int64, same_gpu=True, op="perm")
    ins = [orc.ref_bench_keys(42, r, n + 17 * r, np.dtype(np.int64)) for r in range(world)]
    allk = np.concatenate(ins)
    perm = np.argsort(allk, kind="stable")
    assert np.array_equal(np.concatenate([res[r]["idx"] for r in range(world)]), perm)
    assert np.array_equal(np.concatenate([res[r]["keys"] for r in range(world)]), allk[perm])


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("transport", ["nccl", "ipc"])
def test_one_process_per_gpu(orc, transport, world):
    if gpu_count() < world:
        pytest.skip(f"needs {world} GPUs")
    if not orc.ref_available():
        pytest.skip("oracle/_ref not built")
    res = run_world(transport, world, 1 << 22, np.int64, same_gpu=False)
    check_vs_reference(orc, res, world, 1 << 22, np.int64)


def test_two_devices_in_one_process(ak, orc):
    """Kernel attributes are per device: sorting on device 0 and then on device 1 in one
    process (and from two threads at once) must work (large dynamic shared memory kernels)."""
    if gpu_count() < 2:
        pytest.skip("needs 2 GPUs")
    import threading

    import torch
    x = ak.bench_keys(42, 0, 1 << 24, np.int64)
    want = np.sort(x)
    for d in (0, 1):
        t = torch.from_numpy(x).to(f"cuda:{d}")
        ak.merge_sort(t, ex=ak.ExecBackend(d))
        assert np.array_equal(t.cpu().numpy(), want)
    errs = []

    def job(d):
        try:
            t = torch.from_numpy(x).to(f"cuda:{d}")
            ak.merge_sort(t, ex=ak.ExecBackend(d))
            assert np.array_equal(t.cpu().numpy(), want)
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=job, args=(d,)) for d in (0, 1)]
    [t.start() for t in th]
    [t.join() for t in th]
    assert not errs


@pytest.mark.parametrize("nproc", [2, 3])
def test_torchrun_bench_ranks_sharing_one_gpu(nproc):
    """bench.py's N > 1 path (torchrun, max-over-ranks timing, cross-rank checks, the nvlink
    and e2e objects) with every rank on GPU 0 over the IPC transport (AKB_BENCH_SHARE_GPU=1):
    what the driver's multi-GPU runs execute, runnable on a one-GPU box."""
    env = dict(os.environ, AKB_BENCH_SHARE_GPU="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(nproc),
                        "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.join(ROOT, "bench.py"),
                        "--gpus", str(nproc), "--steps", "2", "--warmup", "3", "--log2n", "22"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == nproc and line["config"]["global_keys"] == nproc << 22
    assert line["config"]["sorted_check"] and line["config"]["multiset_fingerprint_check"]
    assert line["nvlink"]["bytes_sent_per_gpu"] > 0 and line["e2e"]["output_copy_check"]
    assert "test_mode" in line["config"]


@pytest.mark.parametrize("transport", ["nccl", "ipc"])
def test_torchrun_bench_two_gpus(transport):
    if gpu_count() < 2:
        pytest.skip("needs 2 GPUs")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--steps", "2", "--warmup", "3", "--log2n", "24", "--no-e2e",
                        "--transport", transport], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["sorted_check"] and line["config"]["multiset_fingerprint_check"]
    assert line["nvlink"]["bytes_sent_per_gpu"] > 0
