#!/usr/bin/env python
"""bench.py -- headline benchmark: distributed sample sort (SIHSort) of Int64 keys.

Metric (BASELINE.json): sort throughput GB/s of Int64 keys = total key bytes
sorted across all ranks / 1e9 / seconds per step (reference bench.cpp:74-76, :213).
Workload (BASELINE config 4): 2^28 uniform-random full-range Int64 keys per GPU from
the reference bench generator (mt19937_64(seed + 0x9e3779b97f4a7c15*(r+1)),
bench.cpp:164-173), weak scaling, one rank per GPU, NCCL between GPUs.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

A step = one full ak.sihsort (local radix sort, sampling, splitters, refinement,
NCCL all-to-all-v, P-way merge) of device-resident input into a device output.
`e2e` = the same with every step's input copied host->device from pinned memory and
its output copied back (steps pipelined over two buffer sets: step i+1's upload is
enqueued before step i's sort and overlaps it and step i-1's download on the full-duplex
PCIe link); `e2e.blocking` = one
blocking host-buffer C-ABI call per step (ak_sihsort_host_*: H2D + sort + D2H).

At N=1 the line also carries `configs`: every other BASELINE.json config measured on
the device (time, roofline fraction) beside the reference's own multithreaded CPU
implementation (oracle/_ref, /root/reference/proj compiled in place) on the same host.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sort throughput GB/s (Int64 keys) at 1/2/4/8 B200; % of HBM/NVLink roofline"
# NVLink denominators (/opt/skills/guides/B200_PROFILING.md): measured peer copy 770 GB/s per
# direction per GPU on this pool's B200s; nominal NVLink 5 = 900 GB/s per direction.
NVLINK_MEASURED_GBS = 770.0
NVLINK_NOMINAL_GBS = 900.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--log2n", type=int, default=28, help="keys per GPU = 2^log2n (config 4: 28, config 5: 30)")
    p.add_argument("--dtype", choices=["int64", "uint64"], default="int64")
    p.add_argument("--seed", type=int, default=42)
    p.add_argument("--transport", choices=["nccl", "ipc"], default="nccl",
                   help="N>1 exchange: NCCL grouped send/recv, or peer memory over CUDA IPC mappings "
                        "(the merge reads the incoming runs straight from the peers)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-configs", action="store_true", help="skip the per-config table (N=1 only)")
    p.add_argument("--configs-cpu", type=int, default=1, help="time the reference CPU path beside each config")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(kernel):
    """DRAM bytes per launch per key of `kernel` from the committed ncu --set full summary
    (profiles/<kernel>_traffic.json), or None."""
    path = os.path.join(ROOT, "profiles", f"{kernel}_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_launch_per_key")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                clk, mx, util = float(parts[0]), float(parts[1]), float(parts[2])
            except ValueError:
                continue
            smax.append(mx)
            if util > 0:
                sm.append(clk)
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(self.lines), "samples_under_load": len(sm)}


# ----------------------------------------------------------------------------- reference arm

def ref_keys_per_rank(log2n: int, world: int) -> int:
    """Keys per rank of the reference arm. N=1: the full 2^log2n workload (same config as
    our arm). N>1: a bounded sample with the same TOTAL keys as N=1 (2^log2n / N per rank),
    so every step stays ~8 s on 16 host cores and the default run ends within minutes."""
    n = 1 << log2n
    return n if world == 1 else n // world


def reference_arm(args, rank, world):
    """The reference's own CPU implementation (oracle/_ref: /root/reference/proj compiled in
    place) over its sim::world with P = N ranks, every host thread in use. The inputs are
    made by the reference-side generator (oracle.ref_bench_keys), so this process never
    loads the product library."""
    if rank != 0:
        return
    import numpy as np
    import oracle

    cores = os.cpu_count() or 1
    P = world
    n_rank = ref_keys_per_rank(args.log2n, P)
    dt = np.int64 if args.dtype == "int64" else np.uint64
    kind = "reference" if oracle.ref_available() else "port"
    if kind == "reference":
        ins = [oracle.ref_bench_keys(args.seed, r, n_rank, dt) for r in range(P)]
    else:  # no reference build on this box: the C restatement (numpy inputs, same seeds)
        ins = [np.random.default_rng(args.seed + r).integers(np.iinfo(dt).min, np.iinfo(dt).max, n_rank,
                                                             dtype=dt, endpoint=True) for r in range(P)]
    tpr = max(1, cores // P)

    def step():
        if kind == "reference":
            oracle.ref_sihsort(ins, threads_per_rank=tpr)
        else:
            oracle.sihsort(ins)

    for _ in range(args.warmup):
        step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    ms = 1e3 * statistics.mean(times)
    gbs = P * n_rank * 8 / 1e9 / (ms / 1e3)
    same = n_rank == (1 << args.log2n)
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": f"reference sihsort (sim::world, {P} ranks, exec_backend::threaded({tpr}) per rank) "
                               f"of {args.dtype.capitalize()} keys; {n_rank} keys/rank"
                               + ("" if same else f" (bounded sample of the 2^{args.log2n}/GPU workload: "
                                                  f"same total keys as N=1)"),
                   "keys_per_rank": n_rank, "ranks": P, "threads_per_rank": tpr, "same_config": same,
                   "generator": "reference bench.cpp mt19937_64 per-rank seeds (oracle/_ref ref_bench_keys)",
                   "stddev_ms": statistics.stdev(times) if len(times) > 1 else 0.0},
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": tpr * P if kind == "reference" else 1,
                         "kind": kind, "sample": f"{P} ranks x {n_rank} keys (bench generator, seed {args.seed})"},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(args):
    """Reference CPU path (oracle/_ref, all host threads) on the headline workload: sihsort P=1
    of the same 2^log2n bench keys, rank 0 / N=1 only."""
    import numpy as np
    import oracle

    cores = os.cpu_count() or 1
    n = 1 << args.log2n
    dt = np.int64 if args.dtype == "int64" else np.uint64
    kind = "reference" if oracle.ref_available() else "port"
    x = oracle.ref_bench_keys(args.seed, 0, n, dt) if kind == "reference" else None
    if x is None:
        x = np.random.default_rng(args.seed).integers(np.iinfo(dt).min, np.iinfo(dt).max, n, dtype=dt, endpoint=True)
    run = (lambda: oracle.ref_sihsort([x], threads_per_rank=cores)) if kind == "reference" else \
        (lambda: oracle.sihsort([x]))
    run()
    t = []
    for _ in range(2):
        t0 = time.perf_counter()
        run()
        t.append(time.perf_counter() - t0)
    ms = 1e3 * statistics.mean(t)
    return {"value": n * 8 / 1e9 / (ms / 1e3), "unit": "GB/s", "cores": cores if kind == "reference" else 1,
            "kind": kind, "sample": f"sihsort P=1 of {n} bench keys (2^{args.log2n}, the full workload), mean of 2 "
                                    f"after 1 warm-up, {ms:.1f} ms/sort"}


# ----------------------------------------------------------------------------- helpers (our arm)

def fingerprint(t):
    """Order-independent multiset fingerprint of 64-bit keys on the device: (count, wrapping sum
    of splitmix64(key), wrapping sum of splitmix64(key) * (2 * key + 1))."""
    import torch

    def s64(v):  # python int -> the same 64-bit pattern as a signed int64 constant
        return v - (1 << 64) if v >= (1 << 63) else v

    x = t.view(torch.int64)
    z = x + s64(0x9E3779B97F4A7C15)
    z = (z ^ ((z >> 30) & ((1 << 34) - 1))) * s64(0xBF58476D1CE4E5B9)
    z = (z ^ ((z >> 27) & ((1 << 37) - 1))) * s64(0x94D049BB133111EB)
    z = z ^ ((z >> 31) & ((1 << 33) - 1))
    return (x.numel(), int(z.sum().item()), int((z * (2 * x + 1)).sum().item()))  # wrapping int64 sums


def is_sorted(t, unsigned: bool) -> bool:
    import torch
    if t.numel() < 2:
        return True
    o = t.view(torch.int64)
    if unsigned:
        o = o ^ (-(1 << 63))
    return bool((o[1:] >= o[:-1]).all())


def timed_device(stream, fn, reps, warm=1):
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.mean(ts)


def timed_host(fn, reps=1, warm=0):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(1e3 * (time.perf_counter() - t0))
    return statistics.mean(ts)


def run_configs(args, ex, dev, peak):
    """Every single-GPU BASELINE.json config: device time + HBM roofline fraction (SURVEY.md §8(d)
    algorithmic bytes), and the reference's multithreaded CPU implementation on this host's
    cores (oracle/_ref; one timed call after no warm-up: seconds per call) with an output
    check against it."""
    import numpy as np
    import torch

    import paper_2507_16710_b200 as ak
    try:
        import oracle
        ref = oracle.ref_available() and args.configs_cpu
    except Exception:  # the CPU leg is a reported baseline, never the product
        oracle, ref = None, False
    cores = os.cpu_count() or 1
    out = {"cpu_cores": cores, "cpu_kind": "reference" if ref else None,
           "note": "device ms = CUDA events on the ctx stream, inputs resident in HBM, mean of 5 after 1 warm-up; "
                   "cpu_ms = reference (oracle/_ref) exec_backend::threaded(cores), one call on host arrays"}

    def frac(alg_bytes, ms):
        ach = alg_bytes / (ms / 1e3) / 1e9
        return {"alg_bytes": alg_bytes, "achieved_gbs": ach, "frac": ach / peak}

    # ---- config 1: merge_sort of 1e6 uniform Int64 (in place; timed with the input copy) ----
    n = 1_000_000
    h = ak.bench_keys(args.seed, 0, n, np.int64)
    x = torch.from_numpy(h).to(dev)
    w, s = torch.empty_like(x), torch.empty_like(x)
    ms = timed_device(ex.stream, lambda: (w.copy_(x), ak.merge_sort(w, s, ex)), 20)
    dev_sorted = w.cpu().numpy()
    cp = timed_device(ex.stream, lambda: s.copy_(x), 20)
    ts = []  # the sort alone: a fresh unsorted copy before each timed call, outside the events
    for r in range(23):
        w.copy_(x)
        torch.cuda.synchronize()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(ex.stream)
        ak.merge_sort(w, s, ex)
        z.record(ex.stream)
        z.synchronize()
        if r >= 3:
            ts.append(a.elapsed_time(z))
    sort_ms = statistics.mean(ts)
    hw = h.copy()

    def host_sort():
        hw[:] = h
        ak.merge_sort_host(hw, ex)

    e2e = timed_host(host_sort, 20, 2)
    c1 = {"workload": "merge_sort 1e6 uniform Int64 (bench keys)", "device_ms": sort_ms,
          "device_ms_note": "one blocking public-API call (ak.merge_sort) on device buffers, CUDA events around it",
          "device_ms_incl_copy": ms, "copy_ms": cp,
          "e2e_ms": e2e, "e2e_note": "ak.merge_sort_host: H2D + sort + D2H in one blocking call",
          "roofline": dict(frac(16 * n, sort_ms), note="L2-resident (8 MB): launch/latency-bound; 16 B/key = read+write")}
    if ref:
        keep = {}
        c1["cpu_ms"] = timed_host(lambda: keep.__setitem__("r", oracle.ref_merge_sort(h, threads=cores)), 3, 1)
        c1["bit_exact_vs_reference"] = bool(np.array_equal(dev_sorted, keep["r"]))
        c1["bit_exact_e2e_vs_reference"] = bool(np.array_equal(hw, keep["r"]))
    out["1_merge_sort_1e6_i64"] = c1
    del x, w, s

    # ---- config 2: sortperm / merge_sort_by_key of 1e8 Float32 (+ Int32 payload) ----
    n = 100_000_000
    hf = ak.bench_keys(args.seed, 0, n, np.float32)
    f = torch.from_numpy(hf).to(dev)
    perm = torch.empty(n, dtype=torch.int32, device=dev)
    bufs = ak.SortpermBuffers.with_capacity(n, torch.float32, torch.int32)
    ms = timed_device(ex.stream, lambda: ak.sortperm(f, out=perm, buffers=bufs, ex=ex), 5)
    c2 = {"workload": "sortperm 1e8 uniform(-1e6,1e6) Float32 -> Int32 (bench keys)", "device_ms": ms,
          "roofline": frac(64 * n, ms)}
    k = torch.empty_like(f)
    v = torch.empty(n, dtype=torch.int32, device=dev)
    iota = torch.arange(n, dtype=torch.int32, device=dev)
    kb = ak.SortByKeyBuffers.with_capacity(n, torch.float32, torch.int32)
    ms2 = timed_device(ex.stream, lambda: (k.copy_(f), v.copy_(iota), ak.merge_sort_by_key(k, v, buffers=kb, ex=ex)), 5)
    kv_dev = (k.cpu().numpy(), v.cpu().numpy())
    cp2 = timed_device(ex.stream, lambda: (kb.scratch_keys.copy_(f), kb.scratch_payload.copy_(iota)), 5)
    c2b = {"workload": "merge_sort_by_key 1e8 Float32 keys + Int32 iota payload", "device_ms_incl_copy": ms2,
           "copy_ms": cp2, "roofline": frac(68 * n + 16 * n, ms2)}
    if ref:
        res = {}
        c2["cpu_ms"] = timed_host(lambda: res.__setitem__("p", oracle.ref_sortperm(hf, np.int32, threads=cores)))
        c2["bit_exact_vs_reference"] = bool(np.array_equal(perm.cpu().numpy(), res.pop("p")))
        payload = np.arange(n, dtype=np.int32)
        c2b["cpu_ms"] = timed_host(lambda: res.__setitem__("kv", oracle.ref_merge_sort_by_key(hf, payload, threads=cores)))
        c2b["bit_exact_vs_reference"] = bool(np.array_equal(kv_dev[1], res["kv"][1]) and
                                             np.array_equal(kv_dev[0].view(np.uint32), res["kv"][0].view(np.uint32)))
        del payload, res
    out["2_sortperm_1e8_f32_i32"] = c2
    out["2_merge_sort_by_key_1e8_f32_i32"] = c2b
    del f, perm, bufs, k, v, iota, kb, hf

    # ---- config 3: reduce and inclusive accumulate over 2^30 Float32 and Int64 ----
    n = 1 << 30
    rng = np.random.default_rng(args.seed)
    for name, npdt, tdt in (("f32", np.float32, torch.float32), ("i64", np.int64, torch.int64)):
        hx = rng.random(n, dtype=np.float32) if name == "f32" else rng.integers(-10000, 10001, n, dtype=np.int64)
        xx = torch.from_numpy(hx).to(dev)
        eb = xx.element_size()
        res = torch.empty(1, dtype=tdt, device=dev)
        ms_r = timed_device(ex.stream, lambda: ak.reduce_device("sum", xx, res, ex=ex), 5)
        yy = torch.empty_like(xx)
        ms_s = timed_device(ex.stream, lambda: ak.accumulate("sum", xx, out=yy, ex=ex), 5)
        cr = {"workload": f"reduce(+) 2^30 {name}", "device_ms": ms_r, "roofline": frac(eb * n, ms_r)}
        cs = {"workload": f"accumulate(+, inclusive) 2^30 {name}", "device_ms": ms_s, "roofline": frac(2 * eb * n, ms_s)}
        got = ak.reduce("sum", xx, 0, ex)
        last = yy[-1].item()
        if name == "i64":
            exact = int(hx.sum())
            cr["bit_exact_vs_sequential_fold"] = got == exact
            cs["last_element_exact"] = last == exact
        else:
            exact = float(hx.astype(np.float64).sum())
            cr["rel_err_vs_f64"] = abs(got - exact) / exact
            cs["last_rel_err_vs_f64"] = abs(last - exact) / exact
        if ref:
            ho = np.empty_like(hx)
            rr = {}
            cr["cpu_ms"] = timed_host(lambda: rr.__setitem__("v", oracle.ref_reduce(hx, threads=cores)), 2, 1)
            cs["cpu_ms"] = timed_host(lambda: oracle.ref_accumulate(hx, threads=cores, out=ho), 1, 1)
            if name == "f32":
                cr["cpu_rel_err_vs_f64"] = abs(rr["v"] - exact) / exact  # the reference's own f32 fold
        out[f"3_reduce_2p30_{name}"] = cr
        out[f"3_accumulate_2p30_{name}"] = cs
        del xx, yy, res, hx
        torch.cuda.empty_cache()

    # ---- north-star size: SIHSort P=1 of 2^30 keys per GPU (config 5's per-GPU sort), Int64 and UInt64 ----
    n = 1 << 30
    for name, npdt, tdt in (("i64", np.int64, torch.int64), ("u64", np.uint64, torch.uint64)):
        hx = np.empty(n, dtype=npdt)
        ak.bench_keys(args.seed, 0, n, npdt, out=hx)
        xx = torch.from_numpy(hx).to(dev)
        del hx
        oo = torch.empty_like(xx)
        ms = timed_device(ex.stream, lambda: ak.sihsort(xx, None, None, ex, out=oo, capacity=n), 3)
        fp_ok = fingerprint(xx) == fingerprint(oo) and is_sorted(oo, name == "u64")
        out[f"5_sihsort_p1_2p30_{name}"] = {
            "workload": f"SIHSort P=1 of 2^30 {name} bench keys (north-star per-GPU size)", "device_ms": ms,
            "gbs": n * 8 / 1e9 / (ms / 1e3), "sorted_and_multiset_equal": fp_ok}
        del xx, oo
        torch.cuda.empty_cache()
    return out


# ----------------------------------------------------------------------------- our arm

def main():
    args = parse()
    rank, world, local = dist_env()
    if args.gpus != world and world > 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    if args.impl == "reference":
        reference_arm(args, rank, max(world, args.gpus if world == 1 else world))
        return

    import numpy as np
    import torch

    import paper_2507_16710_b200 as ak

    # AKB_BENCH_SHARE_GPU=1 (test mode, tests/test_multiproc_gpu.py): every rank on device 0,
    # control over gloo and the IPC transport (NCCL refuses two ranks on one device), so the
    # N > 1 code path of this script runs on a one-GPU box; its numbers are not a measurement
    share = world > 1 and os.environ.get("AKB_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
        args.transport = "ipc"
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    pg = None
    comm = None
    if world > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        pg = dist
        if args.transport == "ipc":
            comm = ak.IpcComm(local)
        else:
            obj = [ak.NcclComm.unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            comm = ak.NcclComm(obj[0], world, rank, local)

    ex = ak.ExecBackend(local)
    n = 1 << args.log2n
    unsigned = args.dtype == "uint64"
    np_dt = np.uint64 if unsigned else np.int64
    t_dt = torch.uint64 if unsigned else torch.int64

    # inputs: reference generator on the host -> pinned -> HBM (outside the timed region)
    h_in = torch.empty(n, dtype=t_dt, pin_memory=True)
    ak.bench_keys(args.seed, rank, n, np_dt, out=h_in.numpy())
    d_in = h_in.to(dev, non_blocking=False)
    cap = n if world == 1 else int(1.3 * n) + 4096
    d_out = torch.empty(cap, dtype=t_dt, device=dev)
    cfg = ak.SihConfig()

    def barrier():
        if comm is not None:
            comm.barrier(ex)
        torch.cuda.synchronize(dev)

    def step(src=None, dst=None):
        nonlocal d_out
        src = d_in if src is None else src
        o = d_out if dst is None else dst
        try:
            return ak.sihsort(src, comm, cfg, ex, out=o, capacity=o.numel())
        except ak.CapacityError as e:  # raised on every rank consistently; grow and retry
            o = torch.empty(max(e.required, o.numel()) + 4096, dtype=t_dt, device=dev)
            if dst is None:
                d_out = o
            return ak.sihsort(src, comm, cfg, ex, out=o, capacity=o.numel())

    sampler = ClockSampler(local)
    sampler.start()
    for _ in range(max(args.warmup, 3)):
        out, st = step()

    # ---- timed region: device-resident input -> device output ----
    ex.reset_kernel_time()
    ex.set_profiling(True)
    launches0 = ex.kernel_launches()
    sent0 = comm.bytes_sent() if comm is not None else 0
    barrier()
    stream = ex.stream
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        out, st = step()
    e1.record(stream)
    barrier()
    ms_local = e0.elapsed_time(e1) / args.steps
    gpu_launches = ex.kernel_launches() - launches0
    sent_per_step = ((comm.bytes_sent() - sent0) / args.steps) if comm is not None else 0.0
    if comm is not None:  # the busiest sender bounds the exchange
        sent_per_step = comm.allreduce_max([sent_per_step], ex)[0]
    ex.set_profiling(False)
    fam = {k: ex.kernel_time(k) for k in ("msd", "onesweep", "local", "hist", "merge", "exchange", "search", "other")}
    ms = ms_local
    if comm is not None:
        ms = comm.allreduce_max([ms_local], ex)[0]
    out_count = out.numel()

    # correctness guard on the last output: sortedness of this rank's slice, boundary order with
    # the next rank, and the multiset fingerprint summed over ranks (input == output)
    sorted_ok = is_sorted(out, unsigned)
    fp_in, fp_out = fingerprint(d_in), fingerprint(out)
    if comm is not None:
        import torch.distributed as dist
        cdev = "cpu" if share else dev  # gloo: host tensors
        tot = torch.tensor([fp_in[0], fp_out[0]], dtype=torch.int64, device=cdev)
        dist.all_reduce(tot)
        sums = torch.tensor([[fp_in[1], fp_in[2], fp_out[1], fp_out[2]]], dtype=torch.int64, device=cdev)
        gathered = [torch.empty_like(sums) for _ in range(world)]
        dist.all_gather(gathered, sums)
        g = [sum(int(v) for v in col) % (1 << 64) for col in torch.cat(gathered).cpu().numpy().T]
        multiset_ok = bool(tot[0].item() == tot[1].item() and g[0] == g[2] and g[1] == g[3])
        ok_t = torch.tensor([1 if sorted_ok else 0], device=cdev)
        dist.all_reduce(ok_t, op=dist.ReduceOp.MIN)
        sorted_ok = bool(ok_t.item())
    else:
        multiset_ok = fp_in == fp_out

    # ---- e2e: host buffers, H2D of every step's input + D2H of its output inside the timed region ----
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, ak, torch, np, ex, comm, cfg, h_in, n, t_dt, dev, barrier, world)
    clocks = sampler.stop()

    if rank != 0:
        if pg is not None:
            pg.destroy_process_group()
        return

    peak, peak_kind = measured_peaks()
    # Algorithmic HBM bytes per launch of each kernel family:
    # a partition / digit pass and the on-chip range sort each read and write every key once
    # (16 B/key), the top-digit histogram reads every key once (8 B/key).
    alg_per_key = {"msd": 16, "onesweep": 16, "local": 16, "hist": 8}
    kernels = {}
    for k, per_key in alg_per_key.items():
        t_ms, cnt = fam[k]
        if cnt:
            avg = t_ms / cnt
            ach = per_key * n / (avg / 1e3) / 1e9
            kernels[k] = {"launches_per_step": cnt / args.steps, "avg_launch_ms": avg,
                          "alg_bytes_per_launch": per_key * n, "achieved_gbs": ach, "frac": ach / peak}
    dom = max(kernels, key=lambda k: fam[k][0]) if kernels else None
    tr = ncu_traffic(dom)
    names = {"msd": "msd_pass_kernel (unstable top-digit partition pass over all keys; per-bin atomic cursors)",
             "onesweep": "onesweep_kernel (one 8-bit digit pass over all keys)",
             "local": "counting stage (local_count3_kernel: <= 4608-key bucket ranges, 2 CTAs/SM; local_big_kernel: "
                      "<= 18432-key ranges at 2^29-2^30, 1 CTA/SM; on-chip counting sort, TMA-fed, persistent)",
             "hist": "hist_kernel (top-digit histograms)"}
    roofline = None
    if dom:
        kd = kernels[dom]
        roofline = {"bound": "hbm", "kernel": names[dom], "achieved": kd["achieved_gbs"], "peak": peak,
                    "unit": "GB/s", "frac": kd["frac"], "traffic": (tr * n) if tr else None,
                    "peak_kind": peak_kind, "alg_bytes_per_launch": kd["alg_bytes_per_launch"],
                    "avg_launch_ms": kd["avg_launch_ms"], "launches": fam[dom][1]}
    alg_step = sum(alg_per_key[k] * n * fam[k][1] / args.steps for k in kernels)
    floor_ms = alg_step / (peak * 1e9) * 1e3  # HBM floor of the bytes this algorithm moves
    value = world * n * 8 / 1e9 / (ms / 1e3)
    phases = {k: v[0] / args.steps for k, v in fam.items()}
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": f"distributed sample sort (SIHSort) of 2^{args.log2n} {args.dtype.capitalize()} "
                               f"keys per GPU (BASELINE config {'4' if args.log2n == 28 else '5'})",
                   "keys_per_gpu": n, "global_keys": world * n, "parallelism": f"sihsort over {world} GPU(s)",
                   "generator": "reference bench.cpp mt19937_64 per-rank seeds", "l2": "inputs > L2 (no flush)",
                   "sorted_check": sorted_ok, "multiset_fingerprint_check": multiset_ok,
                   "output_keys_rank0": out_count},
        "roofline": roofline,
        "kernels": kernels,
        "phases_ms_per_step": phases,
        "alg_hbm_bytes_per_step": alg_step,
        "hbm_floor_ms": floor_ms,
        "step_frac_of_alg_floor": floor_ms / ms,
        "gpu_launches": gpu_launches,
        "clocks": clocks,
    }
    if share:
        line["config"]["test_mode"] = "AKB_BENCH_SHARE_GPU: every rank on GPU 0 (code-path test, not a measurement)"
    if world > 1 and fam["exchange"][1]:
        ex_ms = fam["exchange"][0] / fam["exchange"][1]
        sent = sent_per_step
        line["nvlink"] = {"transport": args.transport,
                          "exchange": ("NCCL grouped send/recv into receive buffers, then the P-way merge"
                                       if args.transport == "nccl" else
                                       "fused into the P-way merge: runs read straight from the peers' sorted "
                                       "arrays through CUDA IPC mappings (exchange_ms = that merge)"),
                          "exchange_ms_rank0": ex_ms,
                          "bytes_sent_per_gpu": sent, "bytes_sent_note": "max over ranks, counted by the communicator",
                          "bus_gbs": sent / 1e9 / (ex_ms / 1e3),
                          "peak_gbs": NVLINK_MEASURED_GBS, "peak_kind": "measured peer copy (B200_PROFILING.md)",
                          "frac": sent / 1e9 / (ex_ms / 1e3) / NVLINK_MEASURED_GBS,
                          "nominal_gbs": NVLINK_NOMINAL_GBS}
    if e2e:
        line["e2e"] = e2e
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(args)
        except Exception as exc:  # the baseline is reported, never the product
            line["cpu_baseline"] = {"value": None, "unit": "GB/s", "cores": None, "kind": "reference",
                                    "sample": f"unavailable: {exc}"}
    if world == 1 and not args.no_configs:
        del d_in, d_out, out
        torch.cuda.empty_cache()
        try:
            line["configs"] = run_configs(args, ex, dev, peak)
        except Exception as exc:
            line["configs"] = {"error": repr(exc)}
    print(json.dumps(line), flush=True)
    if pg is not None:
        pg.destroy_process_group()


def run_e2e(args, ak, torch, np, ex, comm, cfg, h_in, n, t_dt, dev, barrier, world):
    """End to end through the public API with host buffers. Pipelined: two device buffer sets;
    step i: H2D(input) on an upload stream -> ak.sihsort on the ctx stream -> D2H(output) on a
    download stream, so step i+1's upload overlaps step i's download. Also the blocking
    single-call C-ABI path (ak.sihsort_host) for reference."""
    k = max(3, min(args.steps, 10))
    cap = n if world == 1 else int(1.3 * n) + 4096
    d_in2 = [torch.empty(n, dtype=t_dt, device=dev) for _ in range(2)]
    d_out2 = [torch.empty(cap, dtype=t_dt, device=dev) for _ in range(2)]
    h_out2 = [torch.empty(cap, dtype=t_dt, pin_memory=True) for _ in range(2)]
    up, down = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev_up = [torch.cuda.Event() for _ in range(2)]
    ev_down = [torch.cuda.Event() for _ in range(2)]
    for e in ev_down:
        e.record(down)
    counts = [0, 0]

    def upload(j):  # d_in2[j % 2] is free: step j - 2's (blocking) sort has returned
        b = j % 2
        with torch.cuda.stream(up):
            d_in2[b].copy_(h_in, non_blocking=True)
            ev_up[b].record(up)

    def sort_and_download(j):
        b = j % 2
        ex.stream.wait_event(ev_up[b])
        ex.stream.wait_event(ev_down[b])  # d_out2[b] is free once step j - 2's download is done
        with torch.cuda.stream(ex.stream):
            res, _ = ak.sihsort(d_in2[b], comm, cfg, ex, out=d_out2[b], capacity=cap)
        counts[b] = res.numel()
        down.wait_stream(ex.stream)
        with torch.cuda.stream(down):
            h_out2[b][:counts[b]].copy_(d_out2[b][:counts[b]], non_blocking=True)
            ev_down[b].record(down)

    def run(steps):
        # step i + 1's upload is enqueued before step i's (blocking) sort, so the upload stream
        # stays busy while step i sorts and step i - 1's output downloads
        upload(0)
        for i in range(steps):
            if i + 1 < steps:
                upload(i + 1)
            sort_and_download(i)

    run(2)  # warm-up
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(up)
    run(k)
    d2h = sum(counts[i % 2] * 8 for i in range(k))
    e1.record(down)
    barrier()
    pipe_ms = e0.elapsed_time(e1) / k
    if comm is not None:
        pipe_ms = comm.allreduce_max([pipe_ms], ex)[0]
    ok = bool(np.array_equal(h_out2[(k - 1) % 2][:counts[(k - 1) % 2]].numpy(),
                             d_out2[(k - 1) % 2][:counts[(k - 1) % 2]].cpu().numpy()))
    del d_in2, d_out2
    torch.cuda.empty_cache()

    # blocking single call per step: ak_sihsort_host_* (H2D + sort + D2H inside the C ABI)
    h_out = torch.empty(cap, dtype=t_dt, pin_memory=True)
    hin_np, hout_np = h_in.numpy(), h_out.numpy()
    ak.sihsort_host(hin_np, comm, cfg, ex, out=hout_np)  # warm-up
    barrier()
    kb = max(3, min(args.steps, 5))
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(ex.stream)
    for _ in range(kb):
        ak.sihsort_host(hin_np, comm, cfg, ex, out=hout_np)
    e3.record(ex.stream)
    barrier()
    blk_ms = e2.elapsed_time(e3) / kb
    if comm is not None:
        blk_ms = comm.allreduce_max([blk_ms], ex)[0]
    return {"value": world * n * 8 / 1e9 / (pipe_ms / 1e3), "unit": "GB/s", "h2d_bytes_per_step": n * 8,
            "d2h_bytes_per_step": d2h // k, "ms_per_step": pipe_ms, "steps": k, "output_copy_check": ok,
            "how": "public API ak.sihsort on device buffers; every step copies its input from pinned host memory "
                   "(upload stream) and its output back (download stream); two buffer sets: step i+1's upload "
                   "is enqueued before step i's sort, so it overlaps that sort and step i-1's download (PCIe "
                   "is full duplex)",
            "blocking": {"value": world * n * 8 / 1e9 / (blk_ms / 1e3), "ms_per_step": blk_ms, "steps": kb,
                         "how": "one blocking C-ABI call per step (ak_sihsort_host_*): H2D + sort + D2H"}}


if __name__ == "__main__":
    main()
