"""Every BASELINE.json config on one B200: device time, throughput, HBM roofline fraction.

    python tools/configs.py [--reps 5] [--json out.json]

Inputs are device-resident; times are CUDA events on the ctx stream (mean of reps after
one warm-up). Algorithmic bytes follow SURVEY.md §8(d) / DESIGN.md §2. This is the
evidence table behind profiles/r01_configs.txt; bench.py remains the headline.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_16710_b200 as ak  # noqa: E402


def peak():
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


def timed(ex, fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0.record(ex.stream)
        fn()
        e1.record(ex.stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.mean(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    ex = ak.ExecBackend(0)
    dev = torch.device("cuda:0")
    P = peak()
    rows = []

    def row(name, ms, alg_bytes, keys=None):
        gbs = alg_bytes / (ms / 1e3) / 1e9
        r = {"config": name, "ms": ms, "alg_bytes": alg_bytes, "alg_gbs": gbs, "frac_hbm": gbs / P}
        if keys:
            r["keys_gbs"] = keys / (ms / 1e3) / 1e9
        rows.append(r)
        print(json.dumps(r), flush=True)

    # 1. merge_sort of 1e6 uniform Int64 (bench keys), in place
    n = 1_000_000
    x = torch.from_numpy(ak.bench_keys(42, 0, n, np.int64)).to(dev)
    w, s = torch.empty_like(x), torch.empty_like(x)
    ms = timed(ex, lambda: (w.copy_(x), ak.merge_sort(w, s, ex)), a.reps)
    row("merge_sort 1e6 int64 (incl. 8 MB copy)", ms, 16 * n, keys=8 * n)

    # 2. sortperm / merge_sort_by_key of 1e8 Float32 with Int32 payload
    n = 100_000_000
    f = torch.from_numpy(ak.bench_keys(42, 0, n, np.float32)).to(dev)
    out = torch.empty(n, dtype=torch.int32, device=dev)
    bufs = ak.SortpermBuffers.with_capacity(n, torch.float32, torch.int32)
    ms = timed(ex, lambda: ak.sortperm(f, out=out, buffers=bufs, ex=ex), a.reps)
    row("sortperm 1e8 f32 -> i32", ms, 64 * n, keys=4 * n)
    k = torch.empty_like(f)
    v = torch.empty(n, dtype=torch.int32, device=dev)
    iota = torch.arange(n, dtype=torch.int32, device=dev)
    kb = ak.SortByKeyBuffers.with_capacity(n, torch.float32, torch.int32)
    ms = timed(ex, lambda: (k.copy_(f), v.copy_(iota), ak.merge_sort_by_key(k, v, buffers=kb, ex=ex)), a.reps)
    row("merge_sort_by_key 1e8 f32 + i32 (incl. 800 MB copy)", ms, 68 * n + 16 * n, keys=4 * n)
    del f, out, bufs, k, v, iota, kb

    # 3. reduce and inclusive accumulate over 2^30 Float32 and Int64
    n = 1 << 30
    for dt, tdt in ((np.float32, torch.float32), (np.int64, torch.int64)):
        if tdt == torch.float32:
            xx = torch.rand(n, dtype=tdt, device=dev)
        else:
            xx = torch.randint(-10000, 10001, (n,), dtype=tdt, device=dev)
        res = torch.empty(1, dtype=tdt, device=dev)
        kb_ = xx.element_size()
        ms = timed(ex, lambda: ak.reduce_device("sum", xx, res, ex=ex), a.reps)
        row(f"reduce 2^30 {np.dtype(dt).name}", ms, kb_ * n)
        yy = torch.empty_like(xx)
        ms = timed(ex, lambda: ak.accumulate("sum", xx, out=yy, ex=ex), a.reps)
        row(f"accumulate (inclusive) 2^30 {np.dtype(dt).name}", ms, 2 * kb_ * n)
        del xx, yy, res

    # 4. SIHSort P=1 of 2^28 Int64 (bench.py's headline, device-resident in -> out)
    n = 1 << 28
    x = torch.from_numpy(ak.bench_keys(42, 0, n, np.int64)).to(dev)
    o = torch.empty_like(x)
    ms = timed(ex, lambda: ak.sihsort(x, None, None, ex, out=o, capacity=n), a.reps)
    row("sihsort P=1 2^28 int64", ms, 56 * n, keys=8 * n)
    del x, o

    # 5. local sort of 2^30 UInt64 (the per-GPU sort of config 5)
    n = 1 << 30
    x = torch.from_numpy(ak.bench_keys(42, 0, n, np.uint64).view(np.int64)).to(dev)
    w, s = torch.empty_like(x), torch.empty_like(x)
    ms = timed(ex, lambda: (w.copy_(x), ak.merge_sort(w.view(torch.uint64), s.view(torch.uint64), ex)), max(2, a.reps // 2))
    row("merge_sort 2^30 uint64 (incl. 8 GiB copy)", ms, 16 * n, keys=8 * n)
    if a.json:
        with open(a.json, "w") as fh:
            json.dump({"hbm_peak_gbs": P, "rows": rows}, fh, indent=1)


if __name__ == "__main__":
    main()
