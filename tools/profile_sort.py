"""Small driver for ncu captures of the hot kernels (one process, one GPU).

    python tools/profile_sort.py --what sort --log2n 28 --reps 2
ncu usage (after the same command exited 0 without ncu):
    ncu --set full --clock-control none --import-source on -k regex:onesweep -s 8 -c 2 -o prof \
        python tools/profile_sort.py --what sort
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_16710_b200 as ak  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--what", default="sort", choices=["sort", "sortperm", "bykey", "reduce", "scan", "sihsort"])
    p.add_argument("--log2n", type=int, default=28)
    p.add_argument("--reps", type=int, default=2)
    a = p.parse_args()
    dev = torch.device("cuda:0")
    ex = ak.ExecBackend(0)
    n = 1 << a.log2n
    if a.what in ("sort", "sihsort"):
        x = torch.from_numpy(ak.bench_keys(42, 0, n, np.int64)).to(dev)
    elif a.what in ("sortperm", "bykey"):
        x = torch.from_numpy(ak.bench_keys(42, 0, n, np.float32)).to(dev)
    elif a.what == "reduce":
        x = torch.randint(-10000, 10001, (n,), dtype=torch.int64, device=dev)
    else:
        x = torch.randint(-10000, 10001, (n,), dtype=torch.int64, device=dev)
    torch.cuda.synchronize()
    scratch = torch.empty_like(x)
    work = torch.empty_like(x)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for r in range(a.reps + 1):
        if a.what == "sort":
            work.copy_(x)
            torch.cuda.synchronize()
            ev0.record(ex.stream)
            ak.merge_sort(work, scratch, ex)
            ev1.record(ex.stream)
        elif a.what == "sortperm":
            ev0.record(ex.stream)
            ak.sortperm(x, ex=ex, index_dtype=torch.int32)
            ev1.record(ex.stream)
        elif a.what == "bykey":
            k = x.clone()
            v = torch.arange(n, dtype=torch.int32, device=dev)
            torch.cuda.synchronize()
            ev0.record(ex.stream)
            ak.merge_sort_by_key(k, v, ex=ex)
            ev1.record(ex.stream)
        elif a.what == "reduce":
            ev0.record(ex.stream)
            ak.reduce("sum", x, 0, ex)
            ev1.record(ex.stream)
        elif a.what == "scan":
            ev0.record(ex.stream)
            ak.accumulate("sum", x, out=work, ex=ex)
            ev1.record(ex.stream)
        else:
            ev0.record(ex.stream)
            ak.sihsort(x, None, None, ex, out=work, capacity=n)
            ev1.record(ex.stream)
        torch.cuda.synchronize()
        if r:
            print(f"{a.what} n=2^{a.log2n}: {ev0.elapsed_time(ev1):.3f} ms", flush=True)


if __name__ == "__main__":
    main()
