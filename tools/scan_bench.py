"""Time ak.accumulate (inclusive sum) over 2^log2n elements: CUDA events, mean of reps after
warm-up; prints ms and algorithmic GB/s (2 x bytes: one read, one write).
usage: python tools/scan_bench.py [int64|float32|...] [log2n] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_16710_b200 as ak  # noqa: E402


def main():
    dt = getattr(torch, sys.argv[1] if len(sys.argv) > 1 else "int64")
    n = 1 << int(sys.argv[2] if len(sys.argv) > 2 else 28)
    reps = int(sys.argv[3] if len(sys.argv) > 3 else 10)
    dev = torch.device("cuda:0")
    ex = ak.ExecBackend(0)
    x = (torch.randint(-10000, 10001, (n,), device=dev).to(dt) if not dt.is_floating_point
         else torch.rand(n, device=dev, dtype=dt))
    y = torch.empty_like(x)
    for _ in range(3):
        ak.accumulate("sum", x, out=y, ex=ex)
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):  # events on the handle's stream, around each call
        s.record(ex.stream)
        ak.accumulate("sum", x, out=y, ex=ex)
        e.record(ex.stream)
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ms = sum(ts) / reps
    print(f"scan {dt} 2^{n.bit_length() - 1}: {ms:.4f} ms  {2 * n * x.element_size() / ms / 1e6:.1f} GB/s")


if __name__ == "__main__":
    main()
