"""merge_sort of n int64 bench keys (default 1e6, BASELINE config 1), timed per call with
CUDA events on the handle's stream; for launch lists under ncu.
usage: python tools/small_sort.py [n] [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_16710_b200 as ak  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
ex = ak.ExecBackend(0)
x = torch.from_numpy(ak.bench_keys(42, 0, n, np.int64)).cuda()
w, s = torch.empty_like(x), torch.empty_like(x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for r in range(reps + 3):
    w.copy_(x)
    torch.cuda.synchronize()
    e0.record(ex.stream)
    ak.merge_sort(w, s, ex)
    e1.record(ex.stream)
    torch.cuda.synchronize()
    if r >= 3:
        ts.append(e0.elapsed_time(e1))
print(f"merge_sort {n} int64: {np.mean(ts) * 1e3:.1f} us/call (min {np.min(ts) * 1e3:.1f})")
