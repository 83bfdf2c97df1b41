"""Small runs of the round-2 kernels for compute-sanitizer (one tool per call):
    compute-sanitizer --tool racecheck python tools/sanitize_smoke.py
Counting local stage (device-planned small path and hybrid path), MSD passes, the fused
pull-merge of a 4-rank loopback SIHSort, sortperm / by_key onesweep, scan."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_16710_b200 as ak  # noqa: E402

ex = ak.ExecBackend(0)
dev = torch.device("cuda:0")
for n in (50_000, 1 << 20, (1 << 24) + 3):
    x = ak.bench_keys(7, 0, n, np.int64)
    t = torch.from_numpy(x).to(dev)
    ak.merge_sort(t, ex=ex)
    assert np.array_equal(t.cpu().numpy(), np.sort(x)), n
ins = [torch.from_numpy(ak.bench_keys(9, r, 200_000 + r, np.int64)).to(dev) for r in range(4)]
outs, _ = ak.sihsort_loopback(ins)
allin = np.sort(np.concatenate([t.cpu().numpy() for t in ins]))
assert np.array_equal(np.concatenate([o.cpu().numpy() for o in outs]), allin)
f = torch.from_numpy(ak.bench_keys(3, 0, 300_000, np.float32)).to(dev)
p = ak.sortperm(f, ex=ex, index_dtype=torch.int32)
assert np.array_equal(p.cpu().numpy(), np.argsort(f.cpu().numpy(), kind="stable"))
y = ak.accumulate("sum", torch.arange(1 << 20, dtype=torch.int64, device=dev), ex=ex)
assert int(y[-1]) == (1 << 20) * ((1 << 20) - 1) // 2
print("sanitize smoke ok")
