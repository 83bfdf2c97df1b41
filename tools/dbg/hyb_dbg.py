import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2507_16710_b200 as ak
n = int(sys.argv[1]); ex = ak.ExecBackend(0)
x = ak.bench_keys(42, 3, n, np.int64)
d = torch.from_numpy(x).cuda(); s = torch.empty_like(d)
ak.merge_sort(d, s, ex)
y = d.cpu().numpy(); r = np.sort(x)
bad = np.nonzero(y != r)[0]
print(os.environ.get("AKB_MSD"), os.environ.get("AKB_LOCAL_COUNT"), "n", n, "mismatches", bad.size, bad[:10], "sorted?", bool(np.all(y[1:] >= y[:-1])), "multiset", np.array_equal(np.sort(y), r))
if bad.size:
    i = bad[0]; print(y[i-3:i+5]); print(r[i-3:i+5])
