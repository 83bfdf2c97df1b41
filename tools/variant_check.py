"""Quick correctness + timing of a libak_cuda variant (AKB_LIB=...): int64 merge_sort at 2^log2n
vs numpy, then timing. Experiment tool, not a test."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2507_16710_b200 as ak
log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
ex = ak.ExecBackend(0)
x = ak.bench_keys(42, 0, 1 << 20, np.int64)
d = torch.from_numpy(x).cuda(); ak.merge_sort(d, ex=ex)
ok = np.array_equal(d.cpu().numpy(), np.sort(x, kind="stable"))
n = 1 << log2n
x = torch.from_numpy(ak.bench_keys(42, 0, n, np.int64)).cuda()
w = torch.empty_like(x); s = torch.empty_like(x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for r in range(4):
    w.copy_(x); torch.cuda.synchronize()
    e0.record(ex.stream); ak.merge_sort(w, s, ex); e1.record(ex.stream); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"{os.path.basename(os.environ.get('AKB_LIB','default'))}: correct={ok} sort 2^{log2n} int64 ms={min(ts[1:]):.3f}", flush=True)
