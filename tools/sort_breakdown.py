"""Per-kernel-family device time of one int64 merge_sort at 2^log2n (ctx CUDA-event profiling)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2507_16710_b200 as ak
log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
dt = {"f32": np.float32, "f64": np.float64}.get(sys.argv[2] if len(sys.argv) > 2 else "", np.int64)
n = 1 << log2n
ex = ak.ExecBackend(0)
x = torch.from_numpy(ak.bench_keys(42, 0, n, dt)).cuda()
w = torch.empty_like(x); s = torch.empty_like(x)
for r in range(3):
    w.copy_(x); torch.cuda.synchronize()
    if r == 2:
        ex.reset_kernel_time(); ex.set_profiling(True)
    ak.merge_sort(w, s, ex)
ex.set_profiling(False)
tot = 0
out = []
for f in ("hist", "msd", "onesweep", "local", "other"):
    ms, cnt = ex.kernel_time(f)
    tot += ms
    out.append(f"{f}={ms:.3f}ms/{cnt}")
print(f"AKB_HYBRID={os.environ.get('AKB_HYBRID','auto')} 2^{log2n} {np.dtype(dt).name}: " + " ".join(out) + f" sum={tot:.3f}", flush=True)
