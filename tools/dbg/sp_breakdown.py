import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2507_16710_b200 as ak
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
dt = {"f32": np.float32, "i32": np.int32}[sys.argv[2] if len(sys.argv) > 2 else "f32"]
ex = ak.ExecBackend(0)
x = torch.from_numpy(ak.bench_keys(42, 0, n, dt)).cuda()
for r in range(3):
    torch.cuda.synchronize()
    if r == 2:
        ex.reset_kernel_time(); ex.set_profiling(True)
    p = ak.sortperm(x, ex=ex, index_dtype=torch.int32)
ex.set_profiling(False)
out = []; tot = 0
for f in ("hist", "msd", "onesweep", "local", "other"):
    ms, cnt = ex.kernel_time(f); tot += ms; out.append(f"{f}={ms:.3f}ms/{cnt}")
print(f"sortperm {n} {np.dtype(dt).name}: " + " ".join(out) + f" sum={tot:.3f}", flush=True)
