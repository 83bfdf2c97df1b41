"""SIHSort over the single-GPU loopback world: P logical ranks x 2^log2n keys each, per-phase
device time (ctx kernel families summed over ranks). AKB_MERGE=pairwise selects the old
log2(P)-level merge tree for comparison."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2507_16710_b200 as ak
P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
log2n = int(sys.argv[2]) if len(sys.argv) > 2 else 24
ins = [torch.from_numpy(ak.bench_keys(42, r, 1 << log2n, np.int64)).cuda() for r in range(P)]
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    outs, stats = ak.sihsort_loopback(ins)
    torch.cuda.synchronize(); t1 = time.perf_counter()
tot = sum(o.numel() for o in outs)
cat = torch.cat(outs)
ok = bool((cat[1:] >= cat[:-1]).all()) and tot == P << log2n
print(f"loopback P={P} 2^{log2n}/rank merge={os.environ.get('AKB_MERGE','pway')}: wall {1e3*(t1-t0):.1f} ms (ranks share one GPU) sorted={ok}")
