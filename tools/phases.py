"""Per-phase timing of the onesweep pass kernel (needs lib/libak_cuda_phases.so:
`make -C paper_2507_16710_b200/csrc phases`). Prints mean phase durations per tile
and the tile launch cadence for the last digit pass of a 2^log2n Int64 sort."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["AKB_LIB"] = os.path.join(ROOT, "paper_2507_16710_b200", "lib", "libak_cuda_phases.so")
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_16710_b200 as ak  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
n = 1 << log2n
dev = torch.device("cuda:0")
ex = ak.ExecBackend(0)
x = torch.from_numpy(ak.bench_keys(42, 0, n, np.int64)).to(dev)
tiles = (n + 6143) // 6144
buf = torch.zeros(tiles * 8, dtype=torch.int64, device=dev)
lib = ak.lib()
lib.ak_debug_set_phase_buffer.argtypes = [C.c_void_p]
assert lib.ak_debug_set_phase_buffer(buf.data_ptr()) == 0
for _ in range(2):
    w = x.clone()
    ak.merge_sort(w, ex=ex)
torch.cuda.synchronize()
ph = buf.view(tiles, 8).cpu().numpy().astype(np.float64)
t0 = ph[:, 0].min()
names = ["load+early-count", "rank", "offsets+scan", "stage+lookback", "scatter(thread0)"]
d = np.diff(ph[:, :6], axis=1)
print(f"tiles={tiles} pass span {(ph[:, 5].max() - t0) / 1e3:.1f} us")
for i, nm in enumerate(names):
    print(f"  {nm:18s} mean {d[:, i].mean() / 1e3:7.2f} us  p50 {np.median(d[:, i]) / 1e3:7.2f}  p90 "
          f"{np.percentile(d[:, i], 90) / 1e3:7.2f}")
life = ph[:, 5] - ph[:, 0]
print(f"  tile lifetime mean {life.mean() / 1e3:.2f} us; start cadence {np.median(np.diff(np.sort(ph[:, 0]))):.1f} ns")
conc = life.sum() / (ph[:, 5].max() - t0)
print(f"  mean concurrent tiles {conc:.0f}")
