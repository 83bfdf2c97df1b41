"""Summarise ncu outputs into the tracked profiles/ directory.

    python tools/ncu_summary.py full  <report.ncu-rep | raw.csv> [--keys N]   # --set full capture
    python tools/ncu_summary.py launches <launches.csv>               # gpu__time_duration list

`full` prints, per profiled launch, the metrics the roofline uses (duration, DRAM
bytes read/written, DRAM %, SM/L1 busy, occupancy, registers) and, with --keys,
the DRAM bytes per key. `launches` aggregates a launch list by kernel name and
prints each kernel's share of the total device time.
"""
import csv
import collections
import io
import subprocess
import sys

FULL_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved_occ_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
        "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1.0}


def _val(v, unit):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    return x * UNIT.get(unit, 1.0)


def full(path, keys=None):
    if path.endswith(".csv"):  # `ncu -i rep --page raw --csv` output saved on the GPU box
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    name_i = hdr.index("Kernel Name")
    for r in data:
        print(f"kernel: {r[name_i][:110]}")
        for m, short in FULL_METRICS:
            if m not in hdr:
                continue
            i = hdr.index(m)
            v = _val(r[i], units[i])
            if short == "duration" and isinstance(v, float):
                print(f"  {short:18s} {v * 1e3:.4f} ms")
            elif short.startswith("dram_") and not short.endswith("pct") and isinstance(v, float):
                extra = f"  ({v / keys:.3f} B/key)" if keys else ""
                print(f"  {short:18s} {v / 1e9:.4f} GB{extra}")
            else:
                print(f"  {short:18s} {r[i]} {units[i]}")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        k = r[ki].split("(")[0][:80]
        t = _val(r[vi], r[ui])
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += t
    tot = sum(a[1] for a in agg.values())
    print(f"{'launches':>8} {'total ms':>10} {'avg us':>9} {'share':>6}  kernel")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{c:8d} {t * 1e3:10.3f} {t * 1e6 / c:9.1f} {100 * t / tot:5.1f}%  {k}")
    print(f"{sum(a[0] for a in agg.values()):8d} {tot * 1e3:10.3f}  total")


if __name__ == "__main__":
    if sys.argv[1] == "full":
        k = None
        if "--keys" in sys.argv:
            k = float(sys.argv[sys.argv.index("--keys") + 1])
        full(sys.argv[2], k)
    else:
        launches(sys.argv[2])
