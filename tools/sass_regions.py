"""Print an ncu SASS source page (csv) with per-instruction stall share and executed counts,
collapsing cold stretches; argv[2] = min stall % to show a line (default 0.5)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Address' in r)
h = rows[hi]; ix = {k: i for i, k in enumerate(h)}
seen = set(); L = []
for r in rows[hi + 1:]:
    if len(r) < 5 or r[0] in seen: continue
    seen.add(r[0]); L.append(r)
f = lambda r, k: float(r[ix[k]] or 0)
tot = sum(f(r, 'Warp Stall Sampling (All Samples)') for r in L) or 1
ti = sum(f(r, 'Instructions Executed') for r in L) or 1
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
print(f"{len(L)} instructions, {ti/1e6:.1f}M warp-instr executed")
acc_s = acc_i = 0.0
for i, r in enumerate(L):
    s = f(r, 'Warp Stall Sampling (All Samples)') / tot * 100; e = f(r, 'Instructions Executed')
    acc_s += s; acc_i += e
    if s >= thr or 'BAR' in r[ix['Source']] or 'EXIT' in r[ix['Source']]:
        print(f"{i:5d} {s:5.1f}% {e/1e6:7.1f}M cum[{acc_s:5.1f}% {acc_i/ti*100:5.1f}%] {r[ix['Source']].strip()[:80]}")
