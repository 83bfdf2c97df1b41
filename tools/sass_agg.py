"""Aggregate an ncu SASS source page (csv) by opcode: shared wavefronts, instructions, stall share."""
import csv, collections, re, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]; data = rows[2:]
ix = {k: i for i, k in enumerate(h)}
def f(r, k):
    try: return float(r[ix[k]])
    except Exception: return 0.0
seen = set(); d = []
for r in data:
    a = r[ix['Address']]
    if a in seen: continue
    seen.add(a); d.append(r)
agg = collections.defaultdict(lambda: [0, 0, 0, 0])
for r in d:
    src = r[ix['Source']].strip()
    op = re.sub(r'^@!?U?P\w+\s+', '', src).split()[0] if src else '?'
    a = agg[op]; a[0] += f(r, 'L1 Wavefronts Shared'); a[1] += f(r, 'L1 Wavefronts Shared Ideal')
    a[2] += f(r, 'Instructions Executed'); a[3] += f(r, 'Warp Stall Sampling (All Samples)')
tot = sum(a[0] for a in agg.values()); ti = sum(a[2] for a in agg.values()); ts = sum(a[3] for a in agg.values()) or 1
keys = float(sys.argv[2]) if len(sys.argv) > 2 else 1
print(f'shared wavefronts {tot/1e6:.1f}M ({tot/keys:.3f}/key)  warp-instructions {ti/1e6:.1f}M ({ti/keys:.3f}/key)')
for k, a in sorted(agg.items(), key=lambda x: -x[1][0])[:8]:
    print(f"  {k:22s} wf={a[0]/1e6:7.1f}M ideal={a[1]/1e6:7.1f}M instr={a[2]/1e6:6.1f}M")
print('top by instructions:')
for k, a in sorted(agg.items(), key=lambda x: -x[1][2])[:12]:
    print(f"  {k:22s} instr={a[2]/1e6:6.1f}M stall={100*a[3]/ts:5.1f}%")
