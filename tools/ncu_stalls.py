"""Stall-reason shares (pc sampling) from an ncu --page raw --csv export: tools/ncu_stalls.py <raw.csv>..."""
import csv, sys
for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    h, v = rows[0], rows[2]
    st = {}
    for k, x in zip(h, v):
        if k.startswith('smsp__pcsamp_warps_issue_stalled_') and not k.endswith('not_issued'):
            try: st[k.replace('smsp__pcsamp_warps_issue_stalled_', '')] = float(x.replace(',', ''))
            except ValueError: pass
    tot = sum(st.values()) or 1
    print(f, ' '.join(f"{k}={x / tot * 100:.0f}%" for k, x in sorted(st.items(), key=lambda t: -t[1])[:10]))
