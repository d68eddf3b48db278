"""Summarise an ncu --page source --csv SASS dump: samples / executed instructions by
40-line window with the notable opcodes, plus the top stalled instructions."""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
S = lambda d: float(d['Warp Stall Sampling (All Samples)'] or 0)
E = lambda d: float(d['Instructions Executed'] or 0)
tot = sum(map(S, data)); ex = sum(map(E, data))
W = int(sys.argv[2]) if len(sys.argv) > 2 else 40
KEY = ('UTCHMMA', 'MUFU', 'STTM', 'LDTM', 'SYNCS', 'STS', 'LDS', 'UBLKCP', 'UTMALDG', 'FENCE',
       'BAR', 'RED', 'ATOM', 'LDG', 'STG', 'NANOSLEEP', 'DMUL', 'DFMA', 'MEMBAR', 'SHFL')
for s in range(0, len(data), W):
    seg = data[s:s + W]
    smp = sum(map(S, seg)); e = sum(map(E, seg))
    ops = set()
    for d in seg:
        m = re.match(r'\s*(@!?U?P\w+\s+)?([A-Z0-9_.]+)', d['Source'])
        if m and m.group(2).split('.')[0] in KEY:
            ops.add(m.group(2).split('.')[0])
    if smp / tot > 0.003 or e / ex > 0.003:
        print(f"{s:5d}-{s + W:5d} samp {smp / tot * 100:5.1f}% exec {e / ex * 100:5.1f}%  {sorted(ops)}")
print("top stalls")
for i in sorted(range(len(data)), key=lambda i: -S(data[i]))[:25]:
    d = data[i]
    st = sorted(((k, float(d[k] or 0)) for k in h if k.startswith('stall_') and 'Not Issued' not in k), key=lambda x: -x[1])[:2]
    print(f"{i:5d} {S(d) / tot * 100:5.2f}% ex {E(d) / ex * 100:5.2f}% {d['Source'][:60]:60s} {st}")
