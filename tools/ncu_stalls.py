"""Summarise an ncu source-page CSV (--page source --csv --print-source sass):
top stalled instructions with context, and stall reasons per opcode."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
si = h.index("Warp Stall Sampling (All Samples)")
src = h.index("Source")
ex = h.index("Instructions Executed")
cols = [c for c in h if c.startswith('stall_') and 'Not' not in c]
idx = [h.index(c) for c in cols]
tot = sum(float(r[si] or 0) for r in data)
print("total samples", tot)
addr = {r[0]: i for i, r in enumerate(data)}
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 8
top = sorted(range(len(data)), key=lambda i: -float(data[i][si] or 0))[:ntop]
for i in top:
    r = data[i]
    reasons = sorted(((float(r[j] or 0), c) for c, j in zip(cols, idx)), reverse=True)[:2]
    print(f"{r[0][-5:]} {r[si]:>6} ex={r[ex]:>9} {r[src][:60]:60} {reasons}")
    for rr in data[max(0, i - 4):i]:
        print(f"      {rr[0][-5:]} {rr[src][:70]}")
agg = collections.Counter()
cnt = collections.Counter()
for r in data:
    op = r[src].split()
    if not op:
        continue
    o = op[1] if op[0].startswith('@') else op[0]
    o = o.split('.')[0]
    agg[o] += float(r[si] or 0)
    cnt[o] += float(r[ex] or 0)
print("by opcode (samples, executed):")
for k, v in agg.most_common(15):
    print(f"  {k:10} {v:8.0f} {cnt[k]:12.0f}")
