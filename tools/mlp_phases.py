"""Per-phase warp-sample shares of mlp_train_kernel from an ncu source-page
CSV (--page source --csv --print-source sass).  "wait k" = the mbarrier
try-wait of wait k (SYNCS.PHASECHK) and the predicated branch on its result
(where a not-yet-complete wait stalls); "work after k" = everything between
that wait and the next one (epilogue math, shared stores, barriers, MMA issue)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Source' in r)
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h)]
S = h.index('Warp Stall Sampling (All Samples)')
tot = sum(float(r[S] or 0) for r in data)
names = ['X', 'MMA1', 'MMA2', 'MMA3/6', 'MMA4/5']
syncs = [i for i, r in enumerate(data) if 'SYNCS.PHASECHK' in r[1]][:len(names)]
wait_rows = set()
for k, i in enumerate(syncs):
    wait_rows.add(i)
    for j in range(i + 1, min(i + 12, len(data))):
        if 'BRA' in data[j][1] and '@!P' in data[j][1]:
            wait_rows.add(j)
            break
acc = {}
order = []
for idx, r in enumerate(data):
    k = sum(1 for i in syncs if i <= idx) - 1
    if idx in wait_rows:
        p = 'wait ' + names[k]
    else:
        p = 'prologue' if k < 0 else 'work after ' + names[k]
    if p not in acc:
        order.append(p)
    acc[p] = acc.get(p, 0) + float(r[S] or 0)
for p in sorted(order, key=lambda p: order.index(p)):
    print(f"{p:24s} {acc[p] / tot * 100:5.1f}%")
