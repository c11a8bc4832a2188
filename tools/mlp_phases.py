"""Per-phase warp-sample shares of mlp_train_kernel from an ncu source-page
CSV (--page source --csv --print-source sass).

An MMA wait is the mbarrier try-wait (SYNCS.PHASECHK) that follows a
tcgen05.commit (UTCBAR) in SASS order, plus the predicated branch on its
result where a not-yet-complete wait stalls; they are named MMA1, MMA2,
MMA3/6, MMA4/5 in order.  "work after" a wait is everything up to the next
MMA wait (epilogue math, shared stores, barriers, the next MMA issue); any
other try-wait (the X tile's TMA barrier) counts as work.  Code after the
kernel's last EXIT (out-of-line retry loops) is reported on its own."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Source' in r)
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h)]
S = h.index('Warp Stall Sampling (All Samples)')
tot = sum(float(r[S] or 0) for r in data)
names = ['MMA1', 'MMA2', 'MMA3/6', 'MMA4/5']
last_exit = max(i for i, r in enumerate(data) if 'EXIT' in r[1])
label = ['prologue'] * len(data)
k, pending, cur = 0, False, 'prologue'
i = 0
while i < len(data):
    ins = data[i][1]
    if i > last_exit:
        label[i] = 'out-of-line retry loops'
        i += 1
        continue
    if 'UTCBAR' in ins:
        pending = True
    if 'SYNCS.PHASECHK' in ins and pending and k < len(names):
        nm = 'wait ' + names[k]
        label[i] = nm
        for j in range(i + 1, min(i + 12, len(data))):
            if 'BRA' in data[j][1] and '@!P' in data[j][1]:
                for q in range(i + 1, j + 1):
                    label[q] = nm
                i = j
                break
        cur = 'work after ' + names[k]
        k += 1
        pending = False
        i += 1
        continue
    label[i] = cur
    i += 1
acc, order = {}, []
for r, lb in zip(data, label):
    if lb not in acc:
        order.append(lb)
        acc[lb] = 0.0
    acc[lb] += float(r[S] or 0)
for p in order:
    print(f"{p:26s} {acc[p] / tot * 100:5.1f}%")
