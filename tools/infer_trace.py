"""Summarise FH_INFER_TRACE printf lines (per-CTA globaltimer stamps) of the
LAST fh_infer call in a log: CTA start spread, per-phase medians, CTA end spread."""
import sys
import statistics as st
lines = [l.split() for l in open(sys.argv[1]) if l.startswith("TR ")]
n = max(int(l[1]) for l in lines) + 1
last = lines[-n:]
T = [[int(x) for x in l[2:]] for l in last]
t0 = min(r[0] for r in T)
names = ["start", "levels", "weights", "Xfull", "mma1", "e1", "mma2", "y"]
for i, nm in enumerate(names):
    v = [r[i] - t0 for r in T]
    print(f"{nm:8s} min {min(v):6d} med {int(st.median(v)):6d} max {max(v):6d} ns")
