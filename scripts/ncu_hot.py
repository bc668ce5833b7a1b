"""Summarise an `ncu --page source --csv --print-source sass` dump: top stall sites."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
S = h.index("Warp Stall Sampling (All Samples)")
cols = ["stall_long_sb", "stall_short_sb", "stall_wait", "stall_selected", "stall_not_selected",
        "stall_math", "stall_barrier", "stall_branch_resolving", "stall_no_inst", "stall_lg", "stall_mio"]
ci = [h.index(c) for c in cols]
tot = sum(int(r[S] or 0) for r in data)
agg = {c: sum(int(r[i] or 0) for r in data) for c, i in zip(cols, ci)}
print("total samples", tot, {k: round(v / tot, 3) for k, v in agg.items()})
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for r in sorted(data, key=lambda r: -int(r[S] or 0))[:n]:
    detail = " ".join(f"{c[6:]}={r[i]}" for c, i in zip(cols, ci) if r[i] not in ("0", ""))
    print(f"{r[0][-5:]} {int(r[S]):5d} {r[1].strip()[:60]:60s} {detail}")
