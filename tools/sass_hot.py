"""Summarise an `ncu --page source --csv` (SASS) export: top instructions by stall
samples and by executed instructions, with the dominant stall reasons."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]


def f(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return 0.0


tot = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in data)
ins = sum(f(d["Instructions Executed"]) for d in data)
print("total samples", tot, "instructions", ins)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
key = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
for d in sorted(data, key=lambda d: -f(d[key]))[:n]:
    st = sorted(((f(d[c]), c[6:]) for c in stall_cols), reverse=True)[:3]
    print("%6s %5.1f%% ins %10d  %-60s %s" % (d["Address"], 100 * f(d["Warp Stall Sampling (All Samples)"]) / tot,
                                        f(d["Instructions Executed"]), d["Source"][:60],
                                        " ".join("%s:%d" % (c, v) for v, c in st if v)))

tot_by = {c[6:]: sum(f(d[c]) for d in data) for c in stall_cols}
print("stall totals:", " ".join("%s:%.1f%%" % (k, 100 * v / tot) for k, v in sorted(tot_by.items(), key=lambda kv: -kv[1]) if v > 0.005 * tot))
