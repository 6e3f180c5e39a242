"""Summarise an ncu --page source --csv (SASS) export: stall reasons overall,
on DADD, and the top instructions by warp-stall samples."""
import csv
import sys


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
h, data = rows[1], rows[2:]
isrc, iss = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
st = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
tot = sum(f(r[iss]) for r in data)
print("total samples", tot)
agg = {h[i]: sum(f(r[i]) for r in data) for i in st}
print({k: int(v) for k, v in sorted(agg.items(), key=lambda kv: -kv[1]) if v > 0})
for op in sys.argv[2:]:
    sel = [r for r in data if op in r[isrc]]
    a = {h[i]: sum(f(r[i]) for r in sel) for i in st}
    print(op, len(sel), {k: int(v) for k, v in sorted(a.items(), key=lambda kv: -kv[1]) if v > 0})
for r in sorted(data, key=lambda r: -f(r[iss]))[:int(20)]:
    print(r[0][-6:], int(f(r[iss])), r[isrc][:90])
