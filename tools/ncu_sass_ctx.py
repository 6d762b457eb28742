"""Hot SASS instructions with their stall reasons and preceding context.

    ncu -i rep --page source --print-source sass --csv -k regex:NAME --launch-count 1 > x.csv
    python tools/ncu_sass_ctx.py x.csv [top] [context]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], encoding="latin-1")))
hdr = rows[1]
data = rows[2:]
half = len(data) // 2
if len(data) % 2 == 0 and data[:half] == data[half:]:
    data = data[:half]
i_src, i_s, i_ex = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
stalls = [(i, h[6:]) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 8
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 6


def num(v):
    try:
        return int(v)
    except ValueError:
        return 0


tot = sum(num(r[i_s]) for r in data) or 1
order = sorted(range(len(data)), key=lambda k: -num(data[k][i_s]))[:top]
for k in sorted(order):
    r = data[k]
    why = sorted(((num(r[i]), n) for i, n in stalls), reverse=True)[:3]
    print(f"=== {100 * num(r[i_s]) / tot:.1f}%  " + " ".join(f"{n}:{v}" for v, n in why if v))
    for rr in data[max(0, k - ctx): k + 1]:
        print(f"{rr[i_s]:>6} {rr[i_ex]:>9}  {rr[i_src]}")
