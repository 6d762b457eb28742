"""Top SASS instructions by stall samples from `ncu --page source --print-source sass --csv` output."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
i_src, i_s = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
i_ex = hdr.index("Instructions Executed")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[i_s]), int(r[i_ex]), r[i_src].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
print(f"total samples {tot}, instructions {sum(d[1] for d in data)}")
for s, ex, src in sorted(data, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{100*s/tot:5.1f}% {ex:10d}  {src}")
# opcode histogram of executed instructions
from collections import Counter
c = Counter()
for s, ex, src in data:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    c[op.split(".")[0]] += ex
print("executed by opcode:", ", ".join(f"{k}:{v/1e6:.1f}M" for k, v in c.most_common(14)))
