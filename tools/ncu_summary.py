"""Summarise an ncu report: per kernel time, DRAM bytes, GB/s, occupancy, top stalls."""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[0]
def f(v):
    try: return float(v)
    except: return 0.0
for row in r[2:]:
    g = lambda k: row[h.index(k)] if k in h else ""
    t = f(g("gpu__time_duration.sum")); rd = f(g("dram__bytes_read.sum")); wr = f(g("dram__bytes_write.sum"))
    name = g("Kernel Name").split("(")[0][:34]
    st = sorted([(h[i].replace("smsp__pcsamp_warps_issue_stalled_", ""), f(row[i])) for i in range(len(h))
                 if h[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not h[i].endswith("not_issued")], key=lambda t: -t[1])[:4]
    tot = sum(f(row[i]) for i in range(len(h)) if h[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not h[i].endswith("not_issued")) or 1
    print(f"{name:34s} {t:8.1f}us r={rd:7.1f}MB w={wr:6.1f}MB {1e3*(rd+wr)/max(t,1e-9):6.0f}GB/s "
          f"warps={f(g('sm__warps_active.avg.pct_of_peak_sustained_active')):4.0f}% regs={g('launch__registers_per_thread')} "
          f"inst={f(g('smsp__inst_executed.sum'))/1e6:6.1f}M | " + " ".join(f"{k}:{100*v/tot:.0f}%" for k, v in st))
