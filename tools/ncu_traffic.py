"""Per-step DRAM traffic of one PSDO iteration from an ncu capture of
tools/ncu_target.py, written to profiles/ncu_traffic_<n>.json (read by
bench.py's roofline "traffic" field).

Capture (one GPU; ncu_target runs a 1-iteration warm-up, then the measured
iterations, kernels launched one by one in the body order below):

    ncu --set full --clock-control none -k regex:"k_mixed_down0|k_down_l0|k_cdownz|k_cupz|k_up_l0|k_ortho2|k_update2" \
        -s 14 -c 14 -o prof python tools/ncu_target.py      (depth 6: 2 depth + 2 launches per iteration)

    python tools/ncu_traffic.py prof.ncu-rep 256 [depth]
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
def body(depth: int) -> list[str]:
    """the iteration's launches in order (net_up_L0: tiled and mixed cells, k_up_l0m)"""
    return (["net_mixed_down_L0"] + [f"net_down_L{l}" for l in range(depth - 1)] + [f"net_coarse_L{depth - 1}"] +
            [f"net_up_L{l}" for l in range(depth - 2, -1, -1)] + ["ortho", "update"])


def main() -> None:
    rep, n = sys.argv[1], int(sys.argv[2])
    depth = int(sys.argv[3]) if len(sys.argv) > 3 else 6
    BODY = body(depth)
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    unit = rows[1]
    col = {k: i for i, k in enumerate(h)}

    def val(r, k):
        v = float(r[col[k]].replace(",", ""))
        u = unit[col[k]]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "msecond": 1e3, "nsecond": 1e-3}.get(u, 1)

    data = rows[2:]
    if len(data) < len(BODY):
        raise SystemExit(f"need {len(BODY)} launches, report has {len(data)}")
    res = {"bytes": {}, "time_us": {}, "kernel": {}, "source": Path(rep).name,
           "metric": "dram__bytes_read.sum + dram__bytes_write.sum per launch"}
    for name, r in zip(BODY, data[: len(BODY)]):
        res["bytes"][name] = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
        res["time_us"][name] = val(r, "gpu__time_duration.sum")
        res["kernel"][name] = r[col["Kernel Name"]].split("(")[0]
    dst = ROOT / "profiles" / f"ncu_traffic_{n}.json"
    dst.write_text(json.dumps(res, indent=1) + "\n")
    print("wrote", dst)
    for k in BODY:
        print(f"{k:18s} {res['kernel'][k]:32s} {res['time_us'][k]:8.1f} us {res['bytes'][k] / 1e6:8.1f} MB")


if __name__ == "__main__":
    main()
