"""The reference's benchmark harness contract on the B200 path.

`run_bench` / `write_bench_outputs` / `write_bench_report` mirror
`npsd::run_bench` and the CSV writers of `src/bench.cpp:35-263`: method tokens
`solver[+precond]` (`parse_method_token`, :20-29), one row per (system, method),
`rows.csv` (+ `traces/<system>__<method>.csv`), `summary.csv` (per-method
means) and `speedup_hist.csv` (speedup over `cg` on the same system, converged
rows, bins 0 .. 64 and overflow) with the reference's column order and number
formats, so the reference's own `load_bench_rows` reads them.

Device methods: `cg`, `pcg+none|jacobi|ic0` (cg.cuh; IC0 by level-scheduled
triangular sweeps), `psd|psdo+neural|none|jacobi` (the device PSDO loop with
the network, IdentityPrecond or JacobiPrecond). Every solve sets
nullspace_projection = is_pure_neumann(frame) like bench.cpp:52. `fpcg` and
IC0 under psd/psdo are not on the device path; their rows carry an error, like
the reference's rows for failed methods.

    python -m paper_2310_00177_b200.bench_matrix out_dir [--systems C1,C2,C3] [--methods cg,pcg+jacobi,psdo+neural]
"""
from __future__ import annotations

import argparse
import os
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

SOLVERS = ("cg", "pcg", "fpcg", "psd", "psdo")
PRECONDS = ("none", "jacobi", "ic0", "neural")
EDGES = (0.0, 0.5, 1.0, 2.0, 4.0, 8.0, 16.0, 32.0, 64.0)


def parse_method_token(token: str) -> tuple[bool, str, str]:
    """parse_method_token (bench.cpp:20-29): (ok, solver, precond)."""
    solver, _, precond = token.partition("+")
    precond = precond if "+" in token else "none"
    return solver in SOLVERS and precond in PRECONDS, solver, precond


@dataclass
class BenchRow:
    system: str
    method: str
    n_f: int = 0
    iterations: int = 0
    converged: bool = False
    setup_seconds: float = 0.0
    iterate_seconds: float = 0.0
    precond_seconds: float = 0.0
    total_seconds: float = 0.0
    final_rel_residual: float = 0.0
    error: str = ""
    residual_history: list = field(default_factory=list)
    cumulative_seconds: list = field(default_factory=list)


def run_one(ctx_for, system: str, types: np.ndarray, b: np.ndarray, token: str, cfg) -> BenchRow:
    import time

    import paper_2310_00177_b200 as b200

    row = BenchRow(system, token, n_f=int(b.size))
    ok, solver, precond = parse_method_token(token)
    if not ok:
        row.error = "unknown method token"
        return row
    if solver == "fpcg" or (precond == "ic0" and solver != "pcg"):
        row.error = f"{token}: not available on the B200 device path"
        return row
    try:
        ctx = ctx_for(precond)
        t0 = time.perf_counter()
        ctx.set_mask(types)
        setup = time.perf_counter() - t0
        ns = ctx.is_pure_neumann()  # bench.cpp:52
        scfg = b200.SolveConfig(tol_reduction=cfg.tol_reduction, max_iters=cfg.max_iters,
                                n_ortho=0 if solver == "psd" else cfg.n_ortho, nullspace_projection=ns)
        if solver == "cg":
            res = ctx.pcg_solve(b, scfg, precond="identity")
        elif solver == "pcg":
            res = ctx.pcg_solve(b, scfg, precond=precond if precond in ("jacobi", "ic0") else "identity")
        else:
            res = ctx.psdo_solve(b, scfg, precond=precond)
        rep = res.report
        row.iterations, row.converged = rep.iterations, rep.converged
        row.setup_seconds = setup + rep.setup_seconds
        row.iterate_seconds = rep.iterate_seconds
        row.precond_seconds = rep.precond_seconds
        row.total_seconds = setup + rep.setup_seconds + rep.iterate_seconds
        h = list(rep.residual_history)
        row.final_rel_residual = h[-1] / h[0] if h and h[0] > 0 else 0.0
        row.residual_history, row.cumulative_seconds = h, list(rep.cumulative_seconds)
    except Exception as e:  # noqa: BLE001 - the row records the failure
        row.error = str(e)
    return row


def _sanitize(s: str) -> str:
    return s.replace("/", "_").replace("+", "_").replace(" ", "_")


def _f9(v: float) -> str:
    return f"{v:.9f}"


def _g17(v: float) -> str:
    # %.17g
    return "%.17g" % v


def write_bench_outputs(rows: list[BenchRow], out_dir) -> None:
    """write_bench_outputs (bench.cpp:139-167)."""
    d = Path(out_dir)
    (d / "traces").mkdir(parents=True, exist_ok=True)
    with open(d / "rows.csv", "w") as f:
        f.write("system,method,n_f,iterations,converged,setup_seconds,iterate_seconds,"
                "precond_seconds,total_seconds,final_rel_residual,error\n")
        for r in rows:
            f.write(f"{r.system},{r.method},{r.n_f},{r.iterations},{1 if r.converged else 0},"
                    f"{_f9(r.setup_seconds)},{_f9(r.iterate_seconds)},{_f9(r.precond_seconds)},"
                    f"{_f9(r.total_seconds)},{_g17(r.final_rel_residual)},{r.error}\n")
    for r in rows:
        if not r.residual_history:
            continue
        with open(d / "traces" / f"{_sanitize(r.system)}__{_sanitize(r.method)}.csv", "w") as f:
            f.write("iter,residual_norm,cumulative_seconds\n")
            for i, v in enumerate(r.residual_history):
                c = r.cumulative_seconds[i] if i < len(r.cumulative_seconds) else 0.0
                f.write(f"{i},{_g17(v)},{_f9(c)}\n")


def load_bench_rows(csv_path) -> list[BenchRow]:
    """load_bench_rows (bench.cpp:168-201): rows.csv back into rows (no
    traces); the error field is the rest of the line."""
    rows = []
    with open(csv_path) as f:
        next(f)  # header
        for line in f:
            line = line.rstrip("\n")
            if not line:
                continue
            parts = line.split(",", 10)
            rows.append(BenchRow(parts[0], parts[1], n_f=int(parts[2]), iterations=int(parts[3]),
                                 converged=parts[4] == "1", setup_seconds=float(parts[5]),
                                 iterate_seconds=float(parts[6]), precond_seconds=float(parts[7]),
                                 total_seconds=float(parts[8]), final_rel_residual=float(parts[9]),
                                 error=parts[10] if len(parts) > 10 else ""))
    return rows


def write_bench_report(rows: list[BenchRow], out_dir) -> None:
    """write_bench_report (bench.cpp:204-263): summary.csv, speedup_hist.csv."""
    d = Path(out_dir)
    d.mkdir(parents=True, exist_ok=True)
    by_method: dict[str, list[BenchRow]] = {}
    for r in rows:
        by_method.setdefault(r.method, []).append(r)
    methods = sorted(by_method)  # std::map order
    with open(d / "summary.csv", "w") as f:
        f.write("method,n_rows,n_converged,mean_iterations,mean_total_seconds,mean_setup_seconds,"
                "mean_precond_seconds\n")
        for m in methods:
            lst = by_method[m]
            n = float(len(lst))
            f.write(f"{m},{len(lst)},{sum(1 for r in lst if r.converged)},"
                    f"{sum(r.iterations for r in lst) / n:.4f},{_f9(sum(r.total_seconds for r in lst) / n)},"
                    f"{_f9(sum(r.setup_seconds for r in lst) / n)},{_f9(sum(r.precond_seconds for r in lst) / n)}\n")
    cg_time = {r.system: r.total_seconds for r in rows if r.method == "cg" and r.converged}
    with open(d / "speedup_hist.csv", "w") as f:
        f.write("method,bin_lo,bin_hi,count\n")
        for m in methods:
            counts = [0] * len(EDGES)
            for r in by_method[m]:
                if not r.converged or r.system not in cg_time or r.total_seconds <= 0.0:
                    continue
                sp = cg_time[r.system] / r.total_seconds
                b = len(EDGES) - 1
                for e in range(len(EDGES) - 1):
                    if EDGES[e] <= sp < EDGES[e + 1]:
                        b = e
                        break
                counts[b] += 1
            for e in range(len(EDGES) - 1):
                f.write(f"{m},{EDGES[e]:.1f},{EDGES[e + 1]:.1f},{counts[e]}\n")
            f.write(f"{m},{EDGES[-1]:.1f},inf,{counts[-1]}\n")


@dataclass
class BenchConfig:
    tol_reduction: float = 1e-6
    max_iters: int = 10000
    n_ortho: int = 2


def run_bench(systems: dict, methods: list[str], cfg: BenchConfig | None = None, model=None) -> list[BenchRow]:
    """systems: name -> (cell types, reduced b). model: NetParams for +neural."""
    import paper_2310_00177_b200 as b200

    cfg = cfg or BenchConfig()
    rows = []
    for name, (types, b) in systems.items():
        ctxs = {}

        def ctx_for(precond, types=types, ctxs=ctxs):
            key = "neural" if precond == "neural" else "plain"
            if key not in ctxs:
                if key == "neural" and model is None:
                    raise RuntimeError("run_bench: neural method requested without --model")
                # plain methods never run the network: any depth the grid divides
                d = model.depth if model else 4
                while d > 1 and any(n % (1 << (d - 1)) for n in types.shape):
                    d -= 1
                p = model if key == "neural" else b200.identity_params(d)
                ctxs[key] = b200.Context(3, types.shape, p)
            return ctxs[key]

        for m in methods:
            rows.append(run_one(ctx_for, name, types, b, m, cfg))
    return rows


def main() -> None:
    import paper_2310_00177_b200 as b200
    from paper_2310_00177_b200 import scenes

    ap = argparse.ArgumentParser()
    ap.add_argument("out_dir")
    ap.add_argument("--systems", default="C1,C2,C3")
    ap.add_argument("--methods", default="cg,pcg+jacobi,psd+neural,psdo+neural,psdo+none,pcg+ic0")
    ap.add_argument("--model", default=str(Path(__file__).parent / "weights" / "npsd3d_L6.npm"))
    a = ap.parse_args()
    model = b200.load_npm(a.model) if a.model and os.path.exists(a.model) else None
    systems = {}
    for name in a.systems.split(","):
        t, seed = scenes.config(name)
        systems[name] = (t, b200.rhs_normal(seed, t.size)[t.reshape(-1) == 0])
    rows = run_bench(systems, a.methods.split(","), model=model)
    write_bench_outputs(rows, a.out_dir)
    write_bench_report(rows, a.out_dir)
    for r in rows:
        print(f"{r.system:4s} {r.method:12s} it={r.iterations:6d} conv={int(r.converged)} total={r.total_seconds:.4f}s"
              + (f" error={r.error}" if r.error else ""))


if __name__ == "__main__":
    main()
