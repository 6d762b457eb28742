#!/usr/bin/env python
"""bench.py — neural-preconditioned PSDO ("DCDM") time-to-solution on B200.

Metric (BASELINE.json): time-to-solution in ms to relative residual 1e-6 at
256^3 (config C3: free-surface droplet-in-pool), plus per-
iteration ms and HBM GB/s. One step = one frame: set_mask (flags, coarsened
masks, mixed-window kernel tables, linear-block coefficients) + the whole PSDO
solve to 1e-6, with the cell types and the RHS already resident in HBM.
Weights: the repo's trained 3D model (weights/npsd3d_L6.npm) by
default; `--weights identity` gives the identity-equivalent network (PSDO == CG,
the network still runs in full every iteration). The N=1 line also carries the
C4 sequence (32 time-varying 128^3 masks through one context, per-frame
set_mask only) as `sequence_c4`.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N > 1 (torchrun, one rank per GPU): the same frame z-slab sharded across the
ranks (strong scaling): rank r owns a contiguous block of z-planes, ghost planes
move over NCCL before each stencil / conv level, dot products are gathered and
summed in rank order. `--slab` forces that path at N=1
(a one-rank NCCL communicator) to exercise it on one GPU.
"""
from __future__ import annotations

import argparse
import functools
import json
import math
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "DCDM time-to-solution ms (rel-res 1e-6) at 256^3; per-iter ms; HBM GB/s"
UNIT = "ms"


# ------------------------------------------------------------ byte model
def canonical_bytes_per_cell(depth: int) -> dict[str, float]:
    """SURVEY.md §8d canonical algorithmic bytes per fine cell per PSDO
    iteration, split by phase (P1 level-0 down, P2 per coarse kernel, P3
    level-0 up, P4 ortho, P5 update)."""
    m = {"P1": 13.5, "P3": 45.5, "P4": 49.0, "P5": 41.0}
    for l in range(1, depth - 1):
        m[f"P2_down_L{l}"] = 20.5 / 8 ** l
        m[f"P2_up_L{l}"] = 20.5 / 8 ** l
    m[f"P2_coarse_L{depth - 1}"] = 20.0 / 8 ** (depth - 1)
    return m


def processed_bytes(depth: int, n_c: int, n_f: int) -> dict[str, float]:
    """Algorithmic bytes per phase over the cells the launches actually
    process: the f64 solver vectors, the cell byte and the
    level-0 activation y0 exist only at fluid cells (the zero invariant:
    non-fluid entries are exact zeros that are never read); the coarse
    activations x1/out1 and the coarse levels cover their whole grids (the
    network processes all of D).
      P1  r 8 + cell 1 + y0 4 per fluid cell; x1 0.5 per fine cell
      P2  SURVEY §8d per coarse kernel (all cells)
      P3  out1 0.5 per fine cell; cell 1 + y0 4 + d1,Ad1,d2,Ad2 32 + d 8 per fluid cell
      P4  49 per fluid cell (d, d1, d2, r, cell; d', Ad')
      P5  41 per fluid cell (x, d', b, cell; x, r)"""
    m = {"P1": 13.0 * n_f + 0.5 * n_c, "P3": 45.0 * n_f + 0.5 * n_c, "P4": 49.0 * n_f, "P5": 41.0 * n_f}
    for k, v in canonical_bytes_per_cell(depth).items():
        if k.startswith("P2"):
            m[k] = v * n_c
    return m


def phase_of(kernel: str) -> str:
    """Kernel step name (Context.profile_iterations) -> canonical phase."""
    if kernel in ("net_mixed_down_L0", "net_down_L0"):
        return "P1"
    if kernel in ("net_up_L0", "net_mixed_up_L0", "net_out_L0"):
        return "P3"
    if kernel == "ortho":
        return "P4"
    if kernel == "update":
        return "P5"
    return "P2_" + kernel[len("net_"):]


def phase_bytes(model: dict, phase: str) -> float:
    """bytes of a phase in a per-kernel model; "P2" = all coarse kernels"""
    if phase == "P2":
        return sum(v for k, v in model.items() if k.startswith("P2_"))
    return model[phase]


def ncu_traffic(kernels: list, n: int):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of
    the given kernel steps, from the committed ncu capture of this workload
    (profiles/ncu_traffic_<n>.json, written by tools/ncu_traffic.py); None if
    no capture exists."""
    p = ROOT / "profiles" / f"ncu_traffic_{n}.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    vals = [d["bytes"].get(k) for k in kernels]
    return None if any(v is None for v in vals) else float(sum(vals))


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int) -> None:
        self.device = device
        self.proc = None
        self.path = None

    def start(self) -> None:
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "25"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return
        # the timed region starts once samples are flowing (a step is ~20 ms)
        t0 = time.time()
        while time.time() - t0 < 5.0 and not Path(self.path).read_text().strip():
            time.sleep(0.02)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in Path(self.path).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower().startswith("active")})
        loaded = [s for s in sm if s > 0.5 * smax] or sm
        return {"sm_mhz": float(np.median(loaded)) if loaded else None, "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit())}


# -------------------------------------------------------------- workload
@functools.lru_cache(maxsize=None)
def scenes_module():
    """paper_2310_00177_b200/scenes.py (pure numpy geometry) loaded by path, so
    the reference arm never imports the product package or its library."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("npsd_bench_scenes", ROOT / "paper_2310_00177_b200" / "scenes.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def workload(args):
    types, seed = scenes_module().config(args.config, args.n)
    return types, seed


def read_npm(path) -> tuple[int, int, np.ndarray]:
    """Model file ("NPMW", u32 version 1, u32 dim, u32 depth, f32 LE weights;
    net_params.cpp:42-52 layout) parsed with numpy: (dim, depth, weights)."""
    raw = Path(path).read_bytes()
    if raw[:4] != b"NPMW":
        raise ValueError(f"{path}: bad magic")
    ver, dim, depth = np.frombuffer(raw[4:16], "<u4")
    if ver != 1:
        raise ValueError(f"{path}: bad version {ver}")
    return int(dim), int(depth), np.frombuffer(raw[16:], "<f4").copy()


WEIGHTS = ROOT / "paper_2310_00177_b200" / "weights" / "npsd3d_L6.npm"  # = paper_2310_00177_b200.DEFAULT_MODEL


def model_depth() -> int:
    """the depth of the committed model file (its header; no library needed)"""
    return read_npm(WEIGHTS)[1]


def load_weights(kind: str, depth: int):
    import paper_2310_00177_b200 as b200

    if kind == "trained":
        w = b200.load_npm(WEIGHTS)
        if w.depth != depth:
            raise SystemExit(f"trained weights have depth {w.depth}, not {depth}")
        return w
    if kind == "random":
        return b200.init_params(depth, 42)
    return b200.identity_params(depth)


# ------------------------------------------------------------- CPU legs
def reference_weights(kind: str, depth: int) -> np.ndarray:
    """The same weights the B200 arm uses, obtained without the product
    library: the model file parsed with numpy, or the oracle's init/identity
    (bitwise equal to the product's, tests/test_abi.py)."""
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import Oracle  # checker / baseline only

    if kind == "trained":
        dim, d, w = read_npm(WEIGHTS)
        if (dim, d) != (3, depth):
            raise SystemExit(f"trained weights are dim {dim} depth {d}, not 3/{depth}")
        return w
    if kind == "random":
        return Oracle().init_params(3, depth, 42)
    return Oracle().identity_params(3, depth)


def cpu_reference_solve(types, seed, depth, cores, weights="trained", max_iters=20000, name=None):
    """One reference time-to-solution, measured (not extrapolated): the
    unmodified reference psdo_solve (solver.cpp:189-276) on its own
    assemble_poisson_3d + reduce (oracle/_ref), with the 3D network
    restatement as its Preconditioner and the B200 arm's weights, run to
    rel-res 1e-6 on all `cores` host threads. TTS = setup (assembly, reduce,
    NetContext build) + solve, the two spans the reference solver reports."""
    os.environ["OMP_NUM_THREADS"] = str(cores)
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import Ref  # checker / baseline only

    ref = Ref()
    p = reference_weights(weights, depth)
    b = ref.rhs_normal(seed, types.size)[types.reshape(-1) == 0]
    t0 = time.perf_counter()
    r = ref.psdo_solve(types, b, mode="neural", params=p, depth=depth, max_iters=max_iters, tol_reduction=1e-6,
                       n_ortho=2)
    wall = time.perf_counter() - t0
    setup_ms, solve_ms = 1e3 * r["setup_seconds"], 1e3 * r["solve_seconds"]
    it = int(r["iterations"])
    return {
        "value": setup_ms + solve_ms, "unit": UNIT, "cores": cores, "kind": "reference",
        "sample": (f"{types.shape[0]}^3 {name or args_config_name}, {weights} weights: one full reference solve to rel-res "
                   f"1e-6 (measured, not extrapolated): setup {setup_ms:.0f} ms (assemble_poisson_3d + reduce + "
                   f"NeuralPrecond3D build) + {it} PSDO iterations {solve_ms:.0f} ms ({solve_ms / max(it, 1):.1f} "
                   f"ms/iter); {wall:.1f} s wall"),
        "setup_ms": setup_ms, "solve_ms": solve_ms, "iterations": it, "converged": bool(r["converged"]),
        "per_iter_ms": solve_ms / max(it, 1), "wall_s": wall,
    }


args_config_name = "C3"


# ------------------------------------------------------------- reference arm
def run_reference(args) -> None:
    """The reference's CPU implementation of the path (oracle/_ref: the
    unmodified reference solver with the 3D network restatement), each step a
    full measured time-to-solution on the B200 arm's config and weights. The
    steps run until --ref-budget-s is spent (at least one), so `steps` is the
    number actually timed. Nothing here loads the product library."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    global args_config_name
    args_config_name = args.config
    types, seed = workload(args)
    cores = os.cpu_count() or 1
    t_start = time.perf_counter()
    warm = []
    for _ in range(min(args.warmup, 1)):
        warm.append(cpu_reference_solve(types, seed, args.depth, cores, args.weights))
    vals, samples = [], []
    while len(vals) < args.steps:
        s = cpu_reference_solve(types, seed, args.depth, cores, args.weights)
        vals.append(s["value"])
        samples.append(s)
        if time.perf_counter() - t_start + s["wall_s"] > args.ref_budget_s:
            break
    v = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": 0, "steps": len(vals),
        "warmup": len(warm), "ms_per_step": v, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64 solver / f32 network", "data": "synthetic",
        "config": {"workload": f"{args.config} {types.shape[0]}^3 {scenes_module().DESCRIPTION[args.config]} "
                               "(SURVEY §8d), one frame per step: setup + PSDO to rel-res 1e-6",
                   "weights": args.weights, "depth": args.depth, "iterations": samples[-1]["iterations"],
                   "converged": all(x["converged"] for x in samples),
                   "steps_requested": args.steps, "warmup_requested": args.warmup,
                   "budget": f"full solves until {args.ref_budget_s:.0f} s are spent (at least one)"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "reference", "sample": samples[-1]["sample"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "per_iter_ms": float(np.mean([x["per_iter_ms"] for x in samples])),
        "setup_ms": float(np.mean([x["setup_ms"] for x in samples])),
        "step_ms": vals,
        "product_library_loaded": "libnpsd_b200" in Path("/proc/self/maps").read_text(),
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ C4 sequence
def sequence_c4(params, cfg, device: int, frames: int = 32, n: int = 128, repeats: int = 2) -> dict:
    """32 time-varying 128^3 masks (droplet falling into the
    pool), one context, per frame only set_mask + PSDO to 1e-6 (no re-setup),
    RHS seed 2000+f. Types and RHS of every frame resident in HBM; the whole
    sequence is timed with CUDA events on the context stream (host gaps between
    frames included)."""
    import paper_2310_00177_b200 as b200
    from paper_2310_00177_b200 import scenes

    ctx = b200.Context(3, (n, n, n), params, device=device)
    ts, bs = [], []
    for f, t in enumerate(scenes.droplet_frames(n, frames)):
        dt = b200.DeviceBuffer(ctx, t.size)
        db = b200.DeviceBuffer(ctx, 8 * t.size)
        dt.upload(np.ascontiguousarray(t.reshape(-1)))
        db.upload(scenes.full_rhs(t, 2000 + f, b200.rhs_normal))
        ts.append(dt)
        bs.append(db)
    dx = b200.DeviceBuffer(ctx, 8 * n ** 3)
    ctx.synchronize()
    best, iters, conv = None, [], []
    for rep_i in range(repeats + 1):  # first pass is warm-up
        it, cv = [], []
        ctx.event_record(0)
        for f in range(frames):
            ctx.set_mask_device(ts[f].ptr)
            rep = ctx.psdo_solve_device(bs[f].ptr, dx.ptr, cfg)
            it.append(int(rep.iterations))
            cv.append(bool(rep.converged))
        ctx.event_record(1)
        ms = ctx.event_elapsed_ms(0, 1)
        if rep_i and (best is None or ms < best):
            best, iters, conv = ms, it, cv
    for buf in ts + bs + [dx]:
        buf.free()
    ctx.close()
    return {"workload": f"C4: {frames} frames of {n}^3 droplet-in-pool, droplet centre y=(0.85-0.3f/31)n, "
                        "per-frame set_mask + PSDO to 1e-6, one context (no re-setup)",
            "total_ms": best, "ms_per_frame": best / frames, "frames_per_s": 1e3 * frames / best,
            "iterations": iters, "all_converged": all(conv), "repeats": repeats, "timing": "best of repeats"}


# ------------------------------------------------------------------ B200 arm
def timed_frames(ctx, d_types, d_b, d_x, cfg, steps: int, warmup: int, clk=None) -> dict:
    """W untimed frames, then K timed ones: set_mask + PSDO to 1e-6 per step
    between CUDA events on the context stream (inputs resident in HBM)."""
    def step():
        ctx.event_record(0)
        ctx.set_mask_device(d_types.ptr)
        rep = ctx.psdo_solve_device(d_b.ptr, d_x.ptr, cfg)
        ctx.event_record(1)
        return ctx.event_elapsed_ms(0, 1), rep, ctx.last_solve_ms

    for _ in range(warmup):
        step()
    ctx.synchronize()
    if clk:
        clk.start()
    launches0 = ctx.launch_count
    ms, iters, solve_ms, converged = [], [], [], []
    for _ in range(steps):
        t, rep, sm = step()
        ms.append(t)
        iters.append(rep.iterations)
        solve_ms.append(sm)
        converged.append(rep.converged)
    ctx.synchronize()
    out = {"launches": (ctx.launch_count - launches0) / steps, "clocks": clk.stop() if clk else None}
    out["step_ms"] = float(np.mean(ms))
    out["iterations"] = int(np.median(iters))
    out["converged"] = bool(all(converged))
    out["per_iter_ms"] = float(np.mean([s / max(i, 1) for s, i in zip(solve_ms, iters)]))
    out["set_mask_ms"] = out["step_ms"] - float(np.mean(solve_ms))
    return out


def iteration_roofline(depth: int, n_c: int, n_f: int, per_iter_ms: float, peaks: dict) -> dict:
    proc = sum(processed_bytes(depth, n_c, n_f).values())
    canon = sum(canonical_bytes_per_cell(depth).values()) * n_c
    gbs = proc / (per_iter_ms * 1e-3) / 1e9
    cgbs = canon / (per_iter_ms * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": gbs / peaks["hbm_gbs"], "bytes": proc,
            "bytes_model": "processed cells: solver vectors at fluid cells, coarse levels over all cells (DESIGN §4)",
            "canonical_achieved": cgbs, "canonical_frac": cgbs / peaks["hbm_gbs"],
            "canonical_bytes": f"SURVEY §8d B_iter = {canon / n_c:.2f} B x n_c (counts air/solid cells never read)",
            "peak_source": peaks["source"]}


def config_line(name: str, params, cfg, device: int, steps: int, warmup: int, cpu: bool) -> dict:
    """A secondary north_star config (C1 64^3, C2 128^3) measured the same way
    as the headline: TTS, per-iteration time, iteration roofline, and the
    reference CPU solve to convergence beside it."""
    import paper_2310_00177_b200 as b200

    types, seed = scenes_module().config(name)
    n_c, n_f = types.size, int((types == 0).sum())
    ctx = b200.Context(3, types.shape, params, device=device)
    d_types, d_b, d_x = b200.DeviceBuffer(ctx, n_c), b200.DeviceBuffer(ctx, 8 * n_c), b200.DeviceBuffer(ctx, 8 * n_c)
    d_types.upload(np.ascontiguousarray(types.reshape(-1)))
    d_b.upload(scenes_module().full_rhs(types, seed, b200.rhs_normal))
    ctx.synchronize()
    m = timed_frames(ctx, d_types, d_b, d_x, cfg, steps, warmup)
    for buf in (d_types, d_b, d_x):
        buf.free()
    ctx.close()
    out = {"workload": f"{name} {types.shape[0]}^3 {scenes_module().DESCRIPTION[name]} (SURVEY §8d)",
           "n_fluid": n_f, "tts_ms": m["step_ms"], "set_mask_ms": m["set_mask_ms"], "per_iter_ms": m["per_iter_ms"],
           "iterations": m["iterations"], "converged": m["converged"], "gpu_launches": int(round(m["launches"])),
           "steps": steps, "warmup": warmup,
           "iteration_roofline": iteration_roofline(params.depth, n_c, n_f, m["per_iter_ms"], load_peaks())}
    if cpu:
        c = cpu_reference_solve(types, seed, params.depth, os.cpu_count() or 1, "trained", name=name)
        out["cpu_baseline"] = {k: c[k] for k in ("value", "unit", "cores", "kind", "sample")}
    return out


def run_b200(args) -> None:
    import paper_2310_00177_b200 as b200

    global args_config_name
    args_config_name = args.config
    types, seed = workload(args)
    n_c = types.size
    n_f = int((types == 0).sum())
    depth = args.depth
    params = load_weights(args.weights, depth)
    ctx = b200.Context(3, types.shape, params, device=0)
    bfull = scenes_module().full_rhs(types, seed, b200.rhs_normal)
    cfg = b200.SolveConfig(tol_reduction=1e-6, max_iters=args.max_iters, n_ortho=2)

    # device-resident inputs
    d_types = b200.DeviceBuffer(ctx, n_c)
    d_b = b200.DeviceBuffer(ctx, 8 * n_c)
    d_x = b200.DeviceBuffer(ctx, 8 * n_c)
    d_types.upload(np.ascontiguousarray(types.reshape(-1)))
    d_b.upload(bfull)
    ctx.synchronize()
    m = timed_frames(ctx, d_types, d_b, d_x, cfg, args.steps, args.warmup, ClockSampler(0))
    step_ms, n_it, per_iter_ms = m["step_ms"], m["iterations"], m["per_iter_ms"]
    peaks = load_peaks()
    it_roof = iteration_roofline(depth, n_c, n_f, per_iter_ms, peaks)

    # per-kernel device times (kernels launched one by one between events)
    prof = ctx.profile_iterations(d_b.ptr, cfg, args.profile_iters)
    phase_ms: dict[str, float] = {}
    phase_kernels: dict[str, list] = {}
    for k, v in prof.items():
        ph = phase_of(k)
        phase_ms[ph] = phase_ms.get(ph, 0.0) + v
        phase_kernels.setdefault(ph, []).append(k)
    dom = max(phase_ms, key=phase_ms.get)
    dom_bytes = phase_bytes(processed_bytes(depth, n_c, n_f), dom)
    dom_canon = phase_bytes(canonical_bytes_per_cell(depth), dom) * n_c
    dom_gbs = dom_bytes / (phase_ms[dom] * 1e-3) / 1e9
    prof_total = sum(prof.values())
    dom_traffic = ncu_traffic(phase_kernels[dom], types.shape[0])

    # end to end through the public host API: pinned host inputs, H2D each step,
    # solution read back each step (host wall clock around the synchronous calls)
    p_types = b200.PinnedBuffer(ctx, n_c, np.uint8)
    p_b = b200.PinnedBuffer(ctx, n_f, np.float64)
    p_x = b200.PinnedBuffer(ctx, n_f, np.float64)
    p_types.array[:] = types.reshape(-1)
    p_b.array[:] = bfull[types.reshape(-1) == 0]
    e2e = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        ctx.set_mask(p_types.array)
        res = ctx.psdo_solve(p_b.array, cfg, out=p_x.array)
        t1 = time.perf_counter()
        if i >= args.warmup:
            e2e.append(1e3 * (t1 - t0))
    e2e_ms = float(np.mean(e2e))
    hist_bytes = 8 * (res.report.iterations + 1) * 2

    # the same frame with identity-equivalent weights (PSDO == CG, the network
    # still runs in full): what the trained model buys
    alt = {}
    if args.weights != "identity":
        ctx.set_params(b200.identity_params(depth))
        a = timed_frames(ctx, d_types, d_b, d_x, cfg, 1, 1)
        alt = {"weights": "identity", "tts_ms": a["step_ms"], "iterations": a["iterations"],
               "per_iter_ms": a["per_iter_ms"]}
        ctx.set_params(params)
        ctx.set_mask_device(d_types.ptr)

    # the paper's comparison columns on the same device and frame: GPU CG and
    # Jacobi-PCG (pcg_solve, solver.cpp:36-109), device-resident inputs. IC0-PCG
    # is parity-tested but not timed here: its level-scheduled sweeps (766
    # launches per apply at 256^3) are latency-bound by construction.
    baselines = {}
    for kind, name in (("identity", "gpu_cg"), ("jacobi", "gpu_pcg_jacobi")):
        ms_k, it_k = [], []
        for i in range(2):
            rep_k = ctx.pcg_solve_device(d_b.ptr, d_x.ptr, cfg, precond=kind)
            if i:
                ms_k.append(ctx.last_solve_ms)
                it_k.append(rep_k.iterations)
        baselines[name] = {"solve_ms": float(np.mean(ms_k)), "iterations": int(it_k[-1]),
                           "per_iter_ms": float(np.mean(ms_k)) / max(it_k[-1], 1), "converged": bool(rep_k.converged)}
    for buf in (d_types, d_b, d_x):
        buf.free()
    for buf in (p_types, p_b, p_x):
        buf.free()
    ctx.close()

    headline = args.config == "C3" and args.n is None
    seq = sequence_c4(params, cfg, 0) if headline and not args.no_sequence else None
    others = {}
    if headline and not args.no_configs:
        for name in ("C1", "C2"):
            others[name] = config_line(name, params, cfg, 0, args.steps, args.warmup, not args.no_cpu_baseline)

    cpu = None
    if not args.no_cpu_baseline:
        try:
            cpu = cpu_reference_solve(types, seed, depth, os.cpu_count() or 1, args.weights)
            cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    line = {
        "metric": METRIC, "value": step_ms, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64 solver / f32 network", "data": "synthetic",
        "config": {
            "workload": f"{args.config} {types.shape[0]}^3 {scenes_module().DESCRIPTION[args.config]} (SURVEY §8d), "
                        "one frame per step: set_mask + PSDO to rel-res 1e-6",
            "n_fluid": n_f, "depth": depth, "n_ortho": 2, "weights": args.weights,
            "iterations": n_it, "converged": m["converged"], "parallelism": "single",
            "l2": "inputs larger than L2 (solver vectors 8 B x n_c each, ~134 MB at 256^3, >= 126 MB L2)",
        },
        "per_iter_ms": per_iter_ms,
        "setup_ms": m["set_mask_ms"],
        "hbm_gbs_iteration": it_roof["achieved"],
        "iteration_roofline": it_roof,
        "roofline": {"bound": "hbm", "kernel": "+".join(phase_kernels[dom]), "phase": dom, "achieved": dom_gbs,
                     "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": dom_gbs / peaks["hbm_gbs"],
                     "traffic": dom_traffic,
                     "dram_gbs": (dom_traffic / (phase_ms[dom] * 1e-3) / 1e9) if dom_traffic else None,
                     "dram_frac": (dom_traffic / (phase_ms[dom] * 1e-3) / 1e9 / peaks["hbm_gbs"])
                     if dom_traffic else None,
                     "canonical_achieved": dom_canon / (phase_ms[dom] * 1e-3) / 1e9,
                     "canonical_frac": dom_canon / (phase_ms[dom] * 1e-3) / 1e9 / peaks["hbm_gbs"],
                     "note": "achieved/frac: algorithmic bytes over the cells the launch processes (fluid cells for "
                             "the solver vectors; DESIGN §4). canonical_*: SURVEY §8d bytes over every cell, "
                             "including air/solid cells the kernel never reads. dram_*: ncu-measured traffic "
                             "(profiles/ncu_traffic_<n>.json).",
                     "bytes_per_launch": dom_bytes, "ms_per_launch": phase_ms[dom],
                     "share_of_iteration": phase_ms[dom] / prof_total, "peak_source": peaks["source"]},
        "kernel_ms": prof,
        "e2e": {"value": e2e_ms, "unit": UNIT, "h2d_bytes_per_step": int(n_c + 8 * n_f),
                "d2h_bytes_per_step": int(8 * n_f + hist_bytes),
                "how": "Context.set_mask(pinned types) + Context.psdo_solve(pinned b) -> pinned x; host wall clock"},
        "gpu_launches": int(round(m["launches"])),
        "clocks": m["clocks"],
        "cpu_baseline": cpu,
        "baselines_same_gpu": baselines,
        "identity_weights_same_gpu": alt,
        "sequence_c4": seq,
        "configs": others,
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------- B200 arm, z-slab
def run_b200_slab(args, world: int, rank: int, local: int) -> None:
    import threading

    import torch
    import torch.distributed as dist  # plumbing: NCCL id broadcast, barrier, max over ranks (gloo)

    import paper_2310_00177_b200 as b200
    from paper_2310_00177_b200 import scenes

    # a rank that dies mid-collective must not hang the others forever
    def watchdog():
        time.sleep(args.watchdog_s)
        print(json.dumps({"error": f"rank {rank}: watchdog after {args.watchdog_s} s"}), flush=True)
        os._exit(3)

    threading.Thread(target=watchdog, daemon=True).start()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    os.environ.setdefault("RANK", str(rank))
    os.environ.setdefault("WORLD_SIZE", str(world))
    if not dist.is_initialized():
        dist.init_process_group("gloo")
    uid = [b200.Comm.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = b200.Comm.nccl(uid[0], rank, world, device=local)

    global args_config_name
    args_config_name = args.config
    types, seed = workload(args)
    nz, ny, nx = types.shape
    n_c = types.size
    depth = args.depth
    z0, nk = b200.partition(nz, world, depth)[rank]
    own = np.ascontiguousarray(types[z0:z0 + nk])
    params = load_weights(args.weights, depth)
    ctx = b200.Context.slab(comm, rank, types.shape, z0, nk, params, device=local)
    bfull = scenes.full_rhs(types, seed, b200.rhs_normal)
    bown = np.ascontiguousarray(bfull.reshape(nz, ny, nx)[z0:z0 + nk]).reshape(-1)
    cfg = b200.SolveConfig(tol_reduction=1e-6, max_iters=args.max_iters, n_ortho=2)
    d_types = b200.DeviceBuffer(ctx, own.size)
    d_b = b200.DeviceBuffer(ctx, bown.nbytes)
    d_x = b200.DeviceBuffer(ctx, bown.nbytes)
    d_types.upload(own.reshape(-1))
    d_b.upload(bown)
    ctx.synchronize()

    def step():
        ctx.event_record(0)
        ctx.set_mask_device(d_types.ptr)
        rep = ctx.psdo_solve_device(d_b.ptr, d_x.ptr, cfg)
        ctx.event_record(1)
        return ctx.event_elapsed_ms(0, 1), rep, ctx.last_solve_ms

    for _ in range(args.warmup):
        step()
    dist.barrier()
    ctx.synchronize()
    clk = ClockSampler(local)
    clk.start()
    launches0 = ctx.launch_count
    ms, iters, solve_ms, converged = [], [], [], []
    for _ in range(args.steps):
        t, rep, sm = step()
        ms.append(t)
        iters.append(rep.iterations)
        solve_ms.append(sm)
        converged.append(rep.converged)
    ctx.synchronize()
    launches = (ctx.launch_count - launches0) / args.steps
    clocks = clk.stop()

    def max_over_ranks(v: float) -> float:
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    step_ms = max_over_ranks(float(np.mean(ms)))
    per_iter_ms = max_over_ranks(float(np.mean([s / max(i, 1) for s, i in zip(solve_ms, iters)])))
    solve_mean = max_over_ranks(float(np.mean(solve_ms)))
    n_it = int(np.median(iters))

    # end to end through the host API on every rank: pinned owned types and
    # owned fluid entries in, owned solution out
    n_f = int((own == 0).sum())
    p_types = b200.PinnedBuffer(ctx, own.size, np.uint8)
    p_b = b200.PinnedBuffer(ctx, n_f, np.float64)
    p_x = b200.PinnedBuffer(ctx, n_f, np.float64)
    p_types.array[:] = own.reshape(-1)
    p_b.array[:] = bown[own.reshape(-1) == 0]
    e2e = []
    for i in range(args.warmup + args.steps):
        dist.barrier()
        t0 = time.perf_counter()
        ctx.set_mask(p_types.array)
        res = ctx.psdo_solve(p_b.array, cfg, out=p_x.array)
        t1 = time.perf_counter()
        if i >= args.warmup:
            e2e.append(1e3 * (t1 - t0))
    e2e_ms = max_over_ranks(float(np.mean(e2e)))
    hist_bytes = 8 * (res.report.iterations + 1) * 2
    model = canonical_bytes_per_cell(depth)
    b_iter = sum(model.values()) * n_c  # whole grid, all ranks
    peaks = load_peaks()
    agg_gbs = b_iter / (per_iter_ms * 1e-3) / 1e9
    peak_all = world * peaks["hbm_gbs"]
    if rank == 0:
        line = {
            "metric": METRIC, "value": step_ms, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64 solver / f32 network", "data": "synthetic",
            "config": {
                "workload": f"{args.config} {nz}^3 (SURVEY §8d), one frame per step: set_mask + PSDO to rel-res 1e-6, "
                            f"z-slab sharded over {world} GPU(s)",
                "depth": depth, "n_ortho": 2, "weights": args.weights, "iterations": n_it,
                "converged": bool(all(converged)), "parallelism": f"zslab{world}",
                "slabs": b200.partition(nz, world, depth), "chunk_graphs": ctx.slab_graph,
                "l2": "inputs larger than L2 (solver vectors 8 B x n_c each)",
            },
            "per_iter_ms": per_iter_ms,
            "setup_ms": step_ms - solve_mean,
            "hbm_gbs_iteration": agg_gbs,
            "iteration_roofline": {"bound": "hbm", "achieved": agg_gbs, "peak": peak_all, "unit": "GB/s",
                                   "frac": agg_gbs / peak_all,
                                   "bytes": f"canonical B_iter = {sum(model.values()):.2f} B x n_c (SURVEY §8d), "
                                            "whole grid over all ranks",
                                   "peak_source": f"{world} x {peaks['source']}"},
            "roofline": {"bound": "hbm", "kernel": "whole iteration (all ranks)", "achieved": agg_gbs,
                         "peak": peak_all, "unit": "GB/s", "frac": agg_gbs / peak_all, "traffic": None,
                         "peak_source": f"{world} x {peaks['source']}"},
            "e2e": {"value": e2e_ms, "unit": UNIT, "h2d_bytes_per_step": int(own.size + 8 * n_f),
                    "d2h_bytes_per_step": int(8 * n_f + hist_bytes),
                    "how": "per rank: Context.set_mask(pinned owned types) + psdo_solve(pinned owned b) -> pinned x; "
                           "host wall clock, max over ranks (rank 0's slab bytes)"},
            "gpu_launches": int(round(launches)),
            "clocks": clocks,
            "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    for buf in (d_types, d_b, d_x):
        buf.free()
    for buf in (p_types, p_b, p_x):
        buf.free()
    ctx.close()
    dist.barrier()
    comm.close()
    dist.destroy_process_group()
    os._exit(0)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C3", choices=["C1", "C2", "C3", "C5"])
    ap.add_argument("--n", type=int, default=None, help="override the grid size of the config")
    ap.add_argument("--depth", type=int, default=None, help="network depth (default: the trained model's)")
    ap.add_argument("--weights", default="trained", choices=["trained", "identity", "random"])
    ap.add_argument("--max-iters", type=int, default=20000)
    ap.add_argument("--profile-iters", type=int, default=5)
    ap.add_argument("--ref-budget-s", type=float, default=300.0,
                    help="reference arm: full solves until this many seconds are spent (at least one)")
    ap.add_argument("--no-configs", action="store_true", help="skip the C1/C2 lines of the N=1 run")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sequence", action="store_true", help="skip the C4 32-frame 128^3 sequence")
    ap.add_argument("--slab", action="store_true", help="z-slab path even at N=1 (one-rank NCCL)")
    ap.add_argument("--watchdog-s", type=float, default=900.0)
    args = ap.parse_args()
    if args.depth is None:
        args.depth = model_depth() if args.weights == "trained" else 4
    if args.impl == "reference":
        run_reference(args)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.slab:
        run_b200_slab(args, world, int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")))
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
