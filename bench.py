#!/usr/bin/env python
"""bench.py — neural-preconditioned PSDO ("DCDM") time-to-solution on B200.

Metric (BASELINE.json): time-to-solution in ms to relative residual 1e-6 at
256^3 (config C3: free-surface droplet-in-pool), plus per-
iteration ms and HBM GB/s. One step = one frame: set_mask (flags, coarsened
masks, mixed-window kernel tables, linear-block coefficients) + the whole PSDO
solve to 1e-6, with the cell types and the RHS already resident in HBM.
Weights: the repo's trained 3D model (weights/npsd3d_L4.npm) by
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
def workload(args):
    from paper_2310_00177_b200 import scenes

    types, seed = scenes.config(args.config, args.n)
    return types, seed


WEIGHTS = ROOT / "paper_2310_00177_b200" / "weights" / "npsd3d_L4.npm"


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


def iteration_count_fixture(config: str, weights: str = "identity") -> int | None:
    p = ROOT / "tests" / "golden" / "iteration_counts.json"
    key = f"{config}_trained" if weights == "trained" else config
    if p.exists():
        d = json.loads(p.read_text())
        if key in d:
            return int(d[key]["iterations"])
    return None


# ------------------------------------------------------------- CPU legs
def cpu_reference_sample(types, seed, depth, iters_to_solution, sample_iters, cores, weights="identity"):
    """Reference psdo_solve (oracle/_ref: the unmodified reference solver,
    assembly and reduce, with the 3D network restatement as its
    Preconditioner) on a bounded sample: full setup + `sample_iters` PSDO
    iterations on the same 256^3 frame. Time-to-solution = setup +
    iterations-to-solution x measured per-iteration time."""
    os.environ["OMP_NUM_THREADS"] = str(cores)
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import Ref  # checker / baseline only

    ref = Ref()
    import paper_2310_00177_b200 as b200

    p = load_weights(weights, depth).flat
    b = ref.rhs_normal(seed, types.size)[types.reshape(-1) == 0]
    t0 = time.perf_counter()
    r = ref.psdo_solve(types, b, mode="neural", params=p, depth=depth, max_iters=sample_iters,
                       tol_reduction=1e-300)
    wall = time.perf_counter() - t0
    per_iter_ms = 1e3 * r["solve_seconds"] / sample_iters
    setup_ms = 1e3 * r["setup_seconds"]
    return {
        "value": setup_ms + iters_to_solution * per_iter_ms,
        "unit": UNIT,
        "cores": cores,
        "kind": "reference",
        "sample": (f"{types.shape[0]}^3 {args_config_name}, {weights} weights: reference assemble_poisson_3d+reduce+"
                   "NeuralPrecond3D setup "
                   f"({setup_ms:.0f} ms) + {sample_iters} PSDO iterations ({per_iter_ms:.1f} ms/iter); TTS = setup + "
                   f"{iters_to_solution} iterations x per-iter (extrapolated); {wall:.1f} s wall"),
        "setup_ms": setup_ms,
        "per_iter_ms": per_iter_ms,
    }


args_config_name = "C3"


# ------------------------------------------------------------- reference arm
def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    global args_config_name
    args_config_name = args.config
    types, seed = workload(args)
    n_iters = iteration_count_fixture(args.config, args.weights) if args.n is None else None
    if n_iters is None:
        n_iters = args.ref_iters
    cores = os.cpu_count() or 1
    vals, samples = [], []
    for step in range(args.warmup + args.steps):
        s = cpu_reference_sample(types, seed, args.depth, n_iters, args.cpu_sample_iters, cores, args.weights)
        if step >= args.warmup:
            vals.append(s["value"])
            samples.append(s)
    v = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": 0, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": v, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64 solver / f32 network", "data": "synthetic",
        "config": {"workload": f"{args.config} {types.shape[0]}^3 (SURVEY §8d)", "weights": args.weights,
                   "depth": args.depth, "iterations_to_solution": n_iters,
                   "iterations_source": "tests/golden/iteration_counts.json (reference psdo_solve run to 1e-6 with "
                                        "the same weights)"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": samples[-1]["sample"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "per_iter_ms": float(np.mean([s["per_iter_ms"] for s in samples])),
        "setup_ms": float(np.mean([s["setup_ms"] for s in samples])),
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
def run_b200(args) -> None:
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist  # plumbing only: barrier + max over ranks (CPU/gloo)

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo")
    import paper_2310_00177_b200 as b200
    from paper_2310_00177_b200 import scenes

    global args_config_name
    args_config_name = args.config
    types, seed = workload(args)
    n_c = types.size
    depth = args.depth
    params = load_weights(args.weights, depth)
    ctx = b200.Context(3, types.shape, params, device=local)
    bfull = scenes.full_rhs(types, seed, b200.rhs_normal)
    cfg = b200.SolveConfig(tol_reduction=1e-6, max_iters=args.max_iters, n_ortho=2)

    # device-resident inputs
    d_types = b200.DeviceBuffer(ctx, n_c)
    d_b = b200.DeviceBuffer(ctx, 8 * n_c)
    d_x = b200.DeviceBuffer(ctx, 8 * n_c)
    d_types.upload(np.ascontiguousarray(types.reshape(-1)))
    d_b.upload(bfull)
    ctx.synchronize()

    def step():
        ctx.event_record(0)
        ctx.set_mask_device(d_types.ptr)
        rep = ctx.psdo_solve_device(d_b.ptr, d_x.ptr, cfg)
        ctx.event_record(1)
        return ctx.event_elapsed_ms(0, 1), rep, ctx.last_solve_ms

    for _ in range(args.warmup):
        step()
    if dist:
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
    step_ms = float(np.mean(ms))
    if dist:
        import torch

        t = torch.tensor([step_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_ms = float(t.item())
    n_it = int(np.median(iters))
    per_iter_ms = float(np.mean([s / max(i, 1) for s, i in zip(solve_ms, iters)]))
    setup_ms = step_ms - float(np.mean(solve_ms))
    model = canonical_bytes_per_cell(depth)
    b_iter = sum(model.values()) * n_c
    peaks = load_peaks()
    iter_gbs = b_iter / (per_iter_ms * 1e-3) / 1e9

    # per-kernel device times (kernels launched one by one between events)
    prof = ctx.profile_iterations(d_b.ptr, cfg, args.profile_iters)
    phase_ms: dict[str, float] = {}
    phase_kernels: dict[str, list] = {}
    for k, v in prof.items():
        ph = phase_of(k)
        phase_ms[ph] = phase_ms.get(ph, 0.0) + v
        phase_kernels.setdefault(ph, []).append(k)
    dom = max(phase_ms, key=phase_ms.get)
    dom_bytes = model.get(dom, 0.0) * n_c
    dom_gbs = dom_bytes / (phase_ms[dom] * 1e-3) / 1e9
    prof_total = sum(prof.values())
    dom_traffic = ncu_traffic(phase_kernels[dom], types.shape[0])

    # end to end through the public host API: pinned host inputs, H2D each step,
    # solution read back each step (host wall clock around the synchronous calls)
    n_f = int((types == 0).sum())
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
    if dist:
        import torch

        t = torch.tensor([e2e_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # the same frame with identity-equivalent weights (PSDO == CG, the network
    # still runs in full): what the trained model buys
    alt = {}
    if args.weights != "identity":
        ctx.set_params(b200.identity_params(depth))
        t_alt = [step() for _ in range(2)][-1]
        alt = {"weights": "identity", "tts_ms": t_alt[0], "iterations": int(t_alt[1].iterations),
               "per_iter_ms": t_alt[2] / max(t_alt[1].iterations, 1)}
        ctx.set_params(params)
        ctx.set_mask_device(d_types.ptr)

    # the paper's comparison columns on the same device and frame: GPU CG,
    # Jacobi-PCG and IC0-PCG (pcg_solve, solver.cpp:36-109), device-resident inputs
    baselines = {}
    for kind, name in (("identity", "gpu_cg"), ("jacobi", "gpu_pcg_jacobi"), ("ic0", "gpu_pcg_ic0")):
        ms_k, it_k = [], []
        for i in range(2):
            rep_k = ctx.pcg_solve_device(d_b.ptr, d_x.ptr, cfg, precond=kind)
            if i:
                ms_k.append(ctx.last_solve_ms)
                it_k.append(rep_k.iterations)
        baselines[name] = {"solve_ms": float(np.mean(ms_k)), "iterations": int(it_k[-1]),
                           "per_iter_ms": float(np.mean(ms_k)) / max(it_k[-1], 1), "converged": bool(rep_k.converged)}
    baselines["gpu_pcg_ic0"]["note"] = ("IC0 factor (per solve, level-scheduled) outside solve_ms; each apply is two "
                                        "sweeps of one launch per hyperplane x+y+z=h (766 at 256^3)")

    seq = None
    if world == 1 and args.config == "C3" and args.n is None and not args.no_sequence:
        seq = sequence_c4(params, cfg, local)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference_sample(types, seed, depth, n_it, args.cpu_sample_iters, os.cpu_count() or 1,
                                       args.weights)
            cpu.pop("setup_ms", None)
            cpu.pop("per_iter_ms", None)
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": step_ms, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64 solver / f32 network", "data": "synthetic",
            "config": {
                "workload": f"{args.config} {types.shape[0]}^3 droplet-in-pool (SURVEY §8d), one frame per step: "
                            "set_mask + PSDO to rel-res 1e-6",
                "n_fluid": n_f, "depth": depth, "n_ortho": 2, "weights": args.weights,
                "iterations": n_it, "converged": bool(all(converged)),
                "parallelism": "replicas" if world > 1 else "single",
                "l2": "inputs larger than L2 (solver vectors 8 B x n_c each, ~134 MB at 256^3, >= 126 MB L2)",
            },
            "per_iter_ms": per_iter_ms,
            "setup_ms": setup_ms,
            "hbm_gbs_iteration": iter_gbs,
            "iteration_roofline": {"bound": "hbm", "achieved": iter_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                                   "frac": iter_gbs / peaks["hbm_gbs"],
                                   "bytes": f"canonical B_iter = {sum(model.values()):.2f} B x n_c (SURVEY §8d)",
                                   "peak_source": peaks["source"]},
            "roofline": {"bound": "hbm", "kernel": "+".join(phase_kernels[dom]), "phase": dom, "achieved": dom_gbs,
                         "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": dom_gbs / peaks["hbm_gbs"],
                         "traffic": dom_traffic,
                         "dram_gbs": (dom_traffic / (phase_ms[dom] * 1e-3) / 1e9) if dom_traffic else None,
                         "dram_frac": (dom_traffic / (phase_ms[dom] * 1e-3) / 1e9 / peaks["hbm_gbs"])
                         if dom_traffic else None,
                         "note": "achieved/frac use SURVEY §8d's canonical bytes, which count every cell; the kernel "
                                 "skips air/solid cells (exact zeros, never read), so its DRAM traffic is below the "
                                 "model and frac can exceed 1. dram_gbs/dram_frac use the ncu-measured traffic.",
                         "bytes_per_launch": dom_bytes, "ms_per_launch": phase_ms[dom],
                         "share_of_iteration": phase_ms[dom] / prof_total, "peak_source": peaks["source"],
                         "bytes_model": f"SURVEY §8d canonical {model[dom]:.3f} B/cell x {n_c} cells ({dom})"},
            "kernel_ms": prof,
            "e2e": {"value": e2e_ms, "unit": UNIT, "h2d_bytes_per_step": int(n_c + 8 * n_f),
                    "d2h_bytes_per_step": int(8 * n_f + hist_bytes),
                    "how": "Context.set_mask(pinned types) + Context.psdo_solve(pinned b) -> pinned x; host wall clock"},
            "gpu_launches": int(round(launches)),
            "clocks": clocks,
            "cpu_baseline": cpu,
            "baselines_same_gpu": baselines,
            "identity_weights_same_gpu": alt,
            "sequence_c4": seq,
        }
        print(json.dumps(line), flush=True)
    for buf in (d_types, d_b, d_x):
        buf.free()
    for buf in (p_types, p_b, p_x):
        buf.free()
    ctx.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


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
    ap.add_argument("--depth", type=int, default=4)
    ap.add_argument("--weights", default="trained", choices=["trained", "identity", "random"])
    ap.add_argument("--max-iters", type=int, default=20000)
    ap.add_argument("--profile-iters", type=int, default=5)
    ap.add_argument("--cpu-sample-iters", type=int, default=2)
    ap.add_argument("--ref-iters", type=int, default=1000, help="iterations-to-solution if no fixture exists")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sequence", action="store_true", help="skip the C4 32-frame 128^3 sequence")
    ap.add_argument("--slab", action="store_true", help="z-slab path even at N=1 (one-rank NCCL)")
    ap.add_argument("--watchdog-s", type=float, default=900.0)
    args = ap.parse_args()
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
