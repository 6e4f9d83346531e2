#!/usr/bin/env python
"""Benchmark of the VIPER rod-solver substep on B200 (BASELINE.json metric).

Headline workload: C3, the paper-scale ~26k-DOF synthetic muscle bundle:
4 muscles x 32 rods x 30 vertices, shape matching (120 groups), pill-pill contacts between
muscles, activation; default settings (dt 1/60, 1 substep, 20 iterations) — so one step is one
substep is one frame. `value` = substeps/s with the state resident in HBM, every step a CUDA-
graph replay timed with CUDA events, L2 flushed (256 MiB memset, untimed) between steps.
`e2e` = the same through the public C-ABI (`vrod_solver_step` + a host read of centers, scales
and frames every step, pinned animation-packet upload inside). vs_baseline = value / 140 Hz
(the paper's 26k DOFs at 140 Hz on a GTX 1080).

Secondary: C4, the 1M-vertex rod forest with dense pill contacts (vertex-iters/s and the
per-substep HBM roofline of SURVEY.md §8(d)).

Multi-GPU: one process per GPU (torchrun); each rank steps its own independent C3 scene
(replicas / weak scaling, no inter-GPU collective on the data path); the timed region is
bracketed by barriers and the max over ranks is reported.

Batch (`batch` key): C5, 8192 independent C3 scenes split into contiguous shards over the
ranks (strong scaling), each shard stepped as one device world; per-scene stats are
all-gathered to rank 0 over NCCL at the end — the only collective.

`--impl reference` times the reference's own CPU implementation (oracle/_ref: the reference's
sources compiled against the Eigen shim; else the oracle restatement) on all host threads.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PAPER_HZ = 140.0          # PAPER.md:100 (26k DOFs at 140 Hz, GTX 1080)
L2_FLUSH_BYTES = 256 << 20
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libvrod_ref.so")
ORACLE_LIB = os.path.join(ROOT, "oracle", "lib", "libvrod_oracle.so")


def dist_info():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu capture (profiles/r01_traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_traffic.json")) as f:
            return json.load(f)[kernel]["bytes"]
    except Exception:
        return None


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + ",".join(self.FIELDS),
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) == len(self.FIELDS):
                    rows.append(parts)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        smax = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[2 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows)}


def bind_bench(lib):
    lib.vrod_bench_run.restype = C.c_int
    lib.vrod_bench_run.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
    lib.vrod_bench_kernel_times.restype = C.c_int
    lib.vrod_bench_kernel_times.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
    lib.vrod_bench_last_counts.restype = C.c_int
    lib.vrod_bench_last_counts.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    return lib


CATS = ["predict", "collide", "ext_setup", "ext_solve", "rod_sweep", "shape", "report", "iterate"]


def device_run(lib, solver, steps, flush):
    from paper_1906_05260_b200.scene import check
    ms = C.c_double()
    kern = C.c_int64()
    check(lib, lib.vrod_bench_run(solver._h, steps, flush, C.byref(ms), C.byref(kern)))
    return ms.value, kern.value


def kernel_times(lib, solver, steps):
    from paper_1906_05260_b200.scene import check
    ms = (C.c_double * len(CATS))()
    ln = (C.c_int64 * len(CATS))()
    check(lib, lib.vrod_bench_kernel_times(solver._h, steps, ms, ln))
    return {CATS[i]: (ms[i], ln[i]) for i in range(len(CATS))}


def cpu_sample(lib_path, build_scene, target_s, threads, max_steps=200):
    """Time the CPU implementation at `lib_path` on its own copy of the scene for ~target_s."""
    from paper_1906_05260_b200 import capi
    from paper_1906_05260_b200.handle import SolverHandle
    env_threads = os.environ.get("VROD_THREADS")
    os.environ["VROD_THREADS"] = str(threads)
    lib = capi.bind(C.CDLL(lib_path))
    h = SolverHandle(lib, build_scene(lib))
    h.step()  # warm-up
    n, t0 = 0, time.perf_counter()
    while n < max_steps and (time.perf_counter() - t0) < target_s:
        h.step()
        n += 1
    dt = time.perf_counter() - t0
    if env_threads is None:
        os.environ.pop("VROD_THREADS", None)
    else:
        os.environ["VROD_THREADS"] = env_threads
    return n, dt


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU implementation on the host threads (the fastest
    count of a short sweep), rank 0 only."""
    if rank != 0:
        return
    from paper_1906_05260_b200 import capi, workloads
    from paper_1906_05260_b200.handle import SolverHandle
    # The reference's CPU path is timed through its bitwise-identical restatement (oracle/, "port")
    # on all host threads: the reference's own block-solve threads (VROD_THREADS > 1, parallel.h)
    # crash on the `static thread_local` update buffer of jacobi_sweep (constraints.cpp:497-500:
    # resized on the calling thread only), and oracle/_ref — the reference's sources compiled
    # here — links an Eigen SUBSET SHIM whose dynamic-shape matrices run ~5-10x slower than
    # Eigen's fixed-size expressions, so it would understate the reference's speed.
    # The restatement runs the reference's parallel_for over the block solves (VROD_THREADS).
    # VROD_REF_IMPL=shim times oracle/_ref instead (1 thread).
    # The reference's parallel_for starts its workers per sweep (parallel.h:27-46), so on a host
    # with many cores the thread count that is fastest is found by a short sweep (one step each)
    # rather than assumed to be all of them.
    if os.environ.get("VROD_REF_IMPL") == "shim" and os.path.exists(REF_LIB):
        kind, path, cands = "reference", REF_LIB, [1]
    else:
        ncpu = os.cpu_count() or 1
        kind, path, cands = "port", ORACLE_LIB, sorted({t for t in (1, 2, 4, 8, 16, 32, 64, ncpu) if t <= ncpu})
    lib = capi.bind(C.CDLL(path))
    scene = workloads.c3_muscle_bundle(lib)
    sweep = {}
    base = SolverHandle(lib, scene)  # advance past the contact-free start: later frames cost more
    for _ in range(6):
        base.step()
    st = base.state()
    for t in cands:  # the same two frames from the same advanced state for every candidate
        os.environ["VROD_THREADS"] = str(t)
        hs = SolverHandle(lib, scene)
        for _ in range(6):
            hs.step()
        hs.set_state(**st)
        t0 = time.perf_counter()
        hs.step()
        hs.step()
        sweep[t] = time.perf_counter() - t0
        hs.close()
    base.close()
    h = SolverHandle(lib, scene)
    threads = min(sweep, key=sweep.get)
    os.environ["VROD_THREADS"] = str(threads)
    for _ in range(min(args.warmup, 3)):
        h.step()
    t0 = time.perf_counter()
    done = 0
    while done < args.steps and (done == 0 or time.perf_counter() - t0 < args.ref_seconds):
        h.step()
        done += 1
    dt = time.perf_counter() - t0
    args.steps = done  # bounded sample: at most --ref-seconds of CPU work
    substeps = scene.settings.substeps
    value = done * substeps / dt
    line = {"metric": "substeps/sec", "value": value, "unit": "substeps/s", "impl": "reference",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": value / PAPER_HZ, "dtype": "f64",
            "data": "synthetic", "config": {"workload": "C3 muscle bundle 4x32x30 (26,496 DOF), 20 iterations",
                                            "rods": len(scene.rods), "dof": h.dof_count()},
            "cpu_baseline": {"value": value, "unit": "substeps/s", "cores": threads, "kind": kind,
                             "sample": f"{args.steps} C3 frames after {args.warmup} warm-up, VROD_THREADS={threads} "
                                       f"(fastest of {sorted(sweep)} over two frames after six), {os.path.basename(path)}"},
            "e2e": {"value": value, "unit": "substeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-secondary", action="store_true", help="skip the C4 1M-vertex measurement")
    ap.add_argument("--secondary-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-seconds", type=float, default=90.0, help="cap of the --impl reference timed sample")
    ap.add_argument("--no-batch", action="store_true", help="skip the C5 sharded-batch measurement")
    ap.add_argument("--no-skin", action="store_true", help="skip the skinning (deform_mesh) measurement")
    ap.add_argument("--skin-rings", type=int, default=1000, help="skin mesh: rings x segments vertices")
    ap.add_argument("--batch-scenes", type=int, default=8192, help="C5 batch size, sharded over the ranks")
    ap.add_argument("--batch-steps", type=int, default=3)
    args = ap.parse_args()
    rank, world, local = dist_info()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    args.warmup = max(args.warmup, 3)
    if world > 1:
        # one process per GPU: pin this rank to its GPU before any CUDA runtime initialises
        # (the product library links its own static cudart)
        os.environ["CUDA_VISIBLE_DEVICES"] = str(local)

    import paper_1906_05260_b200 as pb
    from paper_1906_05260_b200 import workloads

    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist
        # host-side barrier / max-over-ranks only: the replicas exchange no data
        from datetime import timedelta
        tdist.init_process_group("gloo", timeout=timedelta(seconds=900))
        dist = (torch, tdist)

    lib = bind_bench(pb.library())
    scene = workloads.c3_muscle_bundle(lib)
    solver = pb.Solver(scene)
    S, I = scene.settings.substeps, scene.settings.iterations
    V, E = solver.total_vertices, solver.total_elements
    for _ in range(args.warmup):
        rep = solver.step()

    def barrier():
        if dist:
            dist[1].barrier()

    # ---- device-resident throughput (value) ----
    barrier()
    with ClockSampler(local) as clk:
        ms_total, kern = device_run(lib, solver, args.steps, L2_FLUSH_BYTES)
    barrier()
    if dist:
        t = dist[0].tensor([ms_total], dtype=dist[0].float64)
        dist[1].all_reduce(t, op=dist[1].ReduceOp.MAX)
        ms_total = float(t.item())
    clocks = clk.summary()
    value = world * args.steps * S / (ms_total / 1e3)

    # ---- end-to-end through the C-ABI with host buffers ----
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        rep = solver.step()
        st = solver.state()
    e2e_dt = time.perf_counter() - t0
    barrier()
    if dist:
        t = dist[0].tensor([e2e_dt], dtype=dist[0].float64)
        dist[1].all_reduce(t, op=dist[1].ReduceOp.MAX)
        e2e_dt = float(t.item())
    e2e_value = world * args.steps * S / e2e_dt
    vpad = max(32, (V + 31) // 32 * 32)
    h2d = 8 * S * (1 + 3 * 0 + len(scene.activations) + 14 * len(scene.bones) + 8 * len(scene.kinematic_pills))
    d2h = 8 * (8 + 7) * vpad + 160  # state + velocity fields of get_state, plus the StepReport

    # ---- C5: the 8192-scene batch sharded over the ranks (every rank takes part) ----
    batch = None
    if not args.no_batch:
        try:
            batch = run_c5(lib, args, rank, world, dist, barrier)
        except Exception as exc:  # report, do not lose the headline
            batch = {"error": f"{type(exc).__name__}: {exc}"}

    if rank != 0:
        if dist:
            dist[1].destroy_process_group()
        return

    # ---- per-kernel attribution and roofline. Dominant kernel: the persistent iteration kernel
    # k_iterate (all I sweeps + external blocks + shape matching of a substep in one launch) when
    # the world fits on chip (C3), else the per-sweep fused rod sweep k_rod_sweep ----
    kt = kernel_times(lib, solver, 5)
    peak, peak_kind = load_peaks()
    persistent = kt["iterate"][1] > 0
    sweep_ms, sweep_n = kt["iterate"] if persistent else kt["rod_sweep"]
    sweep_avg_s = sweep_ms / max(sweep_n, 1) / 1e3
    # read+write c,s (vertex) / q (element) per sweep; the persistent kernel runs I
    sweep_bytes = 64 * (V + E) * (I if persistent else 1)
    achieved = sweep_bytes / sweep_avg_s / 1e9
    total_dev_ms = sum(v[0] for v in kt.values())
    nc = rep.contact_count
    b_sub = workloads.algorithmic_bytes(V, E, I, True, E, nc)
    t_sub = ms_total / 1e3 / args.steps / S
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": load_traffic("k_iterate" if persistent else "k_rod_sweep"),
                "kernel": "k_iterate" if persistent else "k_rod_sweep", "bytes_per_launch": sweep_bytes,
                "avg_launch_us": sweep_avg_s * 1e6, "share_of_step": sweep_ms / total_dev_ms,
                "peak_source": peak_kind,
                "substep": {"algorithmic_bytes": b_sub, "seconds": t_sub, "achieved_gbs": b_sub / t_sub / 1e9,
                            "frac": b_sub / t_sub / 1e9 / peak}}
    breakdown = {k: {"ms_per_step": v[0] / 5, "launch_groups": v[1] // 5} for k, v in kt.items()}

    # ---- CPU baseline: the oracle restatement, single thread, bounded sample ----
    n_cpu, dt_cpu = cpu_sample(ORACLE_LIB, workloads.c3_muscle_bundle, args.cpu_seconds, 1)
    cpu = {"value": n_cpu * S / dt_cpu, "unit": "substeps/s", "cores": 1, "kind": "port",
           "sample": f"{n_cpu} C3 frames ({dt_cpu:.1f} s) of oracle/vrod_oracle.cpp (bitwise equal to the "
                     f"reference), 1 thread"}

    line = {"metric": "substeps/sec", "value": value, "unit": "substeps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": value / world / PAPER_HZ, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C3 muscle bundle 4x32x30 rods (26,496 DOF), 120 shape-match groups, "
                                   "inter-muscle pill contacts, activation; dt 1/60, 1 substep, 20 iterations",
                       "rods": len(scene.rods), "vertices": V, "dof": solver.dof_count(),
                       "contacts_last_step": nc, "l2": "256 MiB memset between timed steps (untimed)",
                       "parallelism": f"replicas x{world}"},
            "frames_per_sec": value / world, "vertex_iters_per_sec": value * V * I,
            "e2e": {"value": e2e_value, "unit": "substeps/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": int(kern) * args.steps, "kernels_per_step": int(kern),
            "roofline": roofline, "breakdown": breakdown, "cpu_baseline": cpu, "clocks": clocks}

    if batch is not None:
        line["batch"] = batch
    if not args.no_secondary:
        try:
            line["secondary"] = run_c4(lib, args.secondary_steps, peak)
        except Exception as exc:  # report, do not lose the headline
            line["secondary"] = {"error": f"{type(exc).__name__}: {exc}"}
    if not args.no_skin:
        try:
            line["skin"] = run_skin(lib, solver, peak, args.cpu_seconds)
        except Exception as exc:  # report, do not lose the headline
            line["skin"] = {"error": f"{type(exc).__name__}: {exc}"}
    print(json.dumps(line), flush=True)
    if dist:
        dist[1].destroy_process_group()


def run_c5(lib, args, rank, world, dist, barrier):
    """C5: `--batch-scenes` independent C3 scenes, contiguous shard per rank, each shard ONE device
    world; timed with CUDA events (max over ranks); per-scene stats all-gathered to rank 0 at the
    end (NCCL when N > 1) — the only inter-GPU traffic."""
    import paper_1906_05260_b200 as pb
    from paper_1906_05260_b200 import batch as pbatch
    from paper_1906_05260_b200 import workloads
    n_total = args.batch_scenes
    lo, hi = workloads.shard_range(n_total, rank, world)
    t0 = time.perf_counter()
    solver = pb.BatchSolver(workloads.c5_batch(lib, hi - lo, first=lo))
    setup_s = time.perf_counter() - t0
    scene0 = workloads.c5_scene(lib, lo)
    S, I = scene0.settings.substeps, scene0.settings.iterations
    solver.step()  # warm-up (captures the graph)
    barrier()
    ms, kern = device_run(lib, solver, args.batch_steps, 0)  # >= 3.9M vertices per GPU: working set >> L2
    barrier()
    if dist:
        t = dist[0].tensor([ms], dtype=dist[0].float64)
        dist[1].all_reduce(t, op=dist[1].ReduceOp.MAX)
        ms = float(t.item())
    rows = pbatch.report_rows(solver.scene_reports())
    if dist:
        torch, tdist = dist
        nccl = tdist.new_group(backend="nccl")
        table = pbatch.gather_scene_stats(rows, n_total, device=torch.device("cuda", 0), group=nccl)
    else:
        table = rows
    t_step = ms / 1e3 / args.batch_steps
    V = solver.total_vertices
    out = {"workload": f"C5 batch of {n_total} independent C3 scenes (28 distinct), contiguous shard per GPU, "
                       f"one device world per shard",
           "scenes": n_total, "scenes_per_gpu": hi - lo, "vertices_per_gpu": V, "steps": args.batch_steps,
           "ms_per_step": t_step * 1e3, "scene_substeps_per_sec": n_total * S / t_step,
           "vertex_iters_per_sec": V * world * I * S / t_step, "setup_s": setup_s, "kernels_per_step": int(kern),
           "scaling": "strong (fixed 8192-scene batch split over the GPUs)",
           "stats_gather": "NCCL all_gather of per-scene stats" if dist else "single GPU"}
    if table is not None:
        out["gathered"] = {"scenes": int(table.shape[0]), "contacts": int(table[:, 9].sum()),
                           "broad_pairs": int(table[:, 10].sum()), "max_penetration": float(table[:, 8].max())}
    del solver
    return out


def run_skin(lib, solver, peak, cpu_seconds, rings=1000, segments=1000, k=8, iters=50):
    """Skinning, the consumer of every frame: a rings x segments sleeve
    mesh (1M vertices) bound to the C3 solver's 3,712 rest pills (top-8 inverse-square weights,
    one smoothing pass), then per frame the solver's pill transforms + deform_mesh on the device.
    Algorithmic bytes per vertex: rest 24 + CSR offset 4 + k x (pill 4 + weight 8) + out 24; the
    3,712 x 128 B pill transform tables stay in L2."""
    import paper_1906_05260_b200 as pb
    from paper_1906_05260_b200 import workloads
    from paper_1906_05260_b200.handle import Skin as SkinHandle
    lib.vrod_bench_skin_deform.restype = C.c_int
    lib.vrod_bench_skin_deform.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(C.c_double),
                                           C.POINTER(C.c_double)]
    pills, rest = solver.rest_pills(), solver.rest_pill_transforms()
    V, T = workloads.sleeve_mesh(pills, rings, segments)
    t0 = time.perf_counter()
    sk = pb.Skin(V, T, pills, rest, max_influences=k)
    bind_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    sk.smooth(1)
    smooth_s = time.perf_counter() - t0
    nnz = len(sk.binding()["pills"])
    nv = V.shape[0]
    tot, dfm = C.c_double(), C.c_double()
    lib.vrod_bench_skin_deform(sk._h, solver._h, 3, C.byref(tot), C.byref(dfm))  # warm-up
    from paper_1906_05260_b200.scene import check
    check(lib, lib.vrod_bench_skin_deform(sk._h, solver._h, iters, C.byref(tot), C.byref(dfm)))
    frame_s = tot.value / 1e3 / iters
    deform_s = dfm.value / 1e3
    bytes_v = (24 + 4 + 24) * nv + 12 * nnz
    t0 = time.perf_counter()
    for _ in range(10):
        sk.deform_solver(solver)
    e2e_s = (time.perf_counter() - t0) / 10
    # CPU baseline: the oracle restatement's deform_mesh (1 thread) on a 250x250 sleeve
    orc = capi_bind_oracle()
    hv, ht = workloads.sleeve_mesh(pills, 250, 250)
    osk = SkinHandle(orc, hv, ht, pills, rest, k)
    cur = solver.pill_transforms()
    n_cpu, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < min(cpu_seconds, 5.0):
        osk.deform(cur)
        n_cpu += 1
    cpu_vps = n_cpu * hv.shape[0] / (time.perf_counter() - t0)
    return {"workload": f"sleeve mesh {rings}x{segments} ({nv:,} vertices, {len(T):,} triangles) bound to the C3 "
                        f"rest pills ({len(pills):,}), top-{k} weights, 1 smoothing pass; per frame: pill transforms "
                        "+ deform_mesh",
            "vertices_per_sec": nv / frame_s, "ms_per_frame": frame_s * 1e3, "bind_s": bind_s, "smooth_s": smooth_s,
            "influences": nnz,
            "roofline": {"bound": "hbm", "kernel": "k_skin_deform", "bytes_per_launch": bytes_v,
                         "avg_launch_us": deform_s * 1e6, "achieved": bytes_v / deform_s / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": bytes_v / deform_s / 1e9 / peak,
                         "traffic": load_traffic("k_skin_deform")},
            "e2e": {"value": nv / e2e_s, "unit": "vertices/s", "d2h_bytes_per_frame": 24 * nv},
            "cpu_baseline": {"value": cpu_vps, "unit": "vertices/s", "cores": 1, "kind": "port",
                             "sample": f"{n_cpu} deform_mesh calls of a 250x250 sleeve (oracle restatement)"}}


def capi_bind_oracle():
    from paper_1906_05260_b200 import capi
    return capi.bind(C.CDLL(ORACLE_LIB))


def run_c4(lib, steps, peak):
    import paper_1906_05260_b200 as pb
    from paper_1906_05260_b200 import workloads
    t0 = time.perf_counter()
    scene = workloads.c4_rod_forest(lib)
    solver = pb.Solver(scene)
    setup_s = time.perf_counter() - t0
    S, I = scene.settings.substeps, scene.settings.iterations
    V, E = solver.total_vertices, solver.total_elements
    for _ in range(2):
        rep = solver.step()
    ms, kern = device_run(lib, solver, steps, 0)  # 1M vertices: working set >> L2
    t_sub = ms / 1e3 / steps / S
    kt = kernel_times(lib, solver, 1)
    sweep_ms, sweep_n = kt["rod_sweep"]
    sweep_avg = sweep_ms / max(sweep_n, 1) / 1e3
    nc = rep.contact_count
    b_sub = workloads.algorithmic_bytes(V, E, I, True, E, nc)
    return {"workload": "C4 rod forest 125x250 rods x 32 vertices (1,000,000 vertices), dense pill contacts, "
                        "dt 1/240, 10 iterations",
            "vertex_iters_per_sec": V * I * S / t_sub, "substeps_per_sec": 1.0 / t_sub, "ms_per_substep": t_sub * 1e3,
            "contacts": nc, "broad_pairs": rep.broad_pairs, "steps": steps, "setup_s": setup_s,
            "roofline_substep": {"algorithmic_bytes": b_sub, "achieved_gbs": b_sub / t_sub / 1e9, "peak": peak,
                                 "frac": b_sub / t_sub / 1e9 / peak},
            "rod_sweep": {"avg_launch_us": sweep_avg * 1e6, "bytes_per_launch": 64 * (V + E),
                          "achieved_gbs": 64 * (V + E) / sweep_avg / 1e9, "traffic": load_traffic("k_rod_sweep"),
                          "traffic_gbs": (load_traffic("k_rod_sweep") or 0) / sweep_avg / 1e9},
            "breakdown_ms_per_step": {k: v[0] for k, v in kt.items()}, "kernels_per_step": int(kern)}


if __name__ == "__main__":
    main()
