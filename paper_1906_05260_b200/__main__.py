"""Command line driver on the B200 solver — the reference CLI's `run` and `bench` (vrod_main.cpp:45-158).

    python -m paper_1906_05260_b200 run  <scene.json | builtin:C1..C5> [--steps N] [--out DIR] [--deterministic]
    python -m paper_1906_05260_b200 bench <scene.json | builtin:C1..C5> [--steps N]
    (either: --exact-shape-matching, the bit-identical shape-matching path)

Scene files are the reference's schema-1 JSON (scene_json.py). `builtin:` names the benchmark
workloads of this repository (workloads.CONFIGS); the reference's own builtin scenarios are its
workload source, not part of the solver path. `run` writes metrics.csv and probes.csv in the
reference's format (metrics.py); `bench` prints cmd_bench's lines with the per-phase device times
(phase timing on). There is no CPU path: without a B200 the solver raises DeviceError.
"""
from __future__ import annotations

import argparse
import os
import sys
import time


def resolve_scene(lib, arg: str):
    """resolve_scene, vrod_main.cpp:23-29."""
    from . import workloads
    from .scene_json import load_scene
    prefix = "builtin:"
    if arg.startswith(prefix):
        name = arg[len(prefix):]
        if name not in workloads.CONFIGS:
            raise SystemExit(f"unknown builtin scene '{name}' (known: {', '.join(sorted(workloads.CONFIGS))})")
        return workloads.CONFIGS[name](lib)
    return load_scene(lib, arg)


def run_scene(scene, out_dir: str, steps: int, deterministic: bool, exact: bool = False) -> int:
    """run_scene, vrod_main.cpp:45-101 (OBJ frames are out of scope)."""
    from . import Solver, SimulationError
    from .metrics import MetricsWriter, ProbeWriter
    scene.settings.deterministic = scene.settings.deterministic or deterministic
    os.makedirs(out_dir, exist_ok=True)
    solver = Solver(scene)
    if exact:
        solver.set_option("exact_shape_matching", 1)
    metrics = MetricsWriter(os.path.join(out_dir, "metrics.csv"), scene)
    probes = ProbeWriter(os.path.join(out_dir, "probes.csv"), scene)
    probes.write(0, solver.time(), solver.rod_state)
    singular = 0
    try:
        for _ in range(steps):
            try:
                report = solver.step()
            except SimulationError as e:
                print(f"simulation aborted at step {solver.step_index() + 1} (t={solver.time():.6g} s, "
                      f"{solver.dof_count()} DOFs): {e}", file=sys.stderr)
                return 1
            metrics.write(report, solver)
            probes.write(report.step, report.time, solver.rod_state)
            singular += report.skipped_singular
    finally:
        metrics.close()
        probes.close()
    if singular > 0:
        print(f"note: {singular} singular constraint solve(s) skipped", file=sys.stderr)
    print(f"wrote {os.path.join(out_dir, 'metrics.csv')} ({steps} steps, {solver.dof_count()} DOFs)")
    return 0


def cmd_bench(scene, steps: int, exact: bool = False) -> int:
    """cmd_bench, vrod_main.cpp:127-158, with device phase timings (StepReport.timings)."""
    from . import Solver, SimulationError
    solver = Solver(scene)
    solver.set_option("phase_timing", 1)
    if exact:
        solver.set_option("exact_shape_matching", 1)
    keys = ("predict_ms", "broad_ms", "narrow_ms", "solve_ms", "finalize_ms", "total_ms")
    total = dict.fromkeys(keys, 0.0)
    t0 = time.perf_counter()
    for _ in range(steps):
        try:
            report = solver.step()
        except SimulationError as e:
            print(f"simulation aborted at step {solver.step_index() + 1} (t={solver.time():.6g} s): {e}",
                  file=sys.stderr)
            return 1
        for k in keys:
            total[k] += report.timings[k]
    wall = time.perf_counter() - t0
    n = steps if steps > 0 else 1
    print(f"rods: {len(scene.rods)}, DOFs: {solver.dof_count()}")
    print(f"steps: {steps} in {wall:.3f} s -> {steps / wall if steps > 0 else 0.0:.1f} steps/s")
    print("per-step phase (ms): predict %.3f, broad %.3f, narrow %.3f, solve %.3f, finalize %.3f, total %.3f"
          % tuple(total[k] / n for k in keys))
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1906_05260_b200",
                                 description="tapered-capsule elastic rod simulator (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    run = sub.add_parser("run", help="simulate a scene, writing CSV metrics")
    run.add_argument("scene")
    run.add_argument("--steps", type=int, default=600)
    run.add_argument("--out", default="out")
    run.add_argument("--deterministic", action="store_true")
    bench = sub.add_parser("bench", help="measure stepping throughput")
    bench.add_argument("scene")
    bench.add_argument("--steps", type=int, default=100)
    for p in (run, bench):  # shape matching in the reference's exact operation order (bit-identical results)
        p.add_argument("--exact-shape-matching", action="store_true")
    args = ap.parse_args(argv)
    if args.steps < 0:
        ap.error("--steps must be non-negative")
    from . import library
    from .scene_json import SceneParseError
    lib = library()
    try:
        scene = resolve_scene(lib, args.scene)
    except SceneParseError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    if args.cmd == "run":
        return run_scene(scene, args.out, args.steps, args.deterministic, args.exact_shape_matching)
    return cmd_bench(scene, args.steps, args.exact_shape_matching)


if __name__ == "__main__":
    sys.exit(main())
