"""bench.py's multi-rank plumbing and reference arm, on CPU (no GPU needed).

`--gpus 2 --dry-run` goes through the same spawn (torch.distributed.run, two ranks), gloo
barriers, max over ranks and the C5 per-scene stats all-gather as a real multi-GPU run, with
synthetic per-scene rows tagged by scene index: rank 0 must receive all 8192 rows in scene order
and report n_gpus = 2. `--impl reference` must time the reference's CPU path (the restatement)
and report the thread sweep it chose from, never slower than its 1-thread sample.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

from conftest import ROOT


def run_bench(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_two_rank_dry_run_gathers_every_scene():
    line = run_bench("--gpus", "2", "--dry-run")
    assert line["dry_run"] is True
    assert line["n_gpus"] == 2 == line["gpus_requested"]
    assert line["batch"] == {"scenes": 8192, "gathered_rows": 8192, "scene_order": True, "backend": "gloo"}
    assert line["max_over_ranks"] == 0.002  # rank 1's value wins the max


def test_single_rank_dry_run():
    line = run_bench("--dry-run")
    assert line["n_gpus"] == 1 and line["batch"]["gathered_rows"] == 8192


def test_reference_arm_reports_its_thread_sweep(oracle):
    line = run_bench("--impl", "reference", "--steps", "2", "--warmup", "1", "--ref-seconds", "2")
    assert line["impl"] == "reference" and line["unit"] == "substeps/s" and line["warmup"] == 1
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["value"] == line["value"] == line["e2e"]["value"]
    assert line["value"] >= cb["sweep"]["1"]  # the fastest candidate, 1 thread included
    assert str(cb["cores"]) in cb["sweep"]
    assert line["host"]["nproc"] == os.cpu_count()
