"""The C++ drop-in (include/vrod/b200_solver.h): the reference's own proj/tests/test_solver.cpp and a
cmd_bench loop (vrod_main.cpp:127-158), compiled against vrod::b200::Solver and linked with
libvrod_b200.so (integration/Makefile).

CPU: the binaries build from the reference's sources (when /root/reference is present), link the
product library, and refuse to run without a device (no CPU fallback).
GPU: test_solver.cpp's solver-level cases pass and fail exactly as they do on the reference's own
CPU solver (oracle/_ref/vrod_ref_tests: the reference has five failing checks of its own in that file,
SURVEY.md §4), and every builtin scenario stepped through the facade equals the reference's
vrod::Solver bit for bit.
"""
from __future__ import annotations

import os
import re
import subprocess

import pytest

from conftest import ROOT

BUILD = os.path.join(ROOT, "integration", "_build")
TESTS_BIN = os.path.join(BUILD, "vrod_b200_solver_tests")
BENCH_BIN = os.path.join(BUILD, "vrod_b200_bench")
REF_TESTS = os.path.join(ROOT, "oracle", "_ref", "vrod_ref_tests")
HAVE_REFERENCE = os.path.isdir("/root/reference/proj")

# test_solver.cpp cases that exercise free functions (predict_rod, warm_start_lbs), not the Solver
# class: the drop-in replaces the class, so these stay the reference's and are not run here.
FREE_FUNCTION_CASES = ("predict_rod applies", "warm_start_lbs advances")
EXCLUDE = [f"-tce={c}" for c in FREE_FUNCTION_CASES]


def _gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="module")
def built():
    if HAVE_REFERENCE:
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref", "_ref/vrod_ref_tests"], check=True,
                       stdout=subprocess.DEVNULL)
        subprocess.run(["make", "-C", os.path.join(ROOT, "integration")], check=True, stdout=subprocess.DEVNULL)
    if not (os.path.exists(TESTS_BIN) and os.path.exists(BENCH_BIN)):
        pytest.skip("drop-in binaries not built (needs /root/reference at build time)")
    return True


def test_dropin_links_the_product_library(built):
    for b in (TESTS_BIN, BENCH_BIN):
        out = subprocess.run(["ldd", b], capture_output=True, text=True).stdout
        assert re.search(r"libvrod_b200\.so => .*paper_1906_05260_b200/lib/libvrod_b200\.so", out), out


@pytest.mark.skipif(_gpu_available(), reason="checks the no-device behaviour")
def test_dropin_fails_loudly_without_a_device(built):
    r = subprocess.run([BENCH_BIN, "builtin:floor", "--steps", "1"], capture_output=True, text=True, timeout=120)
    assert r.returncode != 0
    assert "CUDA" in r.stderr


def failures(output: str, path_part: str = "test_solver.cpp") -> set:
    """(line, case) of every failed check in a doctest-shim run, restricted to one test file."""
    out = set()
    for m in re.finditer(r"^(\S+):(\d+): FAILED in \"([^\"]+)\"", output, re.M):
        if path_part in m.group(1) and not any(c in m.group(3) for c in FREE_FUNCTION_CASES):
            out.add((int(m.group(2)), m.group(3)))
    return out


@pytest.mark.gpu
def test_reference_solver_suite_on_the_dropin(built):
    """proj/tests/test_solver.cpp, unmodified, with every Solver a vrod::b200::Solver on the B200:
    the same checks pass and the same checks fail as on the reference's own CPU solver."""
    got = subprocess.run([TESTS_BIN, *EXCLUDE], capture_output=True, text=True, timeout=600)
    assert "unexpected exception" not in got.stdout, got.stdout[-3000:]
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", got.stdout)
    assert m and int(m.group(1)) == 12, got.stdout[-2000:]
    ref = subprocess.run([REF_TESTS], capture_output=True, text=True, timeout=600)
    assert failures(got.stdout) == failures(ref.stdout), (got.stdout[-3000:], sorted(failures(ref.stdout)))


SCENARIOS = [("floor", 60, []), ("stretch", 60, []), ("wave", 60, []), ("activation", 60, []), ("bergou", 60, []),
             ("bergou_baseline", 60, []), ("band", 30, ["--exact"]), ("bench", 10, [])]


@pytest.mark.gpu
@pytest.mark.parametrize("name,steps,extra", SCENARIOS, ids=[s[0] for s in SCENARIOS])
def test_builtin_scenarios_bitwise_through_the_facade(built, name, steps, extra):
    """cmd_bench on the drop-in: the reference's builtin scene stepped by vrod::b200::Solver and by
    vrod::Solver; every state double equal after the run."""
    r = subprocess.run([BENCH_BIN, f"builtin:{name}", "--steps", str(steps), "--impl", "both", *extra],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "parity: bitwise" in r.stdout, r.stdout
    assert re.search(r"\[b200\] steps: \d+ in [\d.]+ s", r.stdout)
