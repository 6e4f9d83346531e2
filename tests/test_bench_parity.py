"""Parity at the benchmarked sizes: the scenes bench.py times, built exactly as
bench.py builds them, against the CPU oracle (the restatement, bitwise equal to the reference —
test_oracle_pinning) or, at C4, against digests of the reference's own output.

- C2 (64 rods x 256 vertices, stretched by pin motions; no contacts, no bundles): bitwise, K = 60.
- C3 (the 26k-DOF muscle bundle, shape matching + contacts), default (latency-tuned) shape
  matching: identical input -> one substep within 1e-10; free-running K = 10 within 1e-6 with the
  contact set (pill_a, pill_b) exact at every substep and alpha/beta within 1e-9. With the
  exact-order shape path (VROD_SHAPE_EXACT=1): bit for bit, K = 10. C3g (SURVEY's literal C3, gravity on, O(10^3) contacts) the same.
- C4 (1,000,000 vertices, ~2.8 M contacts): two substeps, every output array bit for bit
  (SHA-256 against tests/golden/c4_hashes.json, made by tests/golden/make_c4_hashes.py from
  oracle/_ref and the restatement).

Measured maxima are recorded in BASELINE.md §6; set VROD_PARITY_LOG=<path> to dump them as JSON.
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

import paper_1906_05260_b200 as pb
from paper_1906_05260_b200 import workloads
from paper_1906_05260_b200.handle import SolverHandle

HERE = os.path.dirname(os.path.abspath(__file__))
C4_HASHES = os.path.join(HERE, "golden", "c4_hashes.json")
MAXIMA: dict = {}


def rel_err(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b)))) if a.size else 0.0


def quat_err(a, b):
    if not a.size:
        return 0.0
    return float(np.max(np.minimum(np.linalg.norm(a - b, axis=1), np.linalg.norm(a + b, axis=1))))


def state_err(sg, so):
    return {"centers": rel_err(sg["centers"], so["centers"]), "scales": rel_err(sg["scales"], so["scales"]),
            "frames": quat_err(sg["frames"], so["frames"])}


@pytest.fixture(scope="module", autouse=True)
def _dump_maxima():
    yield
    path = os.environ.get("VROD_PARITY_LOG")
    if path and MAXIMA:
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        old = json.load(open(path)) if os.path.exists(path) else {}
        old.update(MAXIMA)
        with open(path, "w") as f:
            json.dump(old, f, indent=1)


@pytest.fixture(scope="module")
def gpu():
    return pb.library()


# ---- C2 --------------------------------------------------------------------------------------

@pytest.mark.gpu
def test_c2_full_size_bitwise(gpu, oracle):
    """C2 at 64 x 256 exactly as bench.py builds it: 60 substeps, every state bit equal."""
    scene = workloads.c2_stretch_grid(gpu)
    g, o = SolverHandle(gpu, scene), SolverHandle(oracle, scene)
    assert g.total_vertices == 16384
    for k in range(60):
        rg, ro = g.step(), o.step()
        assert (rg.contact_count, rg.broad_pairs, rg.skipped_singular) == (ro.contact_count, ro.broad_pairs,
                                                                          ro.skipped_singular), k
        np.testing.assert_allclose(rg.residuals, ro.residuals, rtol=1e-12, atol=0)
    sg, so = g.state(), o.state()
    for k in sg:
        np.testing.assert_array_equal(sg[k], so[k], err_msg=k)
    MAXIMA["C2"] = {"steps": 60, "bitwise": True}


# ---- C3 --------------------------------------------------------------------------------------

C3_VARIANTS = {
    "C3": lambda lib: workloads.c3_muscle_bundle(lib),
    "C3g": lambda lib: workloads.c3_muscle_bundle_gravity(lib),
}
ONE_SUBSTEP_TOL = 1e-10
FREE_TOL = 1e-6
AB_TOL = 1e-9


def _contacts_match(g, o, where):
    cg, co = g.contacts(), o.contacts()
    np.testing.assert_array_equal(cg["pill_a"], co["pill_a"], err_msg=where)
    np.testing.assert_array_equal(cg["pill_b"], co["pill_b"], err_msg=where)
    if not len(cg["alpha"]):
        return 0.0
    return float(max(np.abs(cg["alpha"] - co["alpha"]).max(), np.abs(cg["beta"] - co["beta"]).max()))


@pytest.mark.gpu
@pytest.mark.parametrize("variant", sorted(C3_VARIANTS))
def test_c3_exact_mode_bitwise(oracle, variant, monkeypatch):
    """VROD_SHAPE_EXACT=1 (shape.cuh shape_group_exact): the C3 scenes bench.py times are
    bit-identical to the oracle (= the reference) for K = 10 substeps: states, velocities,
    contacts with alpha/beta, counters, penetration."""
    monkeypatch.setenv("VROD_SHAPE_EXACT", "1")
    lib = pb.library()
    scene = C3_VARIANTS[variant](lib)
    g, o = SolverHandle(lib, scene), SolverHandle(oracle, scene)
    for k in range(10):
        rg, ro = g.step(), o.step()
        assert (rg.contact_count, rg.broad_pairs, rg.skipped_singular, rg.max_penetration) == \
               (ro.contact_count, ro.broad_pairs, ro.skipped_singular, ro.max_penetration), (variant, k)
        cg, co = g.contacts(), o.contacts()
        for key in cg:
            np.testing.assert_array_equal(cg[key], co[key], err_msg=f"{variant} substep {k}: {key}")
        sg, so = g.state(), o.state()
        for key in sg:
            np.testing.assert_array_equal(sg[key], so[key], err_msg=f"{variant} substep {k}: {key}")
    MAXIMA[f"{variant}_exact"] = {"steps": 10, "bitwise": True}


@pytest.mark.gpu
@pytest.mark.parametrize("variant", sorted(C3_VARIANTS))
def test_c3_bench_scene_parity(gpu, oracle, variant):
    """The C3 scene bench.py times: one substep from identical input within 1e-10; free-running
    K = 10 within 1e-6, contact ids exact every substep, alpha/beta within 1e-9; then one substep
    from the oracle's state written into the GPU solver (resync) within 1e-10."""
    scene = C3_VARIANTS[variant](gpu)
    g, o = SolverHandle(gpu, scene), SolverHandle(oracle, scene)
    assert g.dof_count() == 26496
    rec = {"one_substep": None, "free": [], "resync": None, "contacts": []}
    MAXIMA[variant] = rec  # filled as the run goes, so a failing run still reports its maxima
    ab_max = 0.0
    for k in range(10):
        rg, ro = g.step(), o.step()
        assert (rg.contact_count, rg.broad_pairs) == (ro.contact_count, ro.broad_pairs), (variant, k)
        ab_max = max(ab_max, _contacts_match(g, o, f"{variant} substep {k}"))
        e = state_err(g.state(), o.state())
        rec["free"].append(e)
        rec["contacts"].append(rg.contact_count)
        rec["alpha_beta_max"] = ab_max
        if k == 0:
            rec["one_substep"] = e
    # resync: the oracle's state into the GPU solver, one more substep each
    g.set_state(**o.state())
    rg, ro = g.step(), o.step()
    assert rg.contact_count == ro.contact_count
    _contacts_match(g, o, f"{variant} resync")
    rec["resync"] = state_err(g.state(), o.state())
    assert max(rec["one_substep"].values()) <= ONE_SUBSTEP_TOL, rec["one_substep"]
    assert ab_max <= AB_TOL
    assert max(rec["free"][-1].values()) <= FREE_TOL, rec["free"][-1]
    assert max(rec["resync"].values()) <= ONE_SUBSTEP_TOL, rec["resync"]


# ---- C4 --------------------------------------------------------------------------------------

def _c4_golden():
    if not os.path.exists(C4_HASHES):
        pytest.skip("tests/golden/c4_hashes.json not generated")
    return json.load(open(C4_HASHES))


def test_c4_golden_digests_reference_equals_restatement():
    """The committed C4 digests come from the reference (oracle/_ref) and the restatement; both
    must describe the same bits (CPU check of the fixture itself)."""
    data = _c4_golden()
    assert "oracle" in data
    if "ref" not in data:
        pytest.skip("reference digests not generated")
    for a, b in zip(data["ref"]["steps"], data["oracle"]["steps"]):
        assert a["sha256"] == b["sha256"]
        assert (a["contact_count"], a["broad_pairs"], a["max_penetration"]) == \
               (b["contact_count"], b["broad_pairs"], b["max_penetration"])


@pytest.mark.gpu
def test_c4_full_size_bitwise_digests(gpu, oracle):
    """C4 at 1,000,000 vertices, two substeps: every state array, velocity array and the ordered
    contact set (pill ids, alpha, beta) hash to the reference's digests; counters and penetration
    equal."""
    data = _c4_golden()
    want = data["ref"]["steps"] if "ref" in data else data["oracle"]["steps"]
    from golden.make_c4_hashes import scene_builder, step_record
    g = SolverHandle(gpu, scene_builder(oracle))
    assert g.total_vertices == 1_000_000
    for k, exp in enumerate(want):
        rep = g.step()
        got = step_record(g, rep)
        for key in ("contact_count", "broad_pairs", "skipped_singular", "max_penetration", "time", "step"):
            assert got[key] == exp[key], (k, key, got[key], exp[key])
        bad = {a: (got["sample"][a], exp["sample"][a]) for a in exp["sha256"] if got["sha256"][a] != exp["sha256"][a]}
        assert not bad, f"substep {k}: digests differ for {sorted(bad)}; samples (gpu, ref): {bad}"
        # residual RMS: the GPU sums the 7.6 M block norms in per-CTA trees, the reference
        # sequentially; the rounding difference grows with the count (measured 6e-12 here)
        np.testing.assert_allclose(got["residuals"], exp["residuals"], rtol=1e-10, atol=0)
    MAXIMA["C4"] = {"substeps": len(want), "bitwise": True, "contacts": [s["contact_count"] for s in want]}
