"""jacobi_sweep and eval_constraint at the unit level (constraints.h), the way test_sweep.cpp and
test_constraints.cpp drive them: one sweep of a solver's elastic blocks and soft pins with zero
multipliers, and the residual W of every elastic block, on the live state.

CPU: the restatement equals the reference (oracle/_ref) bit for bit. GPU: the product equals the
restatement bit for bit (the sweep kernels keep the reference's operation order, --fmad=false).
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_1906_05260_b200.handle import SolverHandle
from paper_1906_05260_b200.scene import SimulationError

from scenes import SCENES

UNIT_SCENES = ("C1", "floor", "stretch", "activation", "bergou", "bergou_baseline", "crossing", "kitchen_sink", "pile")


def sweep_flow(lib, name, sweeps=3):
    h = SolverHandle(lib, SCENES[name](lib))
    h.step()
    out = {"W0": h.elastic_residuals()}
    for k in range(sweeps):
        beta = 0.75 if k else 1.0
        out[f"outcome{k}"] = np.array(h.jacobi_sweep(1.0 / 60, beta))
        st = h.state()
        for key in ("centers", "scales", "frames"):
            out[f"{key}{k}"] = st[key]
        out[f"W{k + 1}"] = h.elastic_residuals()
    return out


def sweep_error(lib):
    h = SolverHandle(lib, SCENES["C1"](lib))
    c = h.state()["centers"].copy()
    c[5, 1] = np.nan
    h.set_state(centers=c)
    with pytest.raises(SimulationError) as e:
        h.jacobi_sweep(1.0 / 60, 0.75)
    return str(e.value)


@pytest.mark.parametrize("name", UNIT_SCENES)
def test_restatement_sweep_and_residuals_bitwise(ref, oracle, name):
    a, b = sweep_flow(ref, name), sweep_flow(oracle, name)
    for k in a:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)


def test_restatement_sweep_error_names_the_constraint(ref, oracle):
    assert sweep_error(ref) == sweep_error(oracle)
    assert sweep_error(oracle).startswith("non-finite update from constraint ")


def beta_linearity(lib):
    """test_sweep.cpp:68-79: the first Jacobi update of the centers is linear in beta."""
    d = []
    for beta in (0.25, 0.5):
        h = SolverHandle(lib, SCENES["C1"](lib))
        h.step()
        c0 = h.state()["centers"]
        h.jacobi_sweep(1.0 / 60, beta)
        d.append(h.state()["centers"] - c0)
    return d


def test_sweep_update_linear_in_beta(oracle):
    d1, d2 = beta_linearity(oracle)
    assert np.abs(d1).max() > 0
    np.testing.assert_allclose(d2, 2 * d1, rtol=1e-9, atol=1e-15)


@pytest.mark.gpu
@pytest.mark.parametrize("name", [n for n in UNIT_SCENES if n != "kitchen_sink"])  # no shape matching in step()
def test_gpu_sweep_and_residuals_bitwise(oracle, name):
    import paper_1906_05260_b200 as pb
    a, b = sweep_flow(pb.library(), name), sweep_flow(oracle, name)
    for k in a:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)


@pytest.mark.gpu
def test_gpu_sweep_update_linear_in_beta(oracle):
    import paper_1906_05260_b200 as pb
    for x, y in zip(beta_linearity(pb.library()), beta_linearity(oracle)):
        np.testing.assert_array_equal(x, y)


@pytest.mark.gpu
def test_gpu_sweep_error_names_the_constraint(oracle):
    import paper_1906_05260_b200 as pb
    assert sweep_error(pb.library()) == sweep_error(oracle)
