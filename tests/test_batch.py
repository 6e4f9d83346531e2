"""Batches of independent scenes (BASELINE config C5).

The reference has no batch API: a batch is N independent `vrod::Solver(Scene)` stepped in
lockstep. The oracle and the reference adapter implement it exactly so; the product steps the
whole batch as one device world. Every scene of a product batch must equal that scene solved
alone (bitwise on the exact scenes), and the per-scene StepReports must equal the scene's own.
The N>1 sharding (contiguous shards, stats all-gathered to rank 0) is exercised with gloo,
world size 2, on the CPU oracle.
"""
from __future__ import annotations

import copy
import os
import socket

import numpy as np
import pytest

from paper_1906_05260_b200 import batch as pbatch
from paper_1906_05260_b200 import workloads
from paper_1906_05260_b200.handle import SolverHandle

from scenes import SCENES


def variant(scene, k: int):
    """Scene copy with a scene-specific lateral push on every unpinned vertex."""
    s = copy.deepcopy(scene)
    for r, rod in enumerate(s.rods):
        free = rod.pinned == 0
        rod.state.center_vel[free, 0] += 0.05 * (k + 1) * np.cos(0.7 * r + k)
        rod.state.center_vel[free, 1] += 0.05 * (k + 1) * np.sin(0.7 * r + k)
    return s


def run_single(lib, scene, steps):
    h = SolverHandle(lib, scene)
    reps = [h.step() for _ in range(steps)]
    return h.state(), reps[-1]


def run_batch(lib, scenes, steps):
    h = SolverHandle.batch(lib, scenes)
    for _ in range(steps):
        total = h.step()
    return h, total, h.scene_reports()


def split_state(h, scenes, state):
    """Slice a batch's concatenated state back into per-scene states."""
    out, vo, eo = [], 0, 0
    for s in scenes:
        nv = sum(len(r.state.scales) for r in s.rods)
        ne = nv - len(s.rods)
        out.append({k: (v[vo:vo + nv] if k in ("centers", "scales", "center_vel", "scale_vel") else v[eo:eo + ne])
                    for k, v in state.items()})
        vo += nv
        eo += ne
    return out


def compare_reports(a, b, exact_residuals):
    assert a.contact_count == b.contact_count
    assert a.broad_pairs == b.broad_pairs
    assert a.skipped_singular == b.skipped_singular
    assert a.max_penetration == b.max_penetration
    assert a.dof_count == b.dof_count
    if exact_residuals:
        np.testing.assert_array_equal(a.residuals, b.residuals)
    else:  # the product reduces each scene's norms in its own tree
        np.testing.assert_allclose(a.residuals, b.residuals, rtol=1e-12, atol=1e-300)


def check_batch_against_singles(lib, scenes, steps, exact_residuals):
    h, total, reps = run_batch(lib, scenes, steps)
    states = split_state(h, scenes, h.state())
    assert len(reps) == len(scenes)
    for i, s in enumerate(scenes):
        st, rep = run_single(lib, s, steps)
        for k in st:
            np.testing.assert_array_equal(states[i][k], st[k], err_msg=f"scene {i} {k}")
        compare_reports(reps[i], rep, exact_residuals)
    assert total.contact_count == sum(r.contact_count for r in reps)
    assert total.broad_pairs == sum(r.broad_pairs for r in reps)
    assert total.max_penetration == max(r.max_penetration for r in reps)


# ---- CPU: oracle / reference adapter ---------------------------------------------------------

@pytest.mark.parametrize("name", ["pile", "crossing"])
def test_oracle_batch_is_independent_scenes(oracle, name):
    base = SCENES[name](oracle)
    check_batch_against_singles(oracle, [variant(base, k) for k in range(3)], 2, exact_residuals=True)


def test_reference_batch_matches_oracle_batch(oracle, ref):
    base = SCENES["pile"](oracle)
    scenes = [variant(base, k) for k in range(2)]
    ho, _, ro = run_batch(oracle, scenes, 2)
    hr, _, rr = run_batch(ref, scenes, 2)
    for k, v in ho.state().items():
        np.testing.assert_array_equal(v, hr.state()[k], err_msg=k)
    for a, b in zip(ro, rr):
        compare_reports(a, b, exact_residuals=True)


def test_batch_rejects_mixed_settings(oracle):
    a = SCENES["pile"](oracle)
    b = copy.deepcopy(a)
    b.settings.iterations += 1
    from paper_1906_05260_b200.scene import InvalidArgument
    with pytest.raises(InvalidArgument, match="share one SolverSettings"):
        SolverHandle.batch(oracle, [a, b])


def test_shard_range_partitions():
    for n in (1, 7, 28, 8192):
        for world in (1, 2, 3, 4, 8):
            got = [workloads.shard_range(n, r, world) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(got[r][1] == got[r + 1][0] for r in range(world - 1))
            assert max(hi - lo for lo, hi in got) - min(hi - lo for lo, hi in got) <= 1


def test_c5_scenes_vary_by_index(oracle):
    scenes = workloads.c5_batch(oracle, 30)
    assert scenes[0] is scenes[28] and scenes[1] is scenes[29]
    assert scenes[0] is not scenes[1]
    v0 = scenes[0].rods[5].state.center_vel
    v1 = scenes[1].rods[5].state.center_vel
    assert not np.array_equal(v0, v1)
    assert len(scenes[0].activations) == 32  # one muscle activated


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shard_worker(rank, world, port, n_scenes, out_path):
    import ctypes as C

    import torch.distributed as dist

    from paper_1906_05260_b200 import capi
    from conftest import ORACLE_LIB
    from scenes import SCENES as S

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = capi.bind(C.CDLL(ORACLE_LIB))
    base = S["crossing"](lib)
    scenes = [variant(base, k) for k in range(n_scenes)]
    lo, hi = workloads.shard_range(n_scenes, rank, world)
    h = SolverHandle.batch(lib, scenes[lo:hi])
    h.step()
    h.step()
    table = pbatch.gather_scene_stats(pbatch.report_rows(h.scene_reports()), n_scenes)
    if rank == 0:
        np.save(out_path, table)
    dist.destroy_process_group()


def test_sharded_batch_gathers_stats_gloo(oracle, tmp_path):
    import torch.multiprocessing as mp

    n = 5
    out = str(tmp_path / "table.npy")
    mp.spawn(_shard_worker, args=(2, _free_port(), n, out), nprocs=2, join=True)
    table = np.load(out)
    base = SCENES["crossing"](oracle)
    h, _, reps = run_batch(oracle, [variant(base, k) for k in range(n)], 2)
    np.testing.assert_array_equal(table, pbatch.report_rows(reps))


# ---- GPU: the product's batch world ------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("name", ["pile", "crossing", "floor"])
def test_gpu_batch_equals_scenes_alone(name):
    import paper_1906_05260_b200 as pb
    lib = pb.library()
    base = SCENES[name](lib)
    check_batch_against_singles(lib, [variant(base, k) for k in range(3)], 3, exact_residuals=False)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["mini_muscle", "kitchen_sink"])
def test_gpu_batch_with_shape_matching_and_kinematics(name):
    import paper_1906_05260_b200 as pb
    lib = pb.library()
    base = SCENES[name](lib)
    check_batch_against_singles(lib, [variant(base, k) for k in range(2)] + [base], 2, exact_residuals=False)


@pytest.mark.gpu
def test_gpu_batch_matches_oracle_per_scene(oracle):
    import paper_1906_05260_b200 as pb
    lib = pb.library()
    base = SCENES["pile"](lib)
    scenes = [variant(base, k) for k in range(3)]
    h, _, reps = run_batch(lib, scenes, 3)
    ho, _, ro = run_batch(oracle, scenes, 3)
    for k, v in h.state().items():
        np.testing.assert_array_equal(v, ho.state()[k], err_msg=k)
    for a, b in zip(reps, ro):
        compare_reports(a, b, exact_residuals=False)


@pytest.mark.gpu
def test_gpu_c5_shard_equals_scenes_alone():
    import paper_1906_05260_b200 as pb
    lib = pb.library()
    scenes = workloads.c5_batch(lib, 3, first=5)
    check_batch_against_singles(lib, scenes, 2, exact_residuals=False)
