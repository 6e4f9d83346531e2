"""Solver handle over any library exporting include/vrod_capi.h.

`SolverHandle` is the Python face of `vrod::Solver` (solver.h:54-115): construct from a Scene,
`step()`, state access in DofLayout global-slot order, loads, energy queries, contacts, pills,
probe_convergence. The product's `paper_1906_05260_b200.Solver` is this class bound to the
CUDA library; tests bind the same class to the CPU oracle libraries to compare.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import capi
from .scene import InvalidArgument, Scene, check, marshal_scene

KIND_NAMES = ("stretch_z", "cross_section", "surface_stretch", "bend_twist", "surface_bending",
              "volume_stretch", "volume_bend_u", "volume_bend_v")


@dataclass
class StepReport:
    """StepReport, solver.h:23-33 (+ PhaseTimings :14-21)."""
    step: int
    time: float
    residuals: np.ndarray
    max_penetration: float
    contact_count: int
    broad_pairs: int
    skipped_singular: int
    dof_count: int
    timings: dict

    @staticmethod
    def from_c(r: capi.StepReport) -> "StepReport":
        return StepReport(step=r.step, time=r.time, residuals=np.array(r.residuals[:], dtype=np.float64),
                          max_penetration=r.max_penetration, contact_count=r.contact_count,
                          broad_pairs=r.broad_pairs, skipped_singular=r.skipped_singular, dof_count=r.dof_count,
                          timings=dict(predict_ms=r.predict_ms, broad_ms=r.broad_ms, narrow_ms=r.narrow_ms,
                                       solve_ms=r.solve_ms, finalize_ms=r.finalize_ms, total_ms=r.total_ms))


class SolverHandle:
    def __init__(self, lib, scene: Scene | None, *, _batch: list[Scene] | None = None):
        self._lib = lib
        self._h = C.c_void_p()
        if _batch is None:
            sh = marshal_scene(lib, scene)
            try:
                check(lib, lib.vrod_solver_create(sh, C.byref(self._h)))
            finally:
                lib.vrod_scene_destroy(sh)
        else:
            # a Scene object repeated in the batch is marshalled once and referenced again
            unique: dict[int, C.c_void_p] = {}
            try:
                for s in _batch:
                    if id(s) not in unique:
                        unique[id(s)] = marshal_scene(lib, s)
                arr = (C.c_void_p * len(_batch))(*[unique[id(s)].value for s in _batch])
                check(lib, lib.vrod_batch_create(len(_batch), arr, C.byref(self._h)))
            finally:
                for h in unique.values():
                    lib.vrod_scene_destroy(h)
        n = C.c_int32()
        check(lib, lib.vrod_solver_scene_count(self._h, C.byref(n)))
        self.scene_count = n.value
        info = self.info()
        self.rod_count = info.rod_count
        self.total_vertices = info.total_vertices
        self.total_elements = info.total_elements
        sizes = np.zeros(max(self.rod_count, 1), dtype=np.int32)
        check(lib, lib.vrod_solver_get_rod_sizes(self._h, capi.ptr(sizes, C.c_int32)))
        self.rod_sizes = sizes[: self.rod_count].astype(np.int64)
        self.vertex_base = np.concatenate([[0], np.cumsum(self.rod_sizes)])[:-1] if self.rod_count else np.zeros(0)
        self.element_base = self.vertex_base - np.arange(self.rod_count)

    @classmethod
    def batch(cls, lib, scenes: list[Scene]) -> "SolverHandle":
        """A batch of independent scenes stepped together (vrod_batch_create, BASELINE C5)."""
        return cls(lib, None, _batch=list(scenes))

    def scene_reports(self) -> list[StepReport]:
        """Per-scene StepReports of the last step (vrod_solver_scene_reports)."""
        arr = (capi.StepReport * self.scene_count)()
        check(self._lib, self._lib.vrod_solver_scene_reports(self._h, self.scene_count, arr))
        return [StepReport.from_c(r) for r in arr]

    # -- lifetime -------------------------------------------------------------------------------
    def close(self) -> None:
        if self._h:
            self._lib.vrod_solver_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def backend(self) -> str:
        return self._lib.vrod_backend_name().decode()

    # -- product options (vrod_solver_set_option) ----------------------------------------------
    def set_option(self, name: str, value: int | bool) -> None:
        """"state_prefetch", "exact_shape_matching" or "phase_timing" (include/vrod_capi.h)."""
        check(self._lib, self._lib.vrod_solver_set_option(self._h, name.encode(), int(value)))

    # -- stepping -------------------------------------------------------------------------------
    def step(self) -> StepReport:
        """Solver::step(), solver.cpp:363-388."""
        r = capi.StepReport()
        check(self._lib, self._lib.vrod_solver_step(self._h, C.byref(r)))
        return StepReport.from_c(r)

    def probe_convergence(self, iterations: int) -> np.ndarray:
        """Solver::probe_convergence, solver.cpp:390-398 -> (iterations, 8) residual log."""
        out = np.zeros((max(iterations, 1), 8))
        check(self._lib, self._lib.vrod_solver_probe_convergence(self._h, iterations, capi.ptr(out)))
        return out[:iterations]

    # -- queries --------------------------------------------------------------------------------
    def info(self) -> capi.SolverInfo:
        i = capi.SolverInfo()
        check(self._lib, self._lib.vrod_solver_get_info(self._h, C.byref(i)))
        return i

    def time(self) -> float:
        return self.info().time

    def step_index(self) -> int:
        return self.info().step_index

    def dof_count(self) -> int:
        return self.info().dof_count

    def state(self) -> dict:
        """Live state, global slot order: centers (V,3), scales (V,), frames (E,4) wxyz, velocities."""
        V, E = self.total_vertices, self.total_elements
        buf = np.empty(8 * V + 7 * E)  # one allocation, six views (the C-ABI's packed layout)
        o = (0, 3 * V, 4 * V, 4 * V + 4 * E, 7 * V + 4 * E, 8 * V + 4 * E, 8 * V + 7 * E)
        out = dict(centers=buf[o[0]:o[1]].reshape(V, 3), scales=buf[o[1]:o[2]], frames=buf[o[2]:o[3]].reshape(E, 4),
                   center_vel=buf[o[3]:o[4]].reshape(V, 3), scale_vel=buf[o[4]:o[5]],
                   angular_vel=buf[o[5]:o[6]].reshape(E, 3))
        check(self._lib, self._lib.vrod_solver_get_state(
            self._h, capi.ptr(out["centers"]), capi.ptr(out["scales"]), capi.ptr(out["frames"]),
            capi.ptr(out["center_vel"]), capi.ptr(out["scale_vel"]), capi.ptr(out["angular_vel"])))
        return out

    def set_state(self, centers=None, scales=None, frames=None, center_vel=None, scale_vel=None,
                  angular_vel=None) -> None:
        """Write back into the live scene between steps (Solver::scene() mutation)."""
        def p(a, shape):
            if a is None:
                return None
            x = np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(shape))
            keep.append(x)
            return capi.ptr(x)

        keep: list = []
        V, E = self.total_vertices, self.total_elements
        check(self._lib, self._lib.vrod_solver_set_state(
            self._h, p(centers, (V, 3)), p(scales, (V,)), p(frames, (E, 4)), p(center_vel, (V, 3)),
            p(scale_vel, (V,)), p(angular_vel, (E, 3))))

    def rod_state(self, r: int) -> dict:
        st = self.state()
        v0, n = int(self.vertex_base[r]), int(self.rod_sizes[r])
        e0 = int(self.element_base[r])
        return dict(centers=st["centers"][v0:v0 + n], scales=st["scales"][v0:v0 + n],
                    frames=st["frames"][e0:e0 + n - 1], center_vel=st["center_vel"][v0:v0 + n],
                    scale_vel=st["scale_vel"][v0:v0 + n], angular_vel=st["angular_vel"][e0:e0 + n - 1])

    def rest(self) -> dict:
        """Live rest data per element slot (activation rewrites it): lengths, darboux, grads, laplacians."""
        E = self.total_elements
        out = dict(lengths=np.zeros(E), darboux=np.zeros((E, 3)), scale_grads=np.zeros(E),
                   scale_laplacians=np.zeros(E))
        check(self._lib, self._lib.vrod_solver_get_rest(self._h, capi.ptr(out["lengths"]), capi.ptr(out["darboux"]),
                                                        capi.ptr(out["scale_grads"]),
                                                        capi.ptr(out["scale_laplacians"])))
        return out

    def set_loads(self, force_density=None, torque=None, scale_load=None, force_rods=None, torque_rods=None,
                  scale_load_rods=None) -> None:
        """Solver::loads() (ExternalLoads, solver.h:35-41) as global arrays + optional per-rod masks."""
        keep: list = []

        def p(a, shape, ct=C.c_double, dt=np.float64):
            if a is None:
                return None
            x = np.ascontiguousarray(np.asarray(a, dtype=dt).reshape(shape))
            keep.append(x)
            return capi.ptr(x, ct)

        V, E, R = self.total_vertices, self.total_elements, self.rod_count
        check(self._lib, self._lib.vrod_solver_set_loads(
            self._h, p(force_density, (V, 3)), p(force_rods, (R,), C.c_uint8, np.uint8), p(torque, (E, 3)),
            p(torque_rods, (R,), C.c_uint8, np.uint8), p(scale_load, (E,)),
            p(scale_load_rods, (R,), C.c_uint8, np.uint8)))

    def kinetic_energy(self) -> float:
        x = C.c_double()
        check(self._lib, self._lib.vrod_solver_energy(self._h, C.byref(x), None, None))
        return x.value

    def total_volume(self) -> float:
        x = C.c_double()
        check(self._lib, self._lib.vrod_solver_energy(self._h, None, C.byref(x), None))
        return x.value

    def total_rest_volume(self) -> float:
        x = C.c_double()
        check(self._lib, self._lib.vrod_solver_energy(self._h, None, None, C.byref(x)))
        return x.value

    def inverse_weights(self) -> dict:
        V, E = self.total_vertices, self.total_elements
        out = dict(inv_center=np.zeros(V), inv_scale=np.zeros(V), inv_theta=np.zeros((E, 3)))
        check(self._lib, self._lib.vrod_solver_get_inverse_weights(
            self._h, capi.ptr(out["inv_center"]), capi.ptr(out["inv_scale"]), capi.ptr(out["inv_theta"])))
        return out

    def weights(self) -> dict:
        """DofLayout lumped weights (layout.h:25-27): +inf for pinned vertices; theta as of the last substep."""
        V, E = self.total_vertices, self.total_elements
        out = dict(center_weight=np.zeros(V), scale_weight=np.zeros(V), theta_weight=np.zeros((E, 3)))
        check(self._lib, self._lib.vrod_solver_get_weights(
            self._h, capi.ptr(out["center_weight"]), capi.ptr(out["scale_weight"]), capi.ptr(out["theta_weight"])))
        return out

    def contacts(self) -> dict:
        n = C.c_int64()
        check(self._lib, self._lib.vrod_solver_get_contacts(self._h, 0, C.byref(n), None, None, None, None))
        k = n.value
        out = dict(pill_a=np.zeros(k, dtype=np.int32), pill_b=np.zeros(k, dtype=np.int32), alpha=np.zeros(k),
                   beta=np.zeros(k))
        if k:
            check(self._lib, self._lib.vrod_solver_get_contacts(
                self._h, k, C.byref(n), capi.ptr(out["pill_a"], C.c_int32), capi.ptr(out["pill_b"], C.c_int32),
                capi.ptr(out["alpha"]), capi.ptr(out["beta"])))
        return out

    def current_pills(self) -> np.ndarray:
        n = C.c_int64()
        check(self._lib, self._lib.vrod_solver_current_pills(self._h, 0, C.byref(n), None))
        out = np.zeros(n.value, dtype=capi.PILL_DTYPE)
        if n.value:
            check(self._lib, self._lib.vrod_solver_current_pills(self._h, n.value, C.byref(n),
                                                                 out.ctypes.data_as(C.c_void_p)))
        return out


    def shape_match(self) -> np.ndarray:
        """One apply_shape_match pass over the bundle groups in group order (bundling.cpp:116-133)
        on the live state (warm rotations updated); returns the SimilarityFit of every group as
        rows (scale, translation xyz, rotation row-major 3x3, degenerate 0/1)."""
        G = self.info().bundle_count
        out = np.zeros((max(G, 1), 14))
        n = C.c_int32()
        check(self._lib, self._lib.vrod_solver_shape_match(self._h, G, C.byref(n), capi.ptr(out)))
        return out[:n.value]

    def jacobi_sweep(self, h: float, beta: float) -> tuple[int, int]:
        """jacobi_sweep (constraints.cpp:491-556) of the elastic blocks and soft pins with zero
        multipliers on the live state; returns the SweepOutcome (active, skipped_singular)."""
        a, s = C.c_int32(), C.c_int32()
        check(self._lib, self._lib.vrod_solver_jacobi_sweep(self._h, h, beta, C.byref(a), C.byref(s)))
        return a.value, s.value

    def elastic_residuals(self) -> np.ndarray:
        """eval_constraint(...).W of every elastic block in block order, (n, 3)."""
        n = C.c_int64()
        check(self._lib, self._lib.vrod_solver_elastic_residuals(self._h, 0, C.byref(n), None))
        out = np.zeros((n.value, 3))
        if n.value:
            check(self._lib, self._lib.vrod_solver_elastic_residuals(self._h, n.value, C.byref(n), capi.ptr(out)))
        return out

    def _transforms(self, fn) -> np.ndarray:
        n = C.c_int64()
        check(self._lib, fn(self._h, 0, C.byref(n), None))
        out = np.zeros(n.value, dtype=capi.TRANSFORM_DTYPE)
        if n.value:
            check(self._lib, fn(self._h, n.value, C.byref(n), out.ctypes.data_as(C.c_void_p)))
        return out

    def pill_transforms(self) -> np.ndarray:
        """Solver::pill_transforms() (solver.cpp:438-440): rod pills, TRANSFORM_DTYPE records."""
        return self._transforms(self._lib.vrod_solver_pill_transforms)

    def rest_pill_transforms(self) -> np.ndarray:
        """rod_rest_pill_transforms(scene().rods) (skinning.cpp:24-37)."""
        return self._transforms(self._lib.vrod_solver_rest_pill_transforms)

    def rest_pills(self) -> np.ndarray:
        """rod_rest_pills(scene().rods) (skinning.cpp:39-57)."""
        n = C.c_int64()
        check(self._lib, self._lib.vrod_solver_rest_pills(self._h, 0, C.byref(n), None))
        out = np.zeros(n.value, dtype=capi.PILL_DTYPE)
        if n.value:
            check(self._lib, self._lib.vrod_solver_rest_pills(self._h, n.value, C.byref(n),
                                                              out.ctypes.data_as(C.c_void_p)))
        return out


class Skin:
    """SkinBinding + TriMesh (skinning.h:14-63) over any library exporting include/vrod_capi.h:
    bind_skin at construction, smooth_binding, deform_mesh (host transforms) and the fused
    per-frame deform of a solver's live state."""

    def __init__(self, lib, vertices, triangles, rest_pills: np.ndarray, rest_transforms: np.ndarray,
                 max_influences: int = 8, epsilon: float = 1e-4):
        self._lib = lib
        self._h = C.c_void_p()
        v = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
        t = np.ascontiguousarray(triangles if triangles is not None else np.zeros((0, 3)), dtype=np.int32).reshape(-1, 3)
        p = _pills(rest_pills)
        tr = np.ascontiguousarray(rest_transforms, dtype=capi.TRANSFORM_DTYPE)
        if len(tr) != len(p):  # the C-ABI takes one count for both lists (skinning.cpp:63-64)
            raise InvalidArgument("pill list and transform list must match")
        self.vertex_count = v.shape[0]
        check(lib, lib.vrod_skin_bind(v.shape[0], capi.ptr(v), t.shape[0], capi.ptr(t, C.c_int32), len(p),
                                      p.ctypes.data_as(C.c_void_p), tr.ctypes.data_as(C.c_void_p), max_influences,
                                      epsilon, C.byref(self._h)))

    def close(self) -> None:
        if self._h:
            self._lib.vrod_skin_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def smooth(self, iterations: int) -> None:
        check(self._lib, self._lib.vrod_skin_smooth(self._h, iterations))

    def binding(self) -> dict:
        nnz, cl = C.c_int32(), C.c_int32()
        check(self._lib, self._lib.vrod_skin_get_binding(self._h, None, None, None, C.byref(nnz), C.byref(cl)))
        off = np.zeros(self.vertex_count + 1, dtype=np.int32)
        pills = np.zeros(nnz.value, dtype=np.int32)
        w = np.zeros(nnz.value)
        check(self._lib, self._lib.vrod_skin_get_binding(self._h, capi.ptr(off, C.c_int32), capi.ptr(pills, C.c_int32),
                                                         capi.ptr(w), C.byref(nnz), C.byref(cl)))
        return dict(offsets=off, pills=pills, weights=w, clamped_vertices=cl.value)

    def deform(self, transforms: np.ndarray) -> np.ndarray:
        tr = np.ascontiguousarray(transforms, dtype=capi.TRANSFORM_DTYPE)
        out = np.zeros((self.vertex_count, 3))
        check(self._lib, self._lib.vrod_skin_deform(self._h, len(tr), tr.ctypes.data_as(C.c_void_p), capi.ptr(out)))
        return out

    def deform_solver(self, solver: "SolverHandle") -> np.ndarray:
        out = np.zeros((self.vertex_count, 3))
        check(self._lib, self._lib.vrod_skin_deform_solver(self._h, solver._h, capi.ptr(out)))
        return out


# ---- fine-grained collision entry points (collision.h:64-95) -----------------------------------

def _pills(p: np.ndarray) -> np.ndarray:
    p = np.ascontiguousarray(p)
    assert p.dtype == capi.PILL_DTYPE
    return p


def pill_project(lib, points: np.ndarray, pills: np.ndarray):
    x = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    p = _pills(pills)
    n = x.shape[0]
    t, d, g = np.zeros(n), np.zeros(n), np.zeros(n, dtype=np.uint8)
    check(lib, lib.vrod_pill_project(n, capi.ptr(x), p.ctypes.data_as(C.c_void_p), capi.ptr(t), capi.ptr(d),
                                     capi.ptr(g, C.c_uint8)))
    return t, d, g


def deepest_penetration(lib, a: np.ndarray, b: np.ndarray, iterations: int = 10, warm_alpha=None):
    a, b = _pills(a), _pills(b)
    n = a.shape[0]
    w = None if warm_alpha is None else np.ascontiguousarray(warm_alpha, dtype=np.float64)
    al, be, d = np.zeros(n), np.zeros(n), np.zeros(n)
    check(lib, lib.vrod_deepest_penetration(n, a.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p),
                                            iterations, capi.ptr(w), capi.ptr(al), capi.ptr(be), capi.ptr(d)))
    return al, be, d


def broad_phase(lib, pills: np.ndarray) -> np.ndarray:
    p = _pills(pills)
    cnt = C.c_int64()
    check(lib, lib.vrod_broad_phase(p.shape[0], p.ctypes.data_as(C.c_void_p), 0, C.byref(cnt), None))
    out = np.zeros((cnt.value, 2), dtype=np.int32)
    if cnt.value:
        check(lib, lib.vrod_broad_phase(p.shape[0], p.ctypes.data_as(C.c_void_p), cnt.value, C.byref(cnt),
                                        capi.ptr(out, C.c_int32)))
    return out


def find_contacts(lib, pills: np.ndarray, pairs: np.ndarray, iterations: int = 10, warm_keys=None,
                  warm_alpha=None) -> dict:
    p = _pills(pills)
    pr = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
    wk = None if warm_keys is None else np.ascontiguousarray(warm_keys, dtype=np.uint64)
    wa = None if warm_alpha is None else np.ascontiguousarray(warm_alpha, dtype=np.float64)
    nw = 0 if wk is None else wk.size
    cap = pr.shape[0]
    out = dict(pill_a=np.zeros(cap, dtype=np.int32), pill_b=np.zeros(cap, dtype=np.int32), alpha=np.zeros(cap),
               beta=np.zeros(cap), distance=np.zeros(cap))
    cnt = C.c_int64()
    check(lib, lib.vrod_find_contacts(p.shape[0], p.ctypes.data_as(C.c_void_p), pr.shape[0],
                                      capi.ptr(pr, C.c_int32), iterations, nw, capi.ptr(wk, C.c_uint64),
                                      capi.ptr(wa), cap, C.byref(cnt), capi.ptr(out["pill_a"], C.c_int32),
                                      capi.ptr(out["pill_b"], C.c_int32), capi.ptr(out["alpha"]),
                                      capi.ptr(out["beta"]), capi.ptr(out["distance"])))
    return {k: v[: cnt.value] for k, v in out.items()}


def extract_rotation(lib, covariance: np.ndarray, guess: np.ndarray, max_iterations: int = 100,
                     tolerance: float = 1e-9) -> np.ndarray:
    """extract_rotation (bundling.h:42-43) for n problems: covariance (n, 3, 3), guess (n, 4) wxyz."""
    B = np.ascontiguousarray(covariance, dtype=np.float64).reshape(-1, 9)
    g = np.ascontiguousarray(guess, dtype=np.float64).reshape(-1, 4)
    out = np.zeros_like(g)
    check(lib, lib.vrod_extract_rotation(len(B), capi.ptr(B), capi.ptr(g), max_iterations, tolerance, capi.ptr(out)))
    return out


def pair_key(lib, a: np.ndarray, b: np.ndarray) -> int:
    pa = capi.Pill.from_buffer_copy(np.ascontiguousarray(a).tobytes())
    pb = capi.Pill.from_buffer_copy(np.ascontiguousarray(b).tobytes())
    return int(lib.vrod_pair_key(C.byref(pa), C.byref(pb)))
