"""Per-step CSV logs of the reference CLI (metrics.h / metrics.cpp): metrics.csv (residual RMS per
elastic kind normalised by total rest length or rest volume, volumes, kinetic energy, penetration,
wall time), probes.csv (probe vertex centre and scale) and the convergence log. Same columns, same
`%.17g` number format (metrics.cpp:10-14), so the files diff against the reference's."""
from __future__ import annotations

import numpy as np

KINDS = ("stretch_z", "cross_section", "surface_stretch", "bend_twist", "surface_bending", "volume_stretch",
         "volume_bend_u", "volume_bend_v")
VOLUME_KINDS = {5, 6, 7}  # kVolumeStretch, kVolumeBendU, kVolumeBendV (metrics.cpp:43-46)


def _g(x: float) -> str:
    return "%.17g" % x


def metric_normalizers(scene) -> tuple:
    """metric_normalizers, metrics.cpp:18-29: total as-built length and rest volume (1 if zero)."""
    length, volume = 0.0, 0.0
    for rod in scene.rods:
        for l in rod.rest.initial_lengths:
            length += float(l)
        rest = rod.rest
        v = 0.0
        for e in range(rest.element_count()):  # rest_volume, rod.cpp:189-197
            s = 0.5 * (rest.scales[e] + rest.scales[e + 1])
            r = 0.5 * (rest.radii[e] + rest.radii[e + 1])
            v += np.pi * (s * r) * (s * r) * rest.initial_lengths[e]
        volume += v
    return (length if length > 0.0 else 1.0, volume if volume > 0.0 else 1.0)


class MetricsWriter:
    """MetricsWriter, metrics.cpp:31-57."""

    HEADER = ("step,time,stretch_z,cross_section,surface_stretch,bend_twist,surface_bending,volume_stretch,"
              "volume_bend_u,volume_bend_v,total_volume,rest_volume,kinetic_energy,max_penetration,wall_ms\n")

    def __init__(self, path: str, scene):
        try:
            self._out = open(path, "w", newline="")
        except OSError:
            raise RuntimeError(f"cannot write metrics file: {path}") from None
        self._norm_length, self._norm_volume = metric_normalizers(scene)
        self._deterministic = bool(scene.settings.deterministic)
        self._out.write(self.HEADER)

    def write(self, report, solver) -> None:
        f = [str(report.step), _g(report.time)]
        for k in range(8):
            f.append(_g(report.residuals[k] / (self._norm_volume if k in VOLUME_KINDS else self._norm_length)))
        f += [_g(solver.total_volume()), _g(solver.total_rest_volume()), _g(solver.kinetic_energy()),
              _g(report.max_penetration), _g(0.0 if self._deterministic else report.timings["total_ms"])]
        self._out.write(",".join(f) + "\n")
        self._out.flush()

    def close(self) -> None:
        self._out.close()


class ProbeWriter:
    """ProbeWriter, metrics.cpp:59-89: nothing is written for a scene without probes."""

    def __init__(self, path: str, scene):
        self._probes = list(scene.probes)
        self._out = None
        if not self._probes:
            return
        try:
            self._out = open(path, "w", newline="")
        except OSError:
            raise RuntimeError(f"cannot write probe file: {path}") from None
        cols = "".join(f",{p.name}_x,{p.name}_y,{p.name}_z,{p.name}_s" for p in self._probes)
        self._out.write("step,time" + cols + "\n")

    def write(self, step: int, time: float, rod_state) -> None:
        """rod_state(r) -> dict(centers, scales) of rod r (the solver's live state)."""
        if self._out is None:
            return
        f = [str(step), _g(time)]
        cache = {}
        for p in self._probes:
            if p.rod not in cache:
                cache[p.rod] = rod_state(p.rod)
            st = cache[p.rod]
            c = st["centers"][p.vertex]
            f += [_g(c[0]), _g(c[1]), _g(c[2]), _g(st["scales"][p.vertex])]
        self._out.write(",".join(f) + "\n")
        self._out.flush()

    def close(self) -> None:
        if self._out is not None:
            self._out.close()


def write_convergence_csv(path: str, log) -> None:
    """write_convergence_csv, metrics.cpp:91-98: one row per sweep of probe_convergence."""
    with open(path, "w", newline="") as out:
        out.write("iteration," + ",".join(KINDS) + "\n")
        for i, row in enumerate(np.asarray(log)):
            out.write(f"{i + 1}," + ",".join(_g(x) for x in row[:8]) + "\n")
