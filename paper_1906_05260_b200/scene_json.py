"""Scene files (schema 1) and the slice text format — the reference's scene_json.h / scene_json.cpp.

`load_scene` / `parse_scene_text` read a scene with the reference's schema checks and its exact
error messages (source name, then the JSON field path: "scene.json: rods[0].centers: ...",
scene_json.cpp:19-162, 292-462); rest poses come from make_rest_pose and the result is checked by
Scene::validate, both through the product library's host code. `scene_to_text` / `save_scene`
write the same schema (scene_json.cpp:467-661), so a scene round-trips to a textual fixed point.
The JSON itself is Python's `json` module (the reference uses nlohmann::json); only syntax-error
wording differs, which the reference's own tests leave unpinned (test_scene_json.cpp:124-133).
"""
from __future__ import annotations

import json
import math
import os

import numpy as np

from .scene import (Activation, Bone, HalfPlane, InvalidArgument, KinematicPill, MaterialParams, OutOfRange, Pill,
                    PinMotion, Probe, RigidKeyframe, Rod, Scene, SkinSetup, SoftPin, SolverSettings,
                    SCALE_POST_STEP_LENGTH_RATIO, SCALE_SIMULATED, make_rest_pose, make_rest_state, validate)


class SceneParseError(RuntimeError):
    """Malformed or schema-violating scene input (scene_json.h:14-17)."""


_MISSING = object()


def _fail(path: str, what: str):
    raise SceneParseError(what if not path else f"{path}: {what}")


def _item(path: str, key: str) -> str:
    return key if not path else f"{path}.{key}"


def _index(path: str, i: int) -> str:
    return f"{path}[{i}]"


def _check_keys(obj, allowed, path: str) -> None:
    if not isinstance(obj, dict):
        _fail(path, "expected an object")
    for key in obj:
        if key not in allowed:
            _fail(path, f"unknown field '{key}'")


def _find(obj, key):
    v = obj.get(key, None) if isinstance(obj, dict) else None
    return _MISSING if v is None else v


def _field(obj, key: str, path: str):
    v = _find(obj, key)
    if v is _MISSING:
        _fail(path, f"missing field '{key}'")
    return v


def _is_number(v) -> bool:  # JSON numbers; booleans are not numbers (nlohmann is_number)
    return isinstance(v, (int, float)) and not isinstance(v, bool)


def _number(v, path: str) -> float:
    if not _is_number(v):
        _fail(path, "expected a number")
    return float(v)


def _int(v, path: str) -> int:
    if not (isinstance(v, int) and not isinstance(v, bool)):
        _fail(path, "expected an integer")
    return int(v)


def _bool(v, path: str) -> bool:
    if not isinstance(v, bool):
        _fail(path, "expected a boolean")
    return v


def _string(v, path: str) -> str:
    if not isinstance(v, str):
        _fail(path, "expected a string")
    return v


def _array(v, path: str) -> list:
    if not isinstance(v, list):
        _fail(path, "expected an array")
    return v


def _vec3(v, path: str) -> tuple:
    arr = _array(v, path)
    if len(arr) != 3:
        _fail(path, "expected 3 numbers")
    return tuple(_number(arr[i], _index(path, i)) for i in range(3))


def _quat(v, path: str) -> tuple:
    """(x, y, z, w) in the file, normalized (scene_json.cpp:91-99); returned as (w, x, y, z)."""
    arr = _array(v, path)
    if len(arr) != 4:
        _fail(path, "expected 4 numbers (x, y, z, w)")
    x, y, z, w = (_number(arr[i], _index(path, i)) for i in range(4))
    # Eigen's norm / normalize: squared norm over (x, y, z, w) coefficients, then / sqrt(n)
    n2 = (x * x + y * y) + (z * z + w * w)
    norm = math.sqrt(n2)
    if norm < 1e-9:
        _fail(path, "rotation has near-zero norm")
    return (w / norm, x / norm, y / norm, z / norm)


def _opt_number(obj, key, fallback, path):
    v = _find(obj, key)
    return fallback if v is _MISSING else _number(v, _item(path, key))


def _opt_int(obj, key, fallback, path):
    v = _find(obj, key)
    return fallback if v is _MISSING else _int(v, _item(path, key))


def _opt_bool(obj, key, fallback, path):
    v = _find(obj, key)
    return fallback if v is _MISSING else _bool(v, _item(path, key))


def _number_list(v, path):
    arr = _array(v, path)
    return [_number(arr[i], _index(path, i)) for i in range(len(arr))]


def _vec3_list(v, path):
    arr = _array(v, path)
    return [_vec3(arr[i], _index(path, i)) for i in range(len(arr))]


def _parse_settings(obj, path) -> SolverSettings:  # scene_json.cpp:131-162
    _check_keys(obj, ("dt", "iterations", "substeps", "beta", "gravity", "dichotomous_iterations",
                      "shape_match_period", "contact_stiffness", "velocity_damping", "deterministic", "scale_mode"),
                path)
    s = SolverSettings()
    s.dt = _opt_number(obj, "dt", s.dt, path)
    s.iterations = _opt_int(obj, "iterations", s.iterations, path)
    s.substeps = _opt_int(obj, "substeps", s.substeps, path)
    s.beta = _opt_number(obj, "beta", s.beta, path)
    g = _find(obj, "gravity")
    if g is not _MISSING:
        s.gravity = _vec3(g, _item(path, "gravity"))
    s.dichotomous_iterations = _opt_int(obj, "dichotomous_iterations", s.dichotomous_iterations, path)
    s.shape_match_period = _opt_int(obj, "shape_match_period", s.shape_match_period, path)
    s.contact_stiffness = _opt_number(obj, "contact_stiffness", s.contact_stiffness, path)
    s.velocity_damping = _opt_number(obj, "velocity_damping", s.velocity_damping, path)
    s.deterministic = _opt_bool(obj, "deterministic", s.deterministic, path)
    m = _find(obj, "scale_mode")
    if m is not _MISSING:
        mode = _string(m, _item(path, "scale_mode"))
        if mode == "simulated":
            s.scale_mode = SCALE_SIMULATED
        elif mode == "post_step_length_ratio":
            s.scale_mode = SCALE_POST_STEP_LENGTH_RATIO
        else:
            _fail(_item(path, "scale_mode"), f'expected "simulated" or "post_step_length_ratio", got "{mode}"')
    return s


def _parse_material(obj, path) -> MaterialParams:  # scene_json.cpp:164-178
    keys = ("stretch_x", "stretch_y", "stretch_z", "bend_x", "bend_y", "bend_z", "volume", "density")
    _check_keys(obj, keys, path)
    m = MaterialParams()
    for k in keys:
        setattr(m, k, _opt_number(obj, k, getattr(m, k), path))
    return m


def _parse_rod(lib, obj, path) -> Rod:  # scene_json.cpp:180-257
    _check_keys(obj, ("centers", "radius", "radii", "scales", "material", "pinned", "collision_group", "self_collide",
                      "center_velocity", "scale_velocity", "angular_velocity", "bones", "bone_weights"), path)
    centers = _vec3_list(_field(obj, "centers", path), _item(path, "centers"))
    if len(centers) < 2:
        _fail(_item(path, "centers"), "a rod needs at least 2 vertices")
    radius, radii_field = _find(obj, "radius"), _find(obj, "radii")
    if (radius is not _MISSING) == (radii_field is not _MISSING):
        _fail(path, "expected exactly one of 'radius' or 'radii'")
    radii = [_number(radius, _item(path, "radius"))] if radius is not _MISSING else \
        _number_list(radii_field, _item(path, "radii"))
    sv = _find(obj, "scales")
    scales = None if sv is _MISSING else _number_list(sv, _item(path, "scales"))
    try:
        rest = make_rest_pose(lib, centers, radii, scales if scales else None)
    except (InvalidArgument, OutOfRange) as e:
        _fail(path, str(e))
    rod = Rod(rest=rest, state=make_rest_state(rest))
    rod.material = _opt_int(obj, "material", 0, path)
    rod.collision_group = _opt_int(obj, "collision_group", -1, path)
    rod.self_collide = _opt_bool(obj, "self_collide", False, path)
    n = rest.vertex_count()
    rod.pinned = np.zeros(n, dtype=np.uint8)
    pv = _find(obj, "pinned")
    if pv is not _MISSING:
        where = _item(path, "pinned")
        arr = _array(pv, where)
        for i in range(len(arr)):
            vertex = _int(arr[i], _index(where, i))
            if vertex < 0 or vertex >= n:
                _fail(_index(where, i), "pinned vertex out of range")
            rod.pinned[vertex] = 1
    v = _find(obj, "center_velocity")
    if v is not _MISSING:
        vel = _vec3_list(v, _item(path, "center_velocity"))
        if len(vel) != n:
            _fail(_item(path, "center_velocity"), "expected one entry per vertex")
        rod.state.center_vel = np.array(vel, dtype=np.float64).reshape(n, 3)
    v = _find(obj, "scale_velocity")
    if v is not _MISSING:
        vel = _number_list(v, _item(path, "scale_velocity"))
        if len(vel) != n:
            _fail(_item(path, "scale_velocity"), "expected one entry per vertex")
        rod.state.scale_vel = np.array(vel, dtype=np.float64)
    v = _find(obj, "angular_velocity")
    if v is not _MISSING:
        vel = _vec3_list(v, _item(path, "angular_velocity"))
        if len(vel) != rest.element_count():
            _fail(_item(path, "angular_velocity"), "expected one entry per element")
        rod.state.angular_vel = np.array(vel, dtype=np.float64).reshape(-1, 3)
    b = _find(obj, "bones")
    if b is not _MISSING:
        where = _item(path, "bones")
        arr = _array(b, where)
        rod.bones = [_int(arr[i], _index(where, i)) for i in range(len(arr))]
        ww = _item(path, "bone_weights")
        weights = _array(_field(obj, "bone_weights", path), ww)
        if len(weights) != n:
            _fail(ww, "expected one row per vertex")
        rows = [_number_list(weights[i], _index(ww, i)) for i in range(len(weights))]
        # ragged rows are kept as given for Scene::validate to name ("bone weight row size")
        rod.bone_weights = rows if any(len(r) != len(rod.bones) for r in rows) else \
            np.array(rows, dtype=np.float64).reshape(n, len(rod.bones))
    elif _find(obj, "bone_weights") is not _MISSING:
        _fail(path, "'bone_weights' given without 'bones'")
    return rod


def read_obj(path: str):
    """obj_io read_obj for the skin mesh: 'v x y z' and 'f a b c' (1-based; v/vt/vn forms) lines."""
    try:
        text = open(path).read()
    except OSError:
        raise RuntimeError(f"cannot open OBJ file: {path}") from None
    verts, tris = [], []
    for ln, line in enumerate(text.splitlines(), 1):
        parts = line.split("#", 1)[0].split()
        if not parts:
            continue
        if parts[0] == "v":
            verts.append(tuple(float(x) for x in parts[1:4]))
        elif parts[0] == "f":
            idx = [int(p.split("/")[0]) - 1 for p in parts[1:]]
            for k in range(1, len(idx) - 1):  # fan triangulation of polygons
                tris.append((idx[0], idx[k], idx[k + 1]))
    return verts, tris


def _parse_mesh(obj, path, base_dir):  # scene_json.cpp:259-290
    v = _find(obj, "obj")
    if v is not _MISSING:
        mesh_path = _string(v, _item(path, "obj"))
        if base_dir and mesh_path and not mesh_path.startswith("/"):
            mesh_path = base_dir + "/" + mesh_path
        try:
            return read_obj(mesh_path)
        except Exception as e:  # noqa: BLE001 - the reference wraps any read failure
            _fail(_item(path, "obj"), str(e))
    verts = _vec3_list(_field(obj, "vertices", path), _item(path, "vertices"))
    tw = _item(path, "triangles")
    tris_j = _array(_field(obj, "triangles", path), tw)
    tris = []
    for i in range(len(tris_j)):
        where = _index(tw, i)
        tri = _array(tris_j[i], where)
        if len(tri) != 3:
            _fail(where, "expected 3 vertex indices")
        tris.append(tuple(_int(tri[k], _index(where, k)) for k in range(3)))
    return verts, tris


def _parse_scene(lib, root, base_dir) -> Scene:  # scene_json.cpp:292-462
    if not isinstance(root, dict):
        _fail("", "top level must be an object")
    _check_keys(root, ("schema", "settings", "materials", "rods", "planes", "kinematic_pills", "bones", "bundles",
                       "pin_motions", "soft_pins", "activations", "probes", "skin"), "")
    schema = _int(_field(root, "schema", ""), "schema")
    if schema != 1:
        _fail("schema", f"unsupported schema version {schema}")
    scene = Scene()
    v = _find(root, "settings")
    if v is not _MISSING:
        scene.settings = _parse_settings(v, "settings")
    v = _find(root, "materials")
    if v is not _MISSING:
        arr = _array(v, "materials")
        scene.materials = [_parse_material(arr[i], _index("materials", i)) for i in range(len(arr))]
    if not scene.materials:
        scene.materials.append(MaterialParams())
    rods = _array(_field(root, "rods", ""), "rods")
    scene.rods = [_parse_rod(lib, rods[i], _index("rods", i)) for i in range(len(rods))]
    v = _find(root, "planes")
    if v is not _MISSING:
        arr = _array(v, "planes")
        for i in range(len(arr)):
            where = _index("planes", i)
            _check_keys(arr[i], ("normal", "offset"), where)
            nrm = _vec3(_field(arr[i], "normal", where), _item(where, "normal"))
            norm = math.sqrt((nrm[0] * nrm[0] + nrm[1] * nrm[1]) + nrm[2] * nrm[2])
            if norm < 1e-9:
                _fail(_item(where, "normal"), "normal has near-zero norm")
            scene.planes.append(HalfPlane(normal=tuple(c / norm for c in nrm),
                                          offset=_opt_number(arr[i], "offset", 0.0, where)))
    v = _find(root, "bones")
    if v is not _MISSING:
        arr = _array(v, "bones")
        for i in range(len(arr)):
            where = _index("bones", i)
            _check_keys(arr[i], ("keys",), where)
            kw0 = _item(where, "keys")
            keys = _array(_field(arr[i], "keys", where), kw0)
            bone = Bone()
            for k in range(len(keys)):
                kw = _index(kw0, k)
                _check_keys(keys[k], ("t", "position", "rotation"), kw)
                key = RigidKeyframe(t=_number(_field(keys[k], "t", kw), _item(kw, "t")))
                p = _find(keys[k], "position")
                if p is not _MISSING:
                    key.position = _vec3(p, _item(kw, "position"))
                r = _find(keys[k], "rotation")
                if r is not _MISSING:
                    key.rotation = _quat(r, _item(kw, "rotation"))
                bone.keys.append(key)
            scene.bones.append(bone)
    v = _find(root, "kinematic_pills")
    if v is not _MISSING:
        arr = _array(v, "kinematic_pills")
        for i in range(len(arr)):
            where = _index("kinematic_pills", i)
            _check_keys(arr[i], ("c0", "c1", "r0", "r1", "group", "bone"), where)
            pill = Pill(c0=_vec3(_field(arr[i], "c0", where), _item(where, "c0")),
                        c1=_vec3(_field(arr[i], "c1", where), _item(where, "c1")),
                        r0=_number(_field(arr[i], "r0", where), _item(where, "r0")),
                        r1=_number(_field(arr[i], "r1", where), _item(where, "r1")))
            pill.group = _opt_int(arr[i], "group", -1, where)
            scene.kinematic_pills.append(KinematicPill(pill=pill, bone=_opt_int(arr[i], "bone", -1, where)))
    v = _find(root, "bundles")
    if v is not _MISSING:
        arr = _array(v, "bundles")
        for i in range(len(arr)):
            where = _index("bundles", i)
            group = _array(arr[i], where)
            members = []
            for k in range(len(group)):
                mw = _index(where, k)
                _check_keys(group[k], ("rod", "vertex"), mw)
                members.append((_int(_field(group[k], "rod", mw), _item(mw, "rod")),
                                _int(_field(group[k], "vertex", mw), _item(mw, "vertex"))))
            scene.bundles.append(members)
    v = _find(root, "pin_motions")
    if v is not _MISSING:
        arr = _array(v, "pin_motions")
        for i in range(len(arr)):
            where = _index("pin_motions", i)
            _check_keys(arr[i], ("rod", "vertex", "start", "target", "t0", "t1"), where)
            scene.pin_motions.append(PinMotion(
                rod=_int(_field(arr[i], "rod", where), _item(where, "rod")),
                vertex=_int(_field(arr[i], "vertex", where), _item(where, "vertex")),
                start=_vec3(_field(arr[i], "start", where), _item(where, "start")),
                target=_vec3(_field(arr[i], "target", where), _item(where, "target")),
                t0=_opt_number(arr[i], "t0", 0.0, where),
                t1=_number(_field(arr[i], "t1", where), _item(where, "t1"))))
    v = _find(root, "soft_pins")
    if v is not _MISSING:
        arr = _array(v, "soft_pins")
        for i in range(len(arr)):
            where = _index("soft_pins", i)
            _check_keys(arr[i], ("rod", "vertex", "target", "stiffness"), where)
            sp = SoftPin(rod=_int(_field(arr[i], "rod", where), _item(where, "rod")),
                         vertex=_int(_field(arr[i], "vertex", where), _item(where, "vertex")),
                         target=_vec3(_field(arr[i], "target", where), _item(where, "target")))
            sp.stiffness = _opt_number(arr[i], "stiffness", sp.stiffness, where)
            scene.soft_pins.append(sp)
    v = _find(root, "activations")
    if v is not _MISSING:
        arr = _array(v, "activations")
        for i in range(len(arr)):
            where = _index("activations", i)
            _check_keys(arr[i], ("rod", "factor", "t_start", "t_end", "first_element", "last_element"), where)
            a = Activation(rod=_int(_field(arr[i], "rod", where), _item(where, "rod")))
            a.factor = _opt_number(arr[i], "factor", a.factor, where)
            a.t_start = _opt_number(arr[i], "t_start", a.t_start, where)
            a.t_end = _opt_number(arr[i], "t_end", a.t_end, where)
            a.first_element = _opt_int(arr[i], "first_element", a.first_element, where)
            a.last_element = _opt_int(arr[i], "last_element", a.last_element, where)
            scene.activations.append(a)
    v = _find(root, "probes")
    if v is not _MISSING:
        arr = _array(v, "probes")
        for i in range(len(arr)):
            where = _index("probes", i)
            _check_keys(arr[i], ("name", "rod", "vertex"), where)
            scene.probes.append(Probe(name=_string(_field(arr[i], "name", where), _item(where, "name")),
                                      rod=_int(_field(arr[i], "rod", where), _item(where, "rod")),
                                      vertex=_int(_field(arr[i], "vertex", where), _item(where, "vertex"))))
    v = _find(root, "skin")
    if v is not _MISSING:
        _check_keys(v, ("obj", "vertices", "triangles", "max_influences", "epsilon", "smooth_iterations"), "skin")
        verts, tris = _parse_mesh(v, "skin", base_dir)
        skin = SkinSetup(vertices=verts, triangles=tris)
        skin.max_influences = _opt_int(v, "max_influences", skin.max_influences, "skin")
        skin.epsilon = _opt_number(v, "epsilon", skin.epsilon, "skin")
        skin.smooth_iterations = _opt_int(v, "smooth_iterations", skin.smooth_iterations, "skin")
        scene.skin = skin
    validate(lib, scene)  # Scene::validate, scene.cpp:63-157 (its messages, through the same prefix)
    return scene


def parse_scene_text(lib, text: str, source_name: str, base_dir: str = "") -> Scene:
    """parse_scene_text, scene_json.cpp:678-694."""
    try:
        root = json.loads(text)
    except json.JSONDecodeError as e:
        raise SceneParseError(f"{source_name}: [json.exception.parse_error] {e}") from None
    try:
        return _parse_scene(lib, root, base_dir)
    except SceneParseError as e:
        raise SceneParseError(f"{source_name}: {e}") from None
    except (InvalidArgument, OutOfRange) as e:  # Scene::validate failures (std::logic_error)
        raise SceneParseError(f"{source_name}: {e}") from None


def load_scene(lib, path: str) -> Scene:
    """load_scene, scene_json.cpp:670-676."""
    try:
        text = open(path).read()
    except OSError:
        raise SceneParseError(f"{path}: cannot open scene file") from None
    return parse_scene_text(lib, text, path, os.path.dirname(path))


# ---- writer (scene_json.cpp:467-661) ----------------------------------------------------------

def _v3(v) -> list:
    return [float(v[0]), float(v[1]), float(v[2])]


def scene_json(scene: Scene) -> dict:
    s = scene.settings
    root: dict = {"schema": 1}
    settings = {"dt": s.dt, "iterations": s.iterations, "substeps": s.substeps, "beta": s.beta,
                "gravity": _v3(s.gravity), "dichotomous_iterations": s.dichotomous_iterations,
                "shape_match_period": s.shape_match_period}
    if math.isfinite(s.contact_stiffness):
        settings["contact_stiffness"] = s.contact_stiffness
    settings.update({"velocity_damping": s.velocity_damping, "deterministic": bool(s.deterministic),
                     "scale_mode": "simulated" if s.scale_mode == SCALE_SIMULATED else "post_step_length_ratio"})
    root["settings"] = settings
    root["materials"] = [{k: getattr(m, k) for k in ("stretch_x", "stretch_y", "stretch_z", "bend_x", "bend_y",
                                                     "bend_z", "volume", "density")} for m in scene.materials]
    rods = []
    for rod in scene.rods:
        st = rod.state
        r = {"centers": [_v3(c) for c in st.centers], "radii": [float(x) for x in rod.rest.radii],
             "scales": [float(x) for x in st.scales], "material": rod.material,
             "pinned": [int(v) for v in np.nonzero(np.asarray(rod.pinned))[0]],
             "collision_group": rod.collision_group, "self_collide": bool(rod.self_collide)}
        if np.any(np.sum(np.asarray(st.center_vel) ** 2, axis=1) > 0.0):
            r["center_velocity"] = [_v3(v) for v in st.center_vel]
        if np.any(np.asarray(st.scale_vel) != 0.0):
            r["scale_velocity"] = [float(x) for x in st.scale_vel]
        if len(st.angular_vel) and np.any(np.sum(np.asarray(st.angular_vel) ** 2, axis=1) > 0.0):
            r["angular_velocity"] = [_v3(v) for v in st.angular_vel]
        if len(rod.bones):
            r["bones"] = [int(b) for b in rod.bones]
            r["bone_weights"] = [[float(x) for x in row] for row in rod.bone_weights]
        rods.append(r)
    root["rods"] = rods
    if scene.planes:
        root["planes"] = [{"normal": _v3(p.normal), "offset": p.offset} for p in scene.planes]
    if scene.bones:
        root["bones"] = [{"keys": [{"t": k.t, "position": _v3(k.position),
                                    "rotation": [k.rotation[1], k.rotation[2], k.rotation[3], k.rotation[0]]}
                                   for k in b.keys]} for b in scene.bones]
    if scene.kinematic_pills:
        pills = []
        for kp in scene.kinematic_pills:
            p = {"c0": _v3(kp.pill.c0), "c1": _v3(kp.pill.c1), "r0": kp.pill.r0, "r1": kp.pill.r1}
            if kp.pill.group >= 0:
                p["group"] = kp.pill.group
            if kp.bone >= 0:
                p["bone"] = kp.bone
            pills.append(p)
        root["kinematic_pills"] = pills
    if scene.bundles:
        root["bundles"] = [[{"rod": int(r), "vertex": int(v)} for r, v in g] for g in scene.bundles]
    if scene.pin_motions:
        root["pin_motions"] = [{"rod": p.rod, "vertex": p.vertex, "start": _v3(p.start), "target": _v3(p.target),
                                "t0": p.t0, "t1": p.t1} for p in scene.pin_motions]
    if scene.soft_pins:
        pins = []
        for sp in scene.soft_pins:
            p = {"rod": sp.rod, "vertex": sp.vertex, "target": _v3(sp.target)}
            if math.isfinite(sp.stiffness):
                p["stiffness"] = sp.stiffness
            pins.append(p)
        root["soft_pins"] = pins
    if scene.activations:
        root["activations"] = [{"rod": a.rod, "factor": a.factor, "t_start": a.t_start, "t_end": a.t_end,
                                "first_element": a.first_element, "last_element": a.last_element}
                               for a in scene.activations]
    if scene.probes:
        root["probes"] = [{"name": p.name, "rod": p.rod, "vertex": p.vertex} for p in scene.probes]
    if scene.skin is not None:
        sk = scene.skin
        root["skin"] = {"vertices": [_v3(v) for v in sk.vertices], "triangles": [[int(a) for a in t] for t in sk.triangles],
                        "max_influences": sk.max_influences, "epsilon": sk.epsilon,
                        "smooth_iterations": sk.smooth_iterations}
    return root


def scene_to_text(scene: Scene) -> str:
    """scene_to_text, scene_json.cpp:703: two-space indented JSON plus a newline."""
    return json.dumps(scene_json(scene), indent=2) + "\n"


def save_scene(scene: Scene, path: str) -> None:
    try:
        with open(path, "w") as f:
            f.write(scene_to_text(scene))
    except OSError:
        raise RuntimeError(f"{path}: cannot open for writing") from None


# ---- slice text (scene_json.cpp:705-745) and the comb output format (:747-759) -----------------

def parse_slice_text(text: str, source_name: str) -> list:
    slices, current = [], []
    for line_number, line in enumerate(text.split("\n"), 1):
        line = line.split("#", 1)[0]
        fields = line.split()
        x_ok = False
        if fields:
            try:
                float(fields[0])
                x_ok = True
            except ValueError:
                x_ok = False
        if x_ok:
            try:
                if len(fields) != 3:
                    raise ValueError
                current.append(tuple(float(f) for f in fields))
            except ValueError:
                raise SceneParseError(f"{source_name}:{line_number}: expected three numbers per point") from None
        elif current:
            slices.append(current)
            current = []
    if current:
        slices.append(current)
    return slices


def read_slice_file(path: str) -> list:
    try:
        text = open(path).read()
    except OSError:
        raise SceneParseError(f"{path}: cannot open slice file") from None
    return parse_slice_text(text, path)


def write_rod_scene(polylines, radius: float, path: str) -> None:
    root = {"schema": 1, "rods": [{"centers": [_v3(c) for c in line], "radius": radius} for line in polylines]}
    try:
        with open(path, "w") as f:
            f.write(json.dumps(root, indent=2) + "\n")
    except OSError:
        raise RuntimeError(f"{path}: cannot open for writing") from None
