"""Workload generator: parses the reference's scene-script format
(synth.cpp:207-351) and renders frames on the GPU with rf_synth_render
(synth.cpp:136-203 restated as a CUDA kernel, counter-based depth noise).

Used by bench.py to build the BASELINE.json configs without a host
bottleneck; parity tests use the oracle renderer instead (identical bytes to
the reference's mt19937 noise)."""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from . import api


@dataclass
class Primitive:
    name: str
    dynamic: bool
    shape: int  # 0 plane, 1 sphere, 2 box
    a: np.ndarray
    b: np.ndarray
    checker: bool = False
    cell: float = 0.25
    primary: tuple = (200, 200, 200)
    secondary: tuple = (60, 60, 60)
    keyframes: list = field(default_factory=list)  # (t, R 3x3, t 3)


@dataclass
class Scene:
    intrinsics: L.rf_intrinsics
    noise: float
    dropout: float
    seed: int
    prims: list
    camera: list  # (t, pose12)

    def __len__(self):
        return len(self.camera)


# Pose arithmetic in the reference's operation order (Eigen's Quaterniond
# normalized / toRotationMatrix / slerp / quaternion-from-matrix and the 3x3
# products, as synth.cpp and geometry.hpp use them), so the renderer sees the
# same double-precision poses as RenderFrame (synth.cpp:136-203).
def _normalized(w, x, y, z):
    n = math.sqrt(((x * x + y * y) + z * z) + w * w)
    return w / n, x / n, y / n, z / n


def _quat_to_R(w, x, y, z):  # geometry.hpp:78-79: q.normalized().toRotationMatrix()
    w, x, y, z = _normalized(w, x, y, z)
    tx, ty, tz = 2.0 * x, 2.0 * y, 2.0 * z
    twx, twy, twz = tx * w, ty * w, tz * w
    txx, txy, txz = tx * x, ty * x, tz * x
    tyy, tyz, tzz = ty * y, tz * y, tz * z
    return np.array([[1.0 - (tyy + tzz), txy - twz, txz + twy],
                     [txy + twz, 1.0 - (txx + tzz), tyz - twx],
                     [txz - twy, tyz + twx, 1.0 - (txx + tyy)]])


def _R_to_quat(m):  # Eigen's quaternion-from-matrix (Shepperd), as (w, x, y, z)
    m = [[float(m[i][j]) for j in range(3)] for i in range(3)]
    t = (m[0][0] + m[1][1]) + m[2][2]
    if t > 0.0:
        t = math.sqrt(t + 1.0)
        w = 0.5 * t
        t = 0.5 / t
        return (w, (m[2][1] - m[1][2]) * t, (m[0][2] - m[2][0]) * t, (m[1][0] - m[0][1]) * t)
    i = 0
    if m[1][1] > m[0][0]:
        i = 1
    if m[2][2] > m[i][i]:
        i = 2
    j, k = (i + 1) % 3, (i + 2) % 3
    t = math.sqrt(((m[i][i] - m[j][j]) - m[k][k]) + 1.0)
    c = [0.0, 0.0, 0.0]
    c[i] = 0.5 * t
    t = 0.5 / t
    w = (m[k][j] - m[j][k]) * t
    c[j] = (m[j][i] + m[i][j]) * t
    c[k] = (m[k][i] + m[i][k]) * t
    return (w, c[0], c[1], c[2])


def _slerp(a, t, b):  # Eigen QuaternionBase::slerp; quaternions as (w, x, y, z)
    one = 1.0 - 2.220446049250313e-16
    d = ((a[1] * b[1] + a[2] * b[2]) + a[3] * b[3]) + a[0] * b[0]
    absd = abs(d)
    if absd >= one:
        s0, s1 = 1.0 - t, t
    else:
        theta = math.acos(absd)
        st = math.sin(theta)
        s0, s1 = math.sin((1.0 - t) * theta) / st, math.sin(t * theta) / st
    if d < 0:
        s1 = -s1
    return tuple(s0 * a[i] + s1 * b[i] for i in range(4))


def _pose_at(prim: Primitive, time: float):
    """Primitive::PoseAt (synth.cpp:26-45): object-to-world (R, t)."""
    kf = prim.keyframes
    if not kf:
        return np.eye(3), np.zeros(3)
    if time <= kf[0][0]:
        return kf[0][1], kf[0][2]
    if time >= kf[-1][0]:
        return kf[-1][1], kf[-1][2]
    hi = 1
    while kf[hi][0] < time:
        hi += 1
    (t0, R0, p0), (t1, R1, p1) = kf[hi - 1], kf[hi]
    al = (time - t0) / (t1 - t0)
    q = _slerp(_R_to_quat(R0), al, _R_to_quat(R1))
    t = np.array([(1.0 - al) * float(p0[i]) + al * float(p1[i]) for i in range(3)])
    return _quat_to_R(*q), t


def _inverse(R, t):
    """Pose::Inverse (geometry.hpp:93-96): (R^T, -(R^T t)), rows summed left to right."""
    Rt = [[float(R[j][i]) for j in range(3)] for i in range(3)]
    ti = [-((Rt[i][0] * float(t[0]) + Rt[i][1] * float(t[1])) + Rt[i][2] * float(t[2])) for i in range(3)]
    return np.array(Rt), np.array(ti)


def parse(text: str) -> Scene:
    """SceneScript::Parse (synth.cpp:255-343), the subset of checks a workload needs."""
    k = api.intrinsics()
    noise = dropout = 0.0
    seed = 0
    prims, camera = [], []
    for no, line in enumerate(text.splitlines(), 1):
        tok = line.split()
        if not tok or tok[0].startswith("#"):
            continue
        d = tok[0]
        if d == "intrinsics":
            fx, fy, cx, cy, w, h, ds = tok[1:8]
            k = api.intrinsics(float(fx), float(fy), float(cx), float(cy), int(w), int(h), float(ds))
        elif d == "noise":
            noise, dropout = float(tok[1]), float(tok[2])
        elif d == "seed":
            seed = int(tok[1])
        elif d == "primitive":
            name, motion, shape = tok[1:4]
            sh = {"plane": 0, "sphere": 1, "box": 2}[shape]
            nums = 6 if sh != 1 else 4
            vals = [float(x) for x in tok[4:4 + nums]]
            a = np.array(vals[:3])
            b = np.array(vals[3:] + [0.0, 0.0]) if sh == 1 else np.array(vals[3:6])
            if sh == 0:
                b = b / np.linalg.norm(b)
            rest = tok[4 + nums:]
            assert rest[0] == "albedo", f"line {no}: expected albedo"
            p = Primitive(name, motion == "dynamic", sh, a, b)
            if rest[1] == "uniform":
                p.primary = tuple(int(x) for x in rest[2:5])
            else:
                p.checker = True
                p.cell = float(rest[2])
                p.primary = tuple(int(x) for x in rest[3:6])
                p.secondary = tuple(int(x) for x in rest[6:9])
            prims.append(p)
        elif d == "keyframe":
            name, t = tok[1], float(tok[2])
            tx, ty, tz, qx, qy, qz, qw = (float(x) for x in tok[3:10])
            target = next(p for p in prims if p.name == name)
            target.keyframes.append((t, _quat_to_R(*_normalized(qw, qx, qy, qz)), np.array([tx, ty, tz])))
        elif d == "camera":
            t = float(tok[1])
            tx, ty, tz, qx, qy, qz, qw = (float(x) for x in tok[2:9])
            pose = np.concatenate([_quat_to_R(*_normalized(qw, qx, qy, qz)).reshape(9), [tx, ty, tz]])
            camera.append((t, pose))
        else:
            raise ValueError(f"scene line {no}: unknown directive '{d}'")
    return Scene(k, noise, dropout, seed, prims, camera)


class _Prim(C.Structure):  # rf_synth_primitive, 176 bytes
    _fields_ = [("shape", C.c_int32), ("dynamic", C.c_int32), ("checker", C.c_int32), ("pad", C.c_int32),
                ("a", C.c_double * 3), ("b", C.c_double * 3), ("cell", C.c_double), ("w2o", C.c_double * 12),
                ("primary", C.c_uint8 * 4), ("secondary", C.c_uint8 * 4)]


assert C.sizeof(_Prim) == 176


def render(scene: Scene, index: int, depth, rgb, labels, device: int = 0):
    """Renders camera keyframe `index` into device tensors (HxW f32, HxWx3 u8, HxW u8)."""
    t, cam = scene.camera[index]
    arr = (_Prim * len(scene.prims))()
    for i, p in enumerate(scene.prims):
        Rw, tw = _inverse(*_pose_at(p, t))
        w2o = np.concatenate([Rw.reshape(9), tw])
        q = arr[i]
        q.shape, q.dynamic, q.checker = p.shape, int(p.dynamic), int(p.checker)
        q.a[:] = list(p.a)
        q.b[:] = list(p.b)
        q.cell = p.cell
        q.w2o[:] = list(w2o)
        q.primary[:] = list(p.primary) + [0]
        q.secondary[:] = list(p.secondary) + [0]
    pose = (C.c_double * 12)(*cam)
    L.check(L.load().rf_synth_render(arr, len(scene.prims), pose, C.byref(scene.intrinsics), C.c_double(scene.noise),
                                     C.c_double(scene.dropout), C.c_uint64(scene.seed), C.c_uint64(index),
                                     C.c_void_p(depth.data_ptr()), C.c_void_p(rgb.data_ptr()),
                                     C.c_void_p(labels.data_ptr()), device))
