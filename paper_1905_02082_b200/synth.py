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


def _quat_to_R(w, x, y, z):  # Quaterniond::toRotationMatrix after normalize
    n = math.sqrt(w * w + x * x + y * y + z * z)
    w, x, y, z = w / n, x / n, y / n, z / n
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def _R_to_quat(R):
    t = np.trace(R)
    if t > 0:
        s = math.sqrt(t + 1.0) * 2
        return np.array([0.25 * s, (R[2, 1] - R[1, 2]) / s, (R[0, 2] - R[2, 0]) / s, (R[1, 0] - R[0, 1]) / s])
    i = int(np.argmax(np.diag(R)))
    j, k = (i + 1) % 3, (i + 2) % 3
    s = math.sqrt(R[i, i] - R[j, j] - R[k, k] + 1.0) * 2
    q = np.zeros(4)
    q[0] = (R[k, j] - R[j, k]) / s
    q[1 + i] = 0.25 * s
    q[1 + j] = (R[j, i] + R[i, j]) / s
    q[1 + k] = (R[k, i] + R[i, k]) / s
    return q


def _slerp(q0, q1, t):
    d = float(np.dot(q0, q1))
    if abs(d) >= 1 - 1e-15:
        s0, s1 = 1 - t, t
    else:
        th = math.acos(abs(d))
        s0, s1 = math.sin((1 - t) * th) / math.sin(th), math.sin(t * th) / math.sin(th)
    if d < 0:
        s1 = -s1
    return s0 * q0 + s1 * q1


def _pose_at(prim: Primitive, time: float):
    """Primitive::PoseAt (synth.cpp:35-45): object-to-world (R, t)."""
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
    q = _slerp(_R_to_quat(R0), _R_to_quat(R1), al)
    return _quat_to_R(*q), (1 - al) * p0 + al * p1


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
            target.keyframes.append((t, _quat_to_R(qw, qx, qy, qz), np.array([tx, ty, tz])))
        elif d == "camera":
            t = float(tok[1])
            tx, ty, tz, qx, qy, qz, qw = (float(x) for x in tok[2:9])
            pose = np.concatenate([_quat_to_R(qw, qx, qy, qz).reshape(9), [tx, ty, tz]])
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
        R, tr = _pose_at(p, t)
        Rt = R.T
        w2o = np.concatenate([Rt.reshape(9), -(Rt @ tr)])
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
