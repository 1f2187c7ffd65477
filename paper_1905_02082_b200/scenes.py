"""Synthetic scene scripts (the reference's `SceneScript` text format,
proj/include/tsdfslam/synth.hpp:43-67) for the parity tests and the bench.

`room_script` restates the acceptance room of proj/tests/acceptance.cpp:82-113;
`BENCH_CONFIGS` define the BASELINE.json workloads C1/C2 (640x480, 1 cm).
"""
from __future__ import annotations

import math

import numpy as np


def _quat_axis_angle(axis, angle):
    a = np.asarray(axis, dtype=np.float64)
    a = a / np.linalg.norm(a)
    s = math.sin(angle / 2.0)
    return np.array([math.cos(angle / 2.0), a[0] * s, a[1] * s, a[2] * s])


def _quat_mul(p, q):
    w1, x1, y1, z1 = p
    w2, x2, y2, z2 = q
    return np.array([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2, w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2, w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2])


def _camera_line(t, p, q):
    return "camera %.6f %.6f %.6f %.6f %.9f %.9f %.9f %.9f\n" % (t, p[0], p[1], p[2], q[1], q[2], q[3], q[0])


ROOM_PRIMITIVES = (
    "primitive room static box 0 0 0 2.2 1.4 2.2 albedo checker 0.45 225 225 225 45 45 45\n"
    "primitive pillar static box 1.9 -0.85 1.2 0.25 0.55 0.25 albedo checker 0.2 210 80 80 80 80 210\n"
    "primitive ball static sphere -1.6 0.9 1.82 0.35 albedo checker 0.3 240 200 60 60 90 200\n"
    "primitive crate static box -0.2 -1.1 1.6 0.45 0.3 0.35 albedo checker 0.25 90 210 120 40 60 40\n")


def room_script(with_mover=False, width=320, height=240, frames=30, noise=0.001, seed=42):
    """proj/tests/acceptance.cpp:82-113 (RoomScript) at a chosen resolution."""
    f = 262.5 * width / 320.0
    s = "intrinsics %.6f %.6f %.6f %.6f %d %d 5000\n" % (f, f, width / 2.0 - 0.5, height / 2.0 - 0.5, width, height)
    s += "noise %g 0.0\n" % noise
    s += "seed %d\n" % seed
    s += ROOM_PRIMITIVES
    if with_mover:
        s += "primitive mover dynamic sphere 0 0 0 0.55 albedo uniform 235 90 60\n"
        s += "keyframe mover 0 1.05 0.05 1.30 0 0 0 1\n"
        s += "keyframe mover %.9f 0.95 0.05 1.30 0 0 0 1\n" % (1.0 / 30.0)
        s += "keyframe mover %.9f -0.10 0.05 1.30 0 0 0 1\n" % (29.0 / 30.0)
    for i in range(frames):
        t = i / 30.0
        p = (-0.45 + 0.022 * i, 0.08 * math.sin(0.21 * i), -1.35 + 0.012 * i)
        yaw = (18.0 + 0.9 * i) * math.pi / 180.0
        pitch = 2.5 * math.sin(0.3 * i) * math.pi / 180.0
        q = _quat_mul(_quat_axis_angle([0, 1, 0], yaw), _quat_axis_angle([1, 0, 0], pitch))
        s += _camera_line(t, p, q)
    return s


def bench_script(dynamic=True, width=640, height=480, frames=200, noise=0.001, seed=43):
    """BASELINE.json configs[0]/[1]: the acceptance room at 640x480 with a
    smooth 30 Hz hand-held orbit (about 1.6 cm and 1 degree per frame); the
    dynamic variant adds two boxes that cross the view (C2)."""
    f = 525.0 * width / 640.0
    s = "intrinsics %.6f %.6f %.6f %.6f %d %d 5000\n" % (f, f, width / 2.0 - 0.5, height / 2.0 - 0.5, width, height)
    s += "noise %g 0.0\n" % noise
    s += "seed %d\n" % seed
    s += ROOM_PRIMITIVES
    duration = frames / 30.0
    if dynamic:
        s += "primitive box_a dynamic box 0 0 0 0.2 0.35 0.2 albedo checker 0.15 235 90 60 60 60 60\n"
        s += "keyframe box_a 0 -1.5 0.1 1.6 0 0 0 1\n"
        s += "keyframe box_a %.9f 1.4 0.1 1.6 0 0 0 1\n" % duration
        s += "primitive box_b dynamic box 0 0 0 0.25 0.25 0.25 albedo checker 0.2 60 90 235 230 230 60\n"
        s += "keyframe box_b 0 1.3 -0.8 1.9 0 0 0 1\n"
        s += "keyframe box_b %.9f -1.3 -0.8 0.9 0 0 0 1\n" % duration
    for i in range(frames):
        t = i / 30.0
        ph = 2.0 * math.pi * i / frames
        p = (-0.3 + 0.5 * math.sin(ph), 0.08 * math.sin(0.21 * i), -1.0 + 0.4 * (1.0 - math.cos(ph)))
        yaw = (18.0 + 35.0 * math.sin(ph)) * math.pi / 180.0
        pitch = 2.5 * math.sin(0.3 * i) * math.pi / 180.0
        q = _quat_mul(_quat_axis_angle([0, 1, 0], yaw), _quat_axis_angle([1, 0, 0], pitch))
        s += _camera_line(t, p, q)
    return s


def large_scene_script(frames=500, width=640, height=480, noise=0.001, seed=45):
    """BASELINE.json configs[2] (C3): a scaled room,
    box half-extents 6 x 2 x 6 m, with props (12 pillars, crates, spheres) and
    500 frames at 30 Hz along half of a 2.5 m circle looking outward and a little down
    (walls 3.5-6 m away, props 1-3 m, the floor in view). Run with 0.5 cm voxels and a 2^22-entry hash: about
    a million 8^3 bricks (4 GB), far beyond the 126 MB L2."""
    f = 525.0 * width / 640.0
    s = "intrinsics %.6f %.6f %.6f %.6f %d %d 5000\n" % (f, f, width / 2.0 - 0.5, height / 2.0 - 0.5, width, height)
    s += "noise %g 0.0\n" % noise
    s += "seed %d\n" % seed
    s += "primitive hall static box 0 0 0 6 2 6 albedo checker 0.5 220 220 210 50 50 60\n"
    for i in range(12):  # pillars on a 4 m circle, 30 degrees apart: always some in view
        a = 2.0 * math.pi * (i + 0.5) / 12.0
        s += ("primitive pillar%d static box %.4f 0 %.4f 0.18 2 0.18 albedo checker 0.2 %d 90 90 60 60 %d\n"
              % (i, 4.0 * math.sin(a), 4.0 * math.cos(a), 120 + 10 * i, 110 + 10 * i))
    for i in range(6):  # crates on the floor and spheres at eye height between the path and the walls
        a = 2.0 * math.pi * i / 6.0
        if i % 2:
            s += ("primitive ball%d static sphere %.4f %.4f %.4f 0.45 albedo checker 0.25 240 200 60 60 90 200\n"
                  % (i, 3.4 * math.sin(a), 0.2 + 0.1 * i, 3.4 * math.cos(a)))
        else:
            s += ("primitive crate%d static box %.4f 1.4 %.4f 0.5 0.6 0.4 albedo checker 0.3 90 210 120 40 60 40\n"
                  % (i, 3.4 * math.sin(a), 3.4 * math.cos(a)))
    for i in range(frames):
        t = i / 30.0
        th = math.pi * i / 500.0  # half a turn in 500 frames: ~1.6 cm and ~0.5 degree per frame
        p = (2.5 * math.sin(th), 0.3 + 0.1 * math.sin(0.13 * i), 2.5 * math.cos(th))
        yaw = th + 0.15 * math.sin(0.02 * i)
        pitch = (8.0 + 3.0 * math.sin(0.3 * i)) * math.pi / 180.0  # looking a little down: floor in view
        q = _quat_mul(_quat_axis_angle([0, 1, 0], yaw), _quat_axis_angle([1, 0, 0], pitch))
        s += _camera_line(t, p, q)
    return s


def corner_scene():
    """proj/tests/test_registration.cpp:157-162."""
    return ("intrinsics 40 40 31.5 23.5 64 48 5000\n"
            "primitive room static box 0 0 0 1.6 1.6 1.6 albedo checker 0.4 210 210 210 60 60 60\n"
            "primitive ball static sphere 0.55 0.1 0.95 0.25 albedo uniform 230 90 90\n"
            "camera 0.0 0 0 0 0 0.258819 0 0.965926\n")


def pipeline_static_scene(frames=7):
    """proj/tests/test_pipeline.cpp:31-56."""
    s = ("intrinsics 40 40 31.5 23.5 64 48 5000\n"
         "primitive room static box 0 0 0 1.6 1.2 1.6 albedo checker 0.4 230 230 230 40 40 40\n"
         "primitive pillar static box 0.5 0 0.9 0.15 0.6 0.15 albedo checker 0.25 200 60 60 60 60 200\n")
    for i in range(frames):
        q = _quat_axis_angle([0, 1, 0], (30.0 + 0.2 * i) * math.pi / 180.0)
        s += _camera_line(i / 30.0, (0.005 * i, 0.002 * i, 0.003 * i), q)
    return s


BENCH_CONFIGS = {
    # RoomScript(false) at 640x480 with the default K, its path extended to 50 frames
    "C1": dict(dynamic=False, frames=50, seed=42, voxel=0.01),
    # the acceptance room + 2 crossing boxes on a closed 200-frame orbit
    "C2": dict(dynamic=True, frames=200, seed=43, voxel=0.01),
    # large scene at 0.5 cm with the 4M-entry hash (large_scene_script)
    "C3": dict(dynamic=False, frames=500, seed=45, voxel=0.005, hash_capacity=1 << 22, max_blocks=4000000),
    # 1280x720, K = (1050, 1050, 639.5, 359.5), 3 levels, mesh export at the end
    "C4": dict(dynamic=True, frames=1000, seed=44, voxel=0.01, width=1280, height=720),
}


def config_script(name: str, seed: int | None = None) -> str:
    """Scene script of BASELINE.json workload `name` (C1..C4); `seed`
    overrides the noise seed (independent replicas)."""
    c = BENCH_CONFIGS[name]
    s = c["seed"] if seed is None else seed
    if name == "C1":
        return room_script(False, 640, 480, frames=c["frames"], seed=s)
    if name == "C3":
        return large_scene_script(frames=c["frames"], seed=s)
    if name == "C4":
        return bench_script(dynamic=True, width=c["width"], height=c["height"], frames=c["frames"], seed=s)
    return bench_script(dynamic=c["dynamic"], frames=c["frames"], seed=s)
