"""Shared fixtures restating proj/tests/test_util.hpp (FillVolume, MakeFrame,
WavyProbe, SmallPose) on numpy, usable for both the oracle and the CUDA path."""
from __future__ import annotations

import math

import numpy as np

from oracle import oracle as O

VOXEL_DTYPE = O.VOXEL_DTYPE


def floor_div(a, b):
    return a // b  # python floor division == FloorDiv for b > 0


def fill_voxels(voxel_size, block_side, lo, hi, sdf, intensity=None, weight=32):
    """test_util.hpp:26-62: returns (block_coords, voxel_coords, voxel_records)."""
    s = voxel_size
    vlo = [int(math.floor(lo[i] / s)) for i in range(3)]
    vhi = [int(math.ceil(hi[i] / s)) for i in range(3)]
    blocks = []
    for bz in range(floor_div(vlo[2], block_side), floor_div(vhi[2], block_side) + 1):
        for by in range(floor_div(vlo[1], block_side), floor_div(vhi[1], block_side) + 1):
            for bx in range(floor_div(vlo[0], block_side), floor_div(vhi[0], block_side) + 1):
                blocks.append((bx, by, bz))
    zz, yy, xx = np.meshgrid(np.arange(vlo[2], vhi[2] + 1), np.arange(vlo[1], vhi[1] + 1),
                             np.arange(vlo[0], vhi[0] + 1), indexing="ij")
    coords = np.stack([xx.ravel(), yy.ravel(), zz.ravel()], axis=1).astype(np.int32)
    centers = (coords.astype(np.float64) + 0.5) * s
    rec = np.zeros(coords.shape[0], dtype=VOXEL_DTYPE)
    rec["sdf"] = np.array([sdf(p) for p in centers], dtype=np.float64).astype(np.float32)
    rec["weight"] = weight
    if intensity is not None:
        vals = np.clip(np.array([intensity(p) for p in centers]), 0.0, 255.0)
        gray = np.array([int(math.floor(v + 0.5)) for v in vals], dtype=np.uint8)  # lround, v >= 0
        rec["r"] = gray
        rec["g"] = gray
        rec["b"] = gray
    return np.array(blocks, dtype=np.int32), coords, rec


def fill_volume(vol, lo, hi, sdf, intensity=None, weight=32):
    cfg = vol.config
    blocks, coords, rec = fill_voxels(cfg.voxel_size, cfg.block_side, lo, hi, sdf, intensity, weight)
    for b in blocks:
        vol.allocate_block(b)
    missing = vol.set_voxels(coords, rec)
    assert missing == 0
    return coords, rec


def make_frame(k, depth, gray=None):
    """test_util.hpp:65-88 -> (depth f32 HxW, rgb u8 HxWx3 or None)."""
    h, w = k.height, k.width
    d = np.zeros((h, w), dtype=np.float32)
    for v in range(h):
        for u in range(w):
            d[v, u] = np.float32(depth(u, v))
    rgb = None
    if gray is not None:
        rgb = np.zeros((h, w, 3), dtype=np.uint8)
        for v in range(h):
            for u in range(w):
                g = min(max(gray(u, v), 0.0), 255.0)
                rgb[v, u, :] = int(math.floor(g + 0.5))
    return d, rgb


def wavy_probe(p):  # test_util.hpp:91-94
    return 0.06 * math.sin(3.0 * p[0] + 0.7) * math.cos(2.0 * p[1] - 0.4) + 0.04 * math.sin(2.2 * p[2])


def wavy_probe_intensity(p):  # test_util.hpp:96-98
    return 120.0 + 70.0 * math.sin(1.7 * p[0] - 0.3) * math.cos(1.3 * p[2] + 0.2)


def axis_angle_matrix(axis, angle):
    a = np.asarray(axis, dtype=np.float64)
    a = a / np.linalg.norm(a)
    K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + math.sin(angle) * K + (1 - math.cos(angle)) * (K @ K)


def small_pose(t, axis, angle):  # test_util.hpp:100-103
    return O.pose_array(axis_angle_matrix(axis, angle), t)


def rotation_angle(pose):
    R = np.asarray(pose)[:9].reshape(3, 3)
    c = (np.trace(R) - 1.0) / 2.0
    return math.acos(max(-1.0, min(1.0, c)))


def compose(a, b):
    return O.matrix_pose(O.pose_matrix(a) @ O.pose_matrix(b))


def inverse(a):
    return O.matrix_pose(np.linalg.inv(O.pose_matrix(a)))


def quat_from_axis_angle(axis, angle):
    a = np.asarray(axis, dtype=np.float64)
    a = a / np.linalg.norm(a)
    s = math.sin(angle / 2)
    return np.array([math.cos(angle / 2), a[0] * s, a[1] * s, a[2] * s])  # w x y z


def quat_mul(p, q):
    w1, x1, y1, z1 = p
    w2, x2, y2, z2 = q
    return np.array([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2, w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2, w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2])


def ate_rmse(est, gt):
    """evaluation.cpp:26-62: closed-form rigid alignment of positions, RMSE."""
    A = np.array([p[9:] for p in est])
    B = np.array([p[9:] for p in gt])
    ca, cb = A.mean(0), B.mean(0)
    W = (B - cb).T @ (A - ca)
    U, _, Vt = np.linalg.svd(W)
    S = np.eye(3)
    if np.linalg.det(U @ Vt) < 0:
        S[2, 2] = -1
    R = U @ S @ Vt
    t = cb - R @ ca
    al = (R @ A.T).T + t
    return float(np.sqrt(np.mean(np.sum((al - B) ** 2, axis=1))))
