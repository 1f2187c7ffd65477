"""ORACLE — test infrastructure only.

ctypes wrapper over ``liboracle.so``, the CPU restatement of the reference
hot path (``/root/reference/proj``; see ``oracle.hpp``). Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / ``--impl
reference`` leg may import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (g++, -ffp-contract=off)."""
    if force or not os.path.exists(_LIB_PATH):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    else:  # rebuild when a source is newer than the library
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB_PATH


class OIntr(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("depth_scale", C.c_double)]


class OVolCfg(C.Structure):
    _fields_ = [("voxel_size", C.c_double), ("truncation", C.c_double), ("block_side", C.c_int32),
                ("max_weight", C.c_int32), ("carve_weight", C.c_int32), ("pad0", C.c_int32),
                ("min_depth", C.c_double), ("max_depth", C.c_double), ("carve_clip", C.c_double),
                ("max_blocks", C.c_uint64)]


class ORegCfg(C.Structure):
    _fields_ = [("color_weight", C.c_double), ("pyramid_levels", C.c_int32), ("max_iterations", C.c_int32),
                ("lm_lambda_init", C.c_double), ("lm_lambda_up", C.c_double), ("lm_lambda_down", C.c_double),
                ("convergence_eps", C.c_double), ("min_valid_residuals", C.c_int32), ("threads", C.c_int32),
                ("huber_depth", C.c_double), ("huber_color", C.c_double)]


class OMaskCfg(C.Structure):
    _fields_ = [("gamma", C.c_double), ("truncation", C.c_double), ("theta", C.c_double),
                ("erode_radius", C.c_int32), ("dilate_radius", C.c_int32), ("connectivity", C.c_int32),
                ("pad0", C.c_int32), ("free_space", C.c_double)]


class OPipeCfg(C.Structure):
    _fields_ = [("volume", OVolCfg), ("reg", ORegCfg), ("mask", OMaskCfg), ("refine_enabled", C.c_int32),
                ("refine_window", C.c_int32), ("far_value", C.c_double), ("bisection_iterations", C.c_int32),
                ("dynamics_enabled", C.c_int32), ("threads", C.c_int32), ("pad0", C.c_int32)]


class OStats(C.Structure):
    _fields_ = [("frame_index", C.c_uint64), ("timestamp", C.c_double), ("tracking_lost", C.c_int32),
                ("converged", C.c_int32), ("registrations", C.c_int32), ("iterations", C.c_int32),
                ("valid_residuals", C.c_uint64), ("masked_pixels", C.c_uint64), ("final_error", C.c_double),
                ("runtime_ms", C.c_double)]


OK, INVALID, LOST, RESOURCE, OTHER = 0, 1, 2, 3, 5


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


class TrackingLost(OracleError):
    pass


class ResourceLimit(OracleError):
    pass


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        vp = C.c_void_p
        L.o_last_error.restype = C.c_char_p
        for name in ("ov_create", "oh_create", "o_scene_parse", "op_create", "op_volume", "o_mesh_extract"):
            getattr(L, name).restype = vp
        for name in ("ov_num_blocks", "ov_hash_capacity", "ov_last_dda_visits", "oh_size", "oh_capacity",
                     "o_scene_num_frames", "op_losses", "o_hash_coord", "ov_set_voxels"):
            getattr(L, name).restype = C.c_uint64
        L.o_hash_coord.argtypes = [C.c_int32, C.c_int32, C.c_int32]
        for name in ("ov_destroy", "oh_destroy", "o_scene_free", "op_destroy", "o_mesh_free", "ov_num_blocks",
                     "ov_hash_capacity", "ov_last_dda_visits", "oh_size", "oh_capacity", "o_scene_num_frames",
                     "op_losses", "op_finalize"):
            getattr(L, name).argtypes = [vp]
        _lib = L
    return _lib


def _check(code: int):
    if code == OK:
        return
    msg = lib().o_last_error().decode()
    if code == LOST:
        raise TrackingLost(code, msg)
    if code == RESOURCE:
        raise ResourceLimit(code, msg)
    if code == INVALID:
        raise ValueError(msg)
    raise OracleError(code, msg)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def intr(fx=525.0, fy=525.0, cx=319.5, cy=239.5, width=640, height=480, depth_scale=5000.0) -> OIntr:
    return OIntr(fx, fy, cx, cy, width, height, depth_scale)


def small_intrinsics(width=32, height=24, focal=30.0) -> OIntr:  # test_util.hpp:12-21
    return OIntr(focal, focal, width / 2.0 - 0.5, height / 2.0 - 0.5, width, height, 5000.0)


def vol_cfg(**kw) -> OVolCfg:
    c = OVolCfg(0.01, 0.1, 8, 64, 1, 0, 0.1, 5.0, 4.0, 1000000)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def reg_cfg(**kw) -> ORegCfg:
    c = ORegCfg(0.025, 3, 20, 1e-4, 10.0, 2.0, 1e-5, 100, 1, 0.0, 0.0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def mask_cfg(**kw) -> OMaskCfg:
    c = OMaskCfg(0.5, 0.1, 0.007, 2, 2, 4, 0, 0.0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def pipe_cfg(refine=False, window=10, dynamics=True, threads=1, volume=None, reg=None, mask=None) -> OPipeCfg:
    v = volume or vol_cfg()
    m = mask or mask_cfg()
    m.truncation = v.truncation
    return OPipeCfg(v, reg or reg_cfg(), m, int(refine), window, 8.0, 8, int(dynamics), threads, 0)


IDENTITY = np.array([1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0], dtype=np.float64)


def pose_array(R=None, t=None) -> np.ndarray:
    out = IDENTITY.copy()
    if R is not None:
        out[:9] = np.asarray(R, dtype=np.float64).reshape(9)
    if t is not None:
        out[9:] = np.asarray(t, dtype=np.float64)
    return out


def pose_matrix(p) -> np.ndarray:
    p = np.asarray(p, dtype=np.float64)
    M = np.eye(4)
    M[:3, :3] = p[:9].reshape(3, 3)
    M[:3, 3] = p[9:]
    return M


def matrix_pose(M) -> np.ndarray:
    M = np.asarray(M, dtype=np.float64)
    return pose_array(M[:3, :3], M[:3, 3])


def expmap(xi) -> np.ndarray:
    out = np.zeros(12)
    lib().o_expmap(_p(_f64(xi)), _p(out))
    return out


def logmap(pose) -> np.ndarray:
    out = np.zeros(6)
    lib().o_logmap(_p(_f64(pose)), _p(out))
    return out


def hash_coord(x, y, z) -> int:
    return lib().o_hash_coord(int(x), int(y), int(z))


def walk_segment(a, b, ext) -> np.ndarray:
    cells = np.zeros((4096, 3), dtype=np.int32)
    n = lib().o_walk_segment(_p(_f64(a)), _p(_f64(b)), C.c_double(ext), _p(cells), 4096)
    return cells[:n].copy()


class HashMap:
    """CoordHashMap (spatial_hash.hpp:23-86)."""

    def __init__(self, capacity=1024):
        self.h = C.c_void_p(lib().oh_create(C.c_uint64(capacity)))

    def __del__(self):
        if getattr(self, "h", None) is not None and self.h.value:
            lib().oh_destroy(self.h)
            self.h = None

    def size(self):
        return lib().oh_size(self.h)

    def capacity(self):
        return lib().oh_capacity(self.h)

    def insert(self, coords, values):
        coords = _i32(coords).reshape(-1, 3)
        values = np.ascontiguousarray(values, dtype=np.uint32)
        n = coords.shape[0]
        out = np.zeros(n, dtype=np.uint32)
        ins = np.zeros(n, dtype=np.uint8)
        lib().oh_insert_batch(self.h, C.c_uint64(n), _p(coords), _p(values), _p(out), _p(ins))
        return out, ins.astype(bool)

    def find(self, coords):
        coords = _i32(coords).reshape(-1, 3)
        n = coords.shape[0]
        vals = np.zeros(n, dtype=np.uint32)
        found = np.zeros(n, dtype=np.uint8)
        lib().oh_find_batch(self.h, C.c_uint64(n), _p(coords), _p(vals), _p(found))
        return vals, found.astype(bool)


VOXEL_DTYPE = np.dtype([("sdf", "<f4"), ("weight", "u1"), ("r", "u1"), ("g", "u1"), ("b", "u1")])


class Volume:
    """TsdfVolume restated (tsdf_volume.hpp:67-134)."""

    def __init__(self, cfg: OVolCfg | None = None, _borrowed=None, **kw):
        if _borrowed is not None:
            self.v, self.owned = C.c_void_p(_borrowed), False
            self._cfg = cfg
            return
        self._cfg = cfg or vol_cfg(**kw)
        self.v = C.c_void_p(lib().ov_create(C.byref(self._cfg)))
        if not self.v.value:
            raise ValueError(lib().o_last_error().decode())
        self.owned = True

    def __del__(self):
        if getattr(self, "owned", False) and self.v.value:
            lib().ov_destroy(self.v)
            self.v = None

    @property
    def config(self):
        return self._cfg

    def num_blocks(self) -> int:
        return lib().ov_num_blocks(self.v)

    def hash_capacity(self) -> int:
        return lib().ov_hash_capacity(self.v)

    def last_dda_visits(self) -> int:
        return lib().ov_last_dda_visits(self.v)

    def allocate_block(self, coord) -> bool:
        r = lib().ov_allocate_block(self.v, *[int(c) for c in coord])
        if r < 0:
            _check(-r)
        return r == 1

    def export(self, with_voxels=True):
        """Blocks in allocation order: (coords[n,3] i32, voxels[n,side^3] VOXEL_DTYPE)."""
        n = self.num_blocks()
        side = self._cfg.block_side
        coords = np.zeros((n, 3), dtype=np.int32)
        vox = np.zeros((n, side ** 3), dtype=VOXEL_DTYPE) if with_voxels else None
        lib().ov_export(self.v, _p(coords), _p(vox))
        return coords, vox

    def set_voxels(self, coords, voxels) -> int:
        coords = _i32(coords).reshape(-1, 3)
        voxels = np.ascontiguousarray(voxels, dtype=VOXEL_DTYPE)
        return lib().ov_set_voxels(self.v, C.c_uint64(coords.shape[0]), _p(coords), _p(voxels))

    def get_voxels(self, coords):
        coords = _i32(coords).reshape(-1, 3)
        n = coords.shape[0]
        vox = np.zeros(n, dtype=VOXEL_DTYPE)
        found = np.zeros(n, dtype=np.uint8)
        lib().ov_get_voxels(self.v, C.c_uint64(n), _p(coords), _p(vox), _p(found))
        return vox, found.astype(bool)

    def hash_occupancy(self, cap: int) -> np.ndarray:
        bm = np.zeros(cap, dtype=np.uint8)
        _check(lib().ov_hash_occupancy(self.v, C.c_uint64(cap), _p(bm)))
        return bm

    def allocate_for_frame(self, depth, k: OIntr, pose, mask=None):
        _check(lib().ov_allocate_for_frame(self.v, _p(_f32(depth)), C.byref(k), _p(_f64(pose)),
                                           _p(None if mask is None else _u8(mask))))

    def integrate(self, depth, rgb, k: OIntr, pose, mask=None, threads=1):
        _check(lib().ov_integrate(self.v, _p(_f32(depth)), _p(None if rgb is None else _u8(rgb)), C.byref(k),
                                  _p(_f64(pose)), _p(None if mask is None else _u8(mask)), threads))

    def carve(self, depth, k: OIntr, pose, threads=1):
        _check(lib().ov_carve(self.v, _p(_f32(depth)), C.byref(k), _p(_f64(pose)), threads))

    def sample(self, points, mode=0):
        pts = _f64(points).reshape(-1, 3)
        n = pts.shape[0]
        val = np.zeros(n)
        grad = np.zeros((n, 3))
        valid = np.zeros(n, dtype=np.uint8)
        lib().ov_sample(self.v, mode, C.c_uint64(n), _p(pts), _p(val), _p(grad), _p(valid))
        return val, grad, valid.astype(bool)

    # --- registration entry points (registration.hpp:42-85) -------------
    def linearize(self, depth, rgb, k, pose, cfg=None, mask=None):
        cfg = cfg or reg_cfg()
        H = np.zeros(36)
        b = np.zeros(6)
        errs = np.zeros(3)
        valid = C.c_uint64()
        deg = C.c_int32()
        _check(lib().o_linearize(self.v, _p(_f32(depth)), _p(None if rgb is None else _u8(rgb)), C.byref(k),
                                 _p(_f64(pose)), C.byref(cfg), _p(None if mask is None else _u8(mask)), _p(H),
                                 _p(b), _p(errs), C.byref(valid), C.byref(deg)))
        return dict(H=H.reshape(6, 6), b=b, depth_error=errs[0], color_error=errs[1], error=errs[2],
                    valid=valid.value, degenerate=bool(deg.value))

    def evaluate_depth_error(self, depth, k, pose, mask=None, threads=1):
        sq = np.zeros((k.height, k.width), dtype=np.float32)
        valid = np.zeros((k.height, k.width), dtype=np.uint8)
        err = C.c_double()
        _check(lib().o_evaluate_depth_error(self.v, _p(_f32(depth)), C.byref(k), _p(_f64(pose)),
                                            _p(None if mask is None else _u8(mask)), threads, C.byref(err),
                                            _p(sq), _p(valid)))
        return err.value, sq, valid

    def evaluate_color_error(self, depth, rgb, k, pose, mask=None, threads=1):
        err = C.c_double()
        _check(lib().o_evaluate_color_error(self.v, _p(_f32(depth)), _p(_u8(rgb)), C.byref(k), _p(_f64(pose)),
                                            _p(None if mask is None else _u8(mask)), threads, C.byref(err)))
        return err.value

    def register(self, depth, rgb, k, init, mask=None, cfg=None):
        cfg = cfg or reg_cfg()
        pose = np.zeros(12)
        conv = C.c_int32()
        its = C.c_int32()
        valid = C.c_uint64()
        fe = C.c_double()
        sq = np.zeros((k.height, k.width), dtype=np.float32)
        rv = np.zeros((k.height, k.width), dtype=np.uint8)
        _check(lib().o_register(self.v, _p(_f32(depth)), _p(None if rgb is None else _u8(rgb)), C.byref(k),
                                _p(_f64(init)), _p(None if mask is None else _u8(mask)), C.byref(cfg), _p(pose),
                                C.byref(conv), C.byref(its), C.byref(valid), C.byref(fe), _p(sq), _p(rv)))
        return dict(pose=pose, converged=bool(conv.value), iterations=its.value, valid_residuals=valid.value,
                    final_error=fe.value, res_sq=sq, res_valid=rv)

    def raycast(self, pose, k, bisections=8, threads=1):
        out = np.zeros((k.height, k.width), dtype=np.float32)
        _check(lib().o_raycast(self.v, _p(_f64(pose)), C.byref(k), bisections, threads, _p(out)))
        return out

    def save(self, path):
        """TsdfVolume::Save (tsdf_volume.cpp:375-403)."""
        lib().ov_save.argtypes = [C.c_void_p, C.c_char_p]
        _check(lib().ov_save(self.v, str(path).encode()))

    @classmethod
    def load(cls, path):
        """TsdfVolume::Load (tsdf_volume.cpp:405-449)."""
        lib().ov_load.restype = C.c_void_p
        lib().ov_load.argtypes = [C.c_char_p]
        h = lib().ov_load(str(path).encode())
        if not h:
            raise OracleError(OTHER, lib().o_last_error().decode())
        self = cls.__new__(cls)
        self.v, self.owned = C.c_void_p(h), True
        self._cfg = vol_cfg()
        lib().ov_config(self.v, C.byref(self._cfg))
        return self

    def write_ply(self, path, min_weight=2, threads=1):
        """ExtractMesh then WritePly (mesh.cpp:149-225)."""
        m = C.c_void_p(lib().o_mesh_extract(self.v, min_weight, threads))
        lib().o_mesh_write_ply.argtypes = [C.c_void_p, C.c_char_p]
        try:
            _check(lib().o_mesh_write_ply(m, str(path).encode()))
        finally:
            lib().o_mesh_free(m)

    def extract_mesh(self, min_weight=2, threads=1):
        m = C.c_void_p(lib().o_mesh_extract(self.v, min_weight, threads))
        nv, nf = C.c_uint64(), C.c_uint64()
        lib().o_mesh_counts(m, C.byref(nv), C.byref(nf))
        v = np.zeros((nv.value, 3), dtype=np.float32)
        c = np.zeros((nv.value, 3), dtype=np.uint8)
        f = np.zeros((nf.value, 3), dtype=np.int32)
        lib().o_mesh_copy(m, _p(v), _p(c), _p(f))
        lib().o_mesh_free(m)
        return v, c, f


def build_pyramid(depth, rgb, k, levels, mask=None):
    sizes = [(k.width >> l) * (k.height >> l) for l in range(levels)]
    tot = sum(sizes)
    od = np.zeros(tot, dtype=np.float32)
    oi = np.zeros(tot, dtype=np.float32)
    om = np.zeros(tot, dtype=np.uint8)
    ok = np.zeros(4 * levels)
    _check(lib().o_build_pyramid(_p(_f32(depth)), _p(None if rgb is None else _u8(rgb)),
                                 _p(None if mask is None else _u8(mask)), C.byref(k), levels, _p(od), _p(oi),
                                 _p(om), _p(ok)))
    out, off = [], 0
    for l in range(levels):
        w, h = k.width >> l, k.height >> l
        n = w * h
        out.append(dict(depth=od[off:off + n].reshape(h, w), intensity=oi[off:off + n].reshape(h, w),
                        mask=om[off:off + n].reshape(h, w), intr=ok[4 * l:4 * l + 4]))
        off += n
    return out


def ldlt6(A, rhs):
    x = np.zeros(6)
    ok = lib().o_ldlt6(_p(_f64(A)), _p(_f64(rhs)), _p(x))
    return x, bool(ok)


def threshold(res_sq, res_valid, gamma=0.5, truncation=0.1):
    res_sq = _f32(res_sq)
    h, w = res_sq.shape
    out = np.zeros((h, w), dtype=np.uint8)
    lib().o_threshold(_p(res_sq), _p(_u8(res_valid)), w, h, C.c_double(gamma), C.c_double(truncation), _p(out))
    return out


def erode(mask, radius):
    m = _u8(mask)
    h, w = m.shape
    out = np.zeros_like(m)
    lib().o_erode(_p(m), w, h, radius, _p(out))
    return out


def dilate(mask, radius):
    m = _u8(mask)
    h, w = m.shape
    out = np.zeros_like(m)
    lib().o_dilate(_p(m), w, h, radius, _p(out))
    return out


def floodfill(seeds, depth, theta, connectivity=4):
    s = _u8(seeds)
    h, w = s.shape
    out = np.zeros_like(s)
    _check(lib().o_floodfill(_p(s), _p(_f32(depth)), w, h, C.c_double(theta), connectivity, _p(out)))
    return out


def build_mask(res_sq, res_valid, depth, cfg=None):
    cfg = cfg or mask_cfg()
    res_sq = _f32(res_sq)
    h, w = res_sq.shape
    out = np.zeros((h, w), dtype=np.uint8)
    _check(lib().o_build_mask(_p(res_sq), _p(_u8(res_valid)), _p(_f32(depth)), w, h, C.byref(cfg), _p(out)))
    return out


def render_virtual_depth(entries, view, k, vcfg, bisections=8, far_value=8.0, threads=1):
    """RenderVirtualDepth (depth_refinement.cpp:22-80) + RefineDepth (:82-93).
    entries: list of dicts {depth, rgb (or None), mask (or None), pose}; returns
    (virtual depth, refined depth of entries[0])."""
    n = len(entries)
    keep = []
    D = (C.c_void_p * n)()
    R = (C.c_void_p * n)()
    M = (C.c_void_p * n)()
    for i, e in enumerate(entries):
        d = _f32(e["depth"])
        keep.append(d)
        D[i] = d.ctypes.data
        if e.get("rgb") is not None:
            r = _u8(e["rgb"])
            keep.append(r)
            R[i] = r.ctypes.data
        if e.get("mask") is not None:
            m = _u8(e["mask"])
            keep.append(m)
            M[i] = m.ctypes.data
    poses = _f64(np.concatenate([np.asarray(e["pose"], np.float64) for e in entries]))
    out = np.zeros((k.height, k.width), np.float32)
    ref = np.zeros((k.height, k.width), np.float32)
    _check(lib().o_render_virtual_depth(n, D, R, M, _p(poses), C.byref(k), C.byref(vcfg), _p(_f64(view)),
                                        bisections, C.c_double(far_value), threads, _p(out), _p(ref)))
    return out, ref


class Scene:
    """SceneScript + RenderFrame restated (synth.hpp:43-74)."""

    def __init__(self, text: str):
        self.s = C.c_void_p(lib().o_scene_parse(text.encode()))
        if not self.s.value:
            raise ValueError(lib().o_last_error().decode())
        self.k = OIntr()
        lib().o_scene_intrinsics(self.s, C.byref(self.k))

    def __del__(self):
        if getattr(self, "s", None) is not None and self.s.value:
            lib().o_scene_free(self.s)
            self.s = None

    def __len__(self):
        return lib().o_scene_num_frames(self.s)

    def camera(self, i):
        t = C.c_double()
        pose = np.zeros(12)
        lib().o_scene_camera(self.s, C.c_uint64(i), C.byref(t), _p(pose))
        return t.value, pose

    def world_to_object(self, prim, t):
        """World-to-object pose of primitive `prim` at time t (synth.cpp:155-158)."""
        L = lib()
        L.o_scene_w2o.argtypes = [C.c_void_p, C.c_uint64, C.c_double, C.c_void_p]
        pose = np.zeros(12)
        L.o_scene_w2o(self.s, C.c_uint64(prim), C.c_double(t), _p(pose))
        return pose

    def render(self, i):
        h, w = self.k.height, self.k.width
        depth = np.zeros((h, w), dtype=np.float32)
        rgb = np.zeros((h, w, 3), dtype=np.uint8)
        td = np.zeros((h, w), dtype=np.float32)
        labels = np.zeros((h, w), dtype=np.uint8)
        _check(lib().o_render(self.s, C.c_uint64(i), _p(depth), _p(rgb), _p(td), _p(labels)))
        return dict(depth=depth, rgb=rgb, true_depth=td, labels=labels, timestamp=self.camera(i)[0])


class Pipeline:
    """Pipeline restated (pipeline.hpp:51-86)."""

    def __init__(self, cfg: OPipeCfg | None = None):
        self.cfg = cfg or pipe_cfg()
        self.p = C.c_void_p(lib().op_create(C.byref(self.cfg)))
        if not self.p.value:
            raise ValueError(lib().o_last_error().decode())
        self.trajectory = []
        self.stats = []

    def __del__(self):
        if getattr(self, "p", None) is not None and self.p.value:
            lib().op_destroy(self.p)
            self.p = None

    def process_frame(self, depth, rgb, k, timestamp=0.0):
        st = OStats()
        pose = np.zeros(12)
        _check(lib().op_process(self.p, C.c_double(timestamp), _p(_f32(depth)),
                                _p(None if rgb is None else _u8(rgb)), C.byref(k), C.byref(st), _p(pose)))
        s = {f: getattr(st, f) for f, _ in OStats._fields_}
        self.trajectory.append((timestamp, pose))
        self.stats.append(s)
        return s, pose

    def finalize(self):
        _check(lib().op_finalize(self.p))

    def volume(self) -> Volume:
        v = Volume(self.cfg.volume, _borrowed=lib().op_volume(self.p))
        v._owner = self  # keep the pipeline alive while the view exists
        return v

    def losses(self) -> int:
        return lib().op_losses(self.p)

    def last_mask(self, k):
        out = np.zeros((k.height, k.width), dtype=np.uint8)
        has = lib().op_last_mask(self.p, _p(out))
        return out if has else None

    def last_residuals(self, k):
        sq = np.zeros((k.height, k.width), dtype=np.float32)
        v = np.zeros((k.height, k.width), dtype=np.uint8)
        lib().op_last_residuals(self.p, _p(sq), _p(v))
        return sq, v


# ------------------------------------------------------------------ evaluation (evaluation.hpp:12-50)
def _traj(tr):
    """(timestamps[n], poses[n,12]) or a list of (timestamp, pose12)."""
    if isinstance(tr, tuple) and len(tr) == 2 and np.ndim(tr[1]) == 2:
        ts, poses = tr
    else:
        ts = [t for t, _ in tr]
        poses = [np.asarray(p, np.float64).reshape(12) for _, p in tr]
    ts = _f64(np.asarray(ts, np.float64).reshape(-1))
    poses = _f64(np.asarray(poses, np.float64).reshape(-1, 12))
    return ts, poses


def ate_rmse(estimated, ground_truth, max_dt=0.02):
    """AteRmse (evaluation.cpp:26-62) -> (rmse, alignment pose12, pairs)."""
    et, ep = _traj(estimated)
    gt, gp = _traj(ground_truth)
    rmse = C.c_double()
    al = np.zeros(12)
    n = C.c_uint64()
    code = lib().o_ate_rmse(_p(et), _p(ep), C.c_uint64(len(et)), _p(gt), _p(gp), C.c_uint64(len(gt)),
                            C.c_double(max_dt), C.byref(rmse), _p(al), C.byref(n))
    if code:
        raise OracleError(code, lib().o_last_error().decode())
    return rmse.value, al, n.value


def rpe_over_time(estimated, ground_truth, delta=1.0, max_dt=0.02):
    """RpeOverTime (evaluation.cpp:64-92) -> (timestamps, translation errors)."""
    et, ep = _traj(estimated)
    gt, gp = _traj(ground_truth)
    cap = max(len(et), 1)
    ts = np.zeros(cap)
    err = np.zeros(cap)
    f = lib().o_rpe_over_time
    f.restype = C.c_int64
    n = f(_p(et), _p(ep), C.c_uint64(len(et)), _p(gt), _p(gp), C.c_uint64(len(gt)), C.c_double(delta),
          C.c_double(max_dt), _p(ts), _p(err), C.c_uint64(cap))
    if n < 0:
        raise ValueError("delta must be positive")
    return ts[:n].copy(), err[:n].copy()


def nearest_distances(queries, reference):
    """NearestDistances (evaluation.cpp:203-217): f32 xyz clouds -> f64 distances."""
    q = _f32(np.asarray(queries, np.float32).reshape(-1, 3))
    r = _f32(np.asarray(reference, np.float32).reshape(-1, 3))
    out = np.zeros(len(q))
    code = lib().o_nearest_distances(_p(q), C.c_uint64(len(q)), _p(r), C.c_uint64(len(r)), _p(out))
    if code:
        raise ValueError(lib().o_last_error().decode())
    return out


def distance_cdf(distances, bin_edges):
    """DistanceCdf (evaluation.cpp:219-236)."""
    d = _f64(np.asarray(distances, np.float64).reshape(-1))
    e = _f64(np.asarray(bin_edges, np.float64).reshape(-1))
    out = np.zeros(len(e))
    code = lib().o_distance_cdf(_p(d), C.c_uint64(len(d)), _p(e), C.c_uint64(len(e)), _p(out))
    if code:
        raise ValueError(lib().o_last_error().decode())
    return out
