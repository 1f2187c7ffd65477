"""Python mirror of the reference's tracker / map interfaces
(proj/include/tsdfslam) over the C ABI. Same names and argument meaning as the
reference, snake_case; exceptions map onto TrackingLostError /
ResourceLimitError / ValueError like errors.hpp. Images are numpy arrays
(host, copied in) or CUDA torch tensors (device, read in place)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from ._lib import ResourceLimitError, RfError, TrackingLostError, UnsupportedError  # noqa: F401

VOXEL_DTYPE = np.dtype([("sdf", "<f4"), ("weight", "u1"), ("r", "u1"), ("g", "u1"), ("b", "u1")])
IDENTITY = np.array([1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0], dtype=np.float64)


def _lib():
    return L.load()


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


# ------------------------------------------------------------------ configs
def intrinsics(fx=525.0, fy=525.0, cx=319.5, cy=239.5, width=640, height=480, depth_scale=5000.0):
    """CameraIntrinsics (geometry.hpp:11-38) with the reference defaults."""
    return L.rf_intrinsics(fx, fy, cx, cy, width, height, depth_scale)


def volume_config(**kw) -> L.rf_volume_config:
    """VolumeConfig (tsdf_volume.hpp:14-29) defaults."""
    c = L.rf_volume_config(0.01, 0.1, 8, 64, 1, 0, 0.1, 5.0, 4.0, 1000000, 0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def registration_config(**kw) -> L.rf_registration_config:
    """RegistrationConfig (registration.hpp:13-23) defaults; huber_depth /
    huber_color > 0 turn on the Huber-weighted extension (off = reference)."""
    c = L.rf_registration_config(0.025, 3, 20, 1e-4, 10.0, 2.0, 1e-5, 100, 1, 0.0, 0.0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def mask_config(**kw) -> L.rf_mask_config:
    """MaskConfig (dynamics_mask.hpp:10-17) defaults; free_space > 0 turns on
    the free-space seed extension (off = reference)."""
    c = L.rf_mask_config(0.5, 0.1, 0.007, 2, 2, 4, 0, 0.0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def pipeline_config(refine=True, window=10, dynamics=True, threads=1, volume=None, registration=None, mask=None,
                    far_value=8.0, bisection_iterations=8):
    """PipelineConfig (config.hpp:12-24) with the reference's defaults,
    including RefinementConfig::enabled = true (depth_refinement.hpp:13); the
    acceptance / bench configuration (TrackingConfig, acceptance.cpp:136)
    passes refine=False."""
    v = volume or volume_config()
    m = mask or mask_config()
    m.truncation = v.truncation
    return L.rf_pipeline_config(v, registration or registration_config(), m, int(refine), window, far_value,
                                bisection_iterations, int(dynamics), threads, 0)


# ------------------------------------------------------------------ frames
@dataclass
class Frame:
    """One RGB-D measurement (image.hpp:94-103)."""
    depth: object  # HxW float32 numpy array or CUDA tensor
    rgb: object = None  # HxWx3 uint8 numpy array or CUDA tensor
    intrinsics: L.rf_intrinsics = field(default_factory=intrinsics)
    timestamp: float = 0.0

    def c(self) -> L.rf_frame:
        f = L.rf_frame()
        f.intrinsics = self.intrinsics
        f.timestamp = self.timestamp
        dev = _is_cuda(self.depth)
        f.memory = L.RF_MEMORY_DEVICE if dev else L.RF_MEMORY_HOST
        if dev:
            k = self.intrinsics
            _check_device_tensor(self.depth, "float32", (k.height, k.width), "depth")
            if self.rgb is not None:
                _check_device_tensor(self.rgb, "uint8", (k.height, k.width, 3), "rgb", self.depth.device)
            _producer_done(self.depth)
            f.depth = self.depth.data_ptr()
            f.rgb = None if self.rgb is None else self.rgb.data_ptr()
            self._keep = ()
        else:
            d = np.ascontiguousarray(self.depth, dtype=np.float32)
            rgb = None if self.rgb is None else np.ascontiguousarray(self.rgb, dtype=np.uint8)
            self._keep = (d, rgb)
            f.depth = d.ctypes.data
            f.rgb = None if rgb is None else rgb.ctypes.data
        return f


def _is_cuda(x):
    return hasattr(x, "is_cuda") and x.is_cuda


def _check_device_tensor(t, dtype, shape, name, device=None):
    """A CUDA tensor handed to the C ABI as a raw pointer: exact dtype, dense
    row-major layout, the expected size, on the frame's device."""
    if str(t.dtype) != "torch." + dtype:
        raise ValueError(f"{name}: expected a torch.{dtype} tensor, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: tensor must be contiguous")
    if tuple(t.shape) != tuple(shape) and t.numel() != int(np.prod(shape)):
        raise ValueError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    if device is not None and t.device != device:
        raise ValueError(f"{name}: tensor is on {t.device}, the frame on {device}")


def _producer_done(t):
    """The library reads device inputs on its own streams (refusion_b200.h):
    finish the work torch has queued for them first."""
    import torch

    torch.cuda.current_stream(t.device).synchronize()


def _mask_ptr(mask, frame: Frame):
    if mask is None:
        return None, None
    if _is_cuda(frame.depth):
        k = frame.intrinsics
        _check_device_tensor(mask, "uint8", (k.height, k.width), "mask", frame.depth.device)
        _producer_done(mask)
        return C.c_void_p(mask.data_ptr()), mask
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    return C.c_void_p(m.ctypes.data), m


# ------------------------------------------------------------------ volume
class TsdfVolume:
    """TsdfVolume (tsdf_volume.hpp:67-134) on the GPU."""

    def __init__(self, config: L.rf_volume_config | None = None, device: int = 0, _handle=None, **kw):
        self.config = config or volume_config(**kw)
        self.device = device
        if _handle is not None:
            self.h = _handle
            self._owned = False
            return
        h = C.c_void_p()
        L.check(_lib().rf_volume_create(C.byref(self.config), device, C.byref(h)))
        self.h = h
        self._owned = True

    def close(self):
        if getattr(self, "_owned", False) and self.h:
            _lib().rf_volume_destroy(self.h)
            self.h = None
            self._owned = False

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def num_blocks(self) -> int:
        out = C.c_uint64()
        L.check(_lib().rf_volume_num_blocks(self.h, C.byref(out)))
        return out.value

    def hash_capacity(self) -> int:
        out = C.c_uint64()
        L.check(_lib().rf_volume_hash_capacity(self.h, C.byref(out)))
        return out.value

    def allocate_blocks(self, coords):
        c = _i32(coords).reshape(-1, 3)
        created = np.zeros(len(c), dtype=np.int32)
        L.check(_lib().rf_volume_allocate_blocks(self.h, _p(c), C.c_uint64(len(c)), _p(created)))
        return created

    def allocate_block(self, coord) -> bool:  # AllocateBlock (tsdf_volume.cpp:64-77)
        return bool(self.allocate_blocks([coord])[0] == 1)

    def allocate_for_frame(self, frame: Frame, pose, mask=None):
        f = frame.c()
        mp, _keep = _mask_ptr(mask, frame)
        L.check(_lib().rf_volume_allocate_for_frame(self.h, C.byref(f), _p(_f64(pose)), mp))

    def integrate(self, frame: Frame, pose, mask=None):
        f = frame.c()
        mp, _keep = _mask_ptr(mask, frame)
        L.check(_lib().rf_volume_integrate(self.h, C.byref(f), _p(_f64(pose)), mp))

    def carve(self, frame: Frame, pose):  # CarveFreeSpace
        f = frame.c()
        L.check(_lib().rf_volume_carve(self.h, C.byref(f), _p(_f64(pose))))

    def sample(self, points, mode=0):
        pts = _f64(points).reshape(-1, 3)
        n = len(pts)
        val = np.zeros(n)
        grad = np.zeros((n, 3))
        valid = np.zeros(n, dtype=np.uint8)
        L.check(_lib().rf_volume_sample(self.h, mode, _p(pts), C.c_uint64(n), _p(val), _p(grad), _p(valid)))
        return val, grad, valid.astype(bool)

    def get_voxels(self, coords):
        c = _i32(coords).reshape(-1, 3)
        vox = np.zeros(len(c), dtype=VOXEL_DTYPE)
        found = np.zeros(len(c), dtype=np.uint8)
        L.check(_lib().rf_volume_get_voxels(self.h, _p(c), C.c_uint64(len(c)), _p(vox), _p(found)))
        return vox, found.astype(bool)

    def set_voxels(self, coords, voxels) -> int:
        c = _i32(coords).reshape(-1, 3)
        v = np.ascontiguousarray(voxels, dtype=VOXEL_DTYPE)
        missing = C.c_uint64()
        L.check(_lib().rf_volume_set_voxels(self.h, _p(c), C.c_uint64(len(c)), _p(v), C.byref(missing)))
        return missing.value

    def export(self, with_voxels=True):
        """blocks() in pool order: coords (n,3) i32 and voxels (n,512) VOXEL_DTYPE."""
        cnt = C.c_uint64()
        L.check(_lib().rf_volume_export_blocks(self.h, None, None, C.c_uint64(0), C.byref(cnt)))
        n = cnt.value
        coords = np.zeros((n, 3), dtype=np.int32)
        vox = np.zeros((n, 512), dtype=VOXEL_DTYPE) if with_voxels else None
        L.check(_lib().rf_volume_export_blocks(self.h, _p(coords), _p(vox), C.c_uint64(n), C.byref(cnt)))
        return coords, vox

    def find_block(self, block_coord):
        """FindBlock (tsdf_volume.cpp:59-62): the brick's 512 voxels (x fastest)
        or None when the block is not allocated (one hash probe on the device)."""
        c = _i32(block_coord).reshape(3)
        vox = np.zeros(512, dtype=VOXEL_DTYPE)
        found = C.c_int32()
        L.check(_lib().rf_volume_find_block(self.h, _p(c), _p(vox), C.byref(found)))
        return vox if found.value else None

    def write_block(self, block_coord, voxels) -> bool:
        """Writes an allocated brick's 512 voxels; False when it does not exist."""
        c = _i32(block_coord).reshape(3)
        v = np.ascontiguousarray(voxels, dtype=VOXEL_DTYPE).reshape(512)
        found = C.c_int32()
        L.check(_lib().rf_volume_write_block(self.h, _p(c), _p(v), C.byref(found)))
        return bool(found.value)

    def check(self):
        """rf_diag_volume_check: {name: count} of structural invariant violations (all 0 expected)."""
        e = (C.c_uint64 * 5)()
        L.check(_lib().rf_diag_volume_check(self.h, e))
        return dict(zip(("bad_value", "bad_brick_slot", "duplicate_key", "bad_link", "pending_key"), e))

    def hash_occupancy(self) -> np.ndarray:
        bm = np.zeros(self.hash_capacity(), dtype=np.uint8)
        L.check(_lib().rf_volume_hash_occupancy(self.h, _p(bm)))
        return bm

    def reset(self):
        L.check(_lib().rf_volume_reset(self.h))

    def save(self, path: str):
        L.check(_lib().rf_volume_save(self.h, path.encode()))

    @staticmethod
    def load(path: str, device: int = 0) -> "TsdfVolume":
        h = C.c_void_p()
        L.check(_lib().rf_volume_load(path.encode(), device, C.byref(h)))
        v = TsdfVolume.__new__(TsdfVolume)
        v.h, v._owned, v.device = h, True, device
        v.config = volume_config()  # header values are held by the handle
        return v

    # --- registration.hpp:42-85 --------------------------------------------
    def linearize(self, frame: Frame, pose, config=None, mask=None):
        cfg = config or registration_config()
        f = frame.c()
        mp, _keep = _mask_ptr(mask, frame)
        out = L.rf_linearize_result()
        L.check(_lib().rf_linearize(self.h, C.byref(f), _p(_f64(pose)), C.byref(cfg), mp, C.byref(out)))
        return dict(H=np.array(out.H).reshape(6, 6), b=np.array(out.b), depth_error=out.depth_error,
                    color_error=out.color_error, error=out.error, valid=out.valid_count,
                    degenerate=bool(out.degenerate))

    def evaluate_depth_error(self, frame: Frame, pose, mask=None):
        f = frame.c()
        mp, _keep = _mask_ptr(mask, frame)
        k = frame.intrinsics
        sq = np.zeros((k.height, k.width), dtype=np.float32)
        valid = np.zeros((k.height, k.width), dtype=np.uint8)
        err = C.c_double()
        L.check(_lib().rf_evaluate_depth_error(self.h, C.byref(f), _p(_f64(pose)), mp, C.byref(err), _p(sq),
                                               _p(valid)))
        return err.value, sq, valid

    def evaluate_color_error(self, frame: Frame, pose, mask=None):
        f = frame.c()
        mp, _keep = _mask_ptr(mask, frame)
        err = C.c_double()
        L.check(_lib().rf_evaluate_color_error(self.h, C.byref(f), _p(_f64(pose)), mp, C.byref(err)))
        return err.value

    def register(self, frame: Frame, initial_pose, mask=None, config=None):
        cfg = config or registration_config()
        f = frame.c()
        mp, _keep = _mask_ptr(mask, frame)
        k = frame.intrinsics
        out = L.rf_registration_result()
        sq = np.zeros((k.height, k.width), dtype=np.float32)
        rv = np.zeros((k.height, k.width), dtype=np.uint8)
        L.check(_lib().rf_register(self.h, C.byref(f), _p(_f64(initial_pose)), mp, C.byref(cfg), C.byref(out),
                                   _p(sq), _p(rv)))
        return dict(pose=np.array(out.pose), converged=bool(out.converged), iterations=out.iterations,
                    valid_residuals=out.valid_residuals, final_error=out.final_error, res_sq=sq, res_valid=rv)

    def raycast(self, pose, k: L.rf_intrinsics, bisections=8):
        out = np.zeros((k.height, k.width), dtype=np.float32)
        L.check(_lib().rf_raycast(self.h, _p(_f64(pose)), C.byref(k), bisections, _p(out)))
        return out

    def extract_mesh(self, min_weight=2, ply_path=None):
        """ExtractMesh (mesh.hpp:25): (vertices f32 (N,3), colours u8 (N,3),
        faces i32 (M,3)) in the reference's order; optionally WritePly."""
        m = C.c_void_p()
        L.check(_lib().rf_volume_extract_mesh(self.h, int(min_weight), C.byref(m)))
        try:
            nv, nf = C.c_uint64(), C.c_uint64()
            L.check(_lib().rf_mesh_counts(m, C.byref(nv), C.byref(nf)))
            v = np.zeros((nv.value, 3), np.float32)
            c = np.zeros((nv.value, 3), np.uint8)
            f = np.zeros((nf.value, 3), np.int32)
            L.check(_lib().rf_mesh_copy(m, _p(v), _p(c), _p(f)))
            if ply_path is not None:
                L.check(_lib().rf_mesh_write_ply(m, str(ply_path).encode()))
        finally:
            _lib().rf_mesh_destroy(m)
        return v, c, f


def build_pyramid(frame: Frame, mask=None, levels=3, device=0):
    """BuildPyramid (registration.hpp:42, registration.cpp:119-182) on the GPU:
    one dict per level {intrinsics, depth, intensity (None without colour),
    mask (None without a mask)}, level 0 first."""
    k = frame.intrinsics
    sizes = [(k.width >> l) * (k.height >> l) for l in range(max(levels, 0))]
    tot = max(sum(sizes), 1)
    f = frame.c()
    mp, _keep = _mask_ptr(mask, frame)
    depth = np.zeros(tot, np.float32)
    inten = np.zeros(tot, np.float32) if frame.rgb is not None else None
    mout = np.zeros(tot, np.uint8) if mask is not None else None
    ks = (L.rf_intrinsics * max(levels, 1))()
    L.check(_lib().rf_build_pyramid(C.byref(f), mp, int(levels), device, _p(depth), _p(inten), _p(mout), ks))
    out, off = [], 0
    for l, n in enumerate(sizes):
        w, h = k.width >> l, k.height >> l
        out.append(dict(intrinsics=ks[l], depth=depth[off:off + n].reshape(h, w),
                        intensity=None if inten is None else inten[off:off + n].reshape(h, w),
                        mask=None if mout is None else mout[off:off + n].reshape(h, w)))
        off += n
    return out


# ------------------------------------------------------------------ refinement
def render_virtual_depth(frames, poses, masks, view_pose, k: L.rf_intrinsics, volume=None, bisections=8,
                         far_value=8.0, device=0):
    """RenderVirtualDepth + RefineDepth (depth_refinement.cpp:22-93): frames
    is a list of Frame, masks a list of u8 images or None. Returns (virtual
    depth, refined depth of frames[0])."""
    n = len(frames)
    fr = (L.rf_frame * n)(*[f.c() for f in frames])
    keep = list(frames)
    M = None
    if masks is not None:
        M = (C.c_void_p * n)()
        for i, m in enumerate(masks):
            if m is not None:
                a = np.ascontiguousarray(m, np.uint8)
                keep.append(a)
                M[i] = a.ctypes.data
    P = _f64(np.concatenate([np.asarray(p, np.float64) for p in poses]))
    virt = np.zeros((k.height, k.width), np.float32)
    ref = np.zeros((k.height, k.width), np.float32)
    vc = volume or volume_config()
    L.check(_lib().rf_render_virtual_depth(fr, _p(P), M, n, _p(_f64(view_pose)), C.byref(k), C.byref(vc),
                                           bisections, C.c_double(far_value), device, _p(virt), _p(ref)))
    return virt, ref


# ------------------------------------------------------------------ mask
def mask_stages(res_sq, res_valid, depth, config=None, stages=15, device=0):
    """BuildMask (stages=15) or any subset of its stages (dynamics_mask.hpp:21-41)."""
    cfg = config or mask_config()
    rv = np.ascontiguousarray(res_valid, dtype=np.uint8)
    h, w = rv.shape
    sq = None if res_sq is None else np.ascontiguousarray(res_sq, dtype=np.float32)
    d = np.ascontiguousarray(depth, dtype=np.float32)
    out = np.zeros((h, w), dtype=np.uint8)
    n = C.c_uint64()
    L.check(_lib().rf_mask_stages(_p(sq), _p(rv), _p(d), w, h, C.byref(cfg), stages, device, _p(out), C.byref(n)))
    return out


def threshold_residuals(res_sq, res_valid, config=None):
    return mask_stages(res_sq, res_valid, np.zeros_like(res_sq, dtype=np.float32), config, 1)


def erode(mask, radius):
    return mask_stages(None, mask, np.zeros(np.shape(mask), np.float32), mask_config(erode_radius=radius), 2)


def dilate(mask, radius):
    return mask_stages(None, mask, np.zeros(np.shape(mask), np.float32), mask_config(dilate_radius=radius), 8)


def floodfill_depth(seeds, depth, theta, connectivity=4):
    return mask_stages(None, seeds, depth, mask_config(theta=theta, connectivity=connectivity), 4)


def build_mask(res_sq, res_valid, depth, config=None):
    return mask_stages(res_sq, res_valid, depth, config, 15)


# ------------------------------------------------------------------ pipeline
class Pipeline:
    """Pipeline (pipeline.hpp:51-86) with the whole ProcessFrame on the GPU."""

    def __init__(self, config: L.rf_pipeline_config | None = None, device: int = 0):
        self.config = config or pipeline_config()
        h = C.c_void_p()
        L.check(_lib().rf_pipeline_create(C.byref(self.config), device, C.byref(h)))
        self.h = h
        self.device = device
        self.stats = []

    def close(self):
        if getattr(self, "h", None):
            _lib().rf_pipeline_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def process_frame(self, frame: Frame):
        f = frame.c()
        st = L.rf_frame_stats()
        pose = (C.c_double * 12)()
        L.check(_lib().rf_pipeline_process_frame(self.h, C.byref(f), C.byref(st), pose))
        s = {k: getattr(st, k) for k, _ in L.rf_frame_stats._fields_}
        self.stats.append(s)
        return s, np.array(pose)

    def process_frames(self, frames):
        """ProcessFrame over a list of Frame with the GPU work enqueued back to
        back (RunSequence without a host round trip per frame): (stats list,
        poses (n, 12))."""
        n = len(frames)
        fr = (L.rf_frame * n)(*[f.c() for f in frames])
        st = (L.rf_frame_stats * n)()
        poses = np.zeros((n, 12))
        L.check(_lib().rf_pipeline_process_frames(self.h, fr, C.c_uint64(n), st, _p(poses)))
        out = [{k: getattr(st[i], k) for k, _ in L.rf_frame_stats._fields_} for i in range(n)]
        self.stats.extend(out)
        return out, poses

    def process_frame_raw(self, f: L.rf_frame, st: L.rf_frame_stats, pose):
        """Minimal-overhead call for timing loops (no Python-side conversion)."""
        return _lib().rf_pipeline_process_frame(self.h, C.byref(f), C.byref(st), pose)

    def finalize(self):
        L.check(_lib().rf_pipeline_finalize(self.h))

    def volume(self) -> TsdfVolume:
        h = C.c_void_p()
        L.check(_lib().rf_pipeline_volume(self.h, C.byref(h)))
        v = TsdfVolume(self.config.volume, self.device, _handle=h)
        v._owner = self
        return v

    def tracking_losses(self) -> int:
        out = C.c_uint64()
        L.check(_lib().rf_pipeline_tracking_losses(self.h, C.byref(out)))
        return out.value

    def trajectory(self):
        cnt = C.c_uint64()
        L.check(_lib().rf_pipeline_trajectory(self.h, None, None, C.c_uint64(0), C.byref(cnt)))
        ts = np.zeros(cnt.value)
        poses = np.zeros((cnt.value, 12))
        L.check(_lib().rf_pipeline_trajectory(self.h, _p(ts), _p(poses), cnt, C.byref(cnt)))
        return ts, poses

    def last_mask(self):
        has = C.c_int32()
        L.check(_lib().rf_pipeline_last_mask(self.h, None, C.byref(has)))
        if not has.value:
            return None
        return has

    def window_size(self) -> int:
        out = C.c_uint64()
        L.check(_lib().rf_pipeline_window_size(self.h, C.byref(out)))
        return out.value

    def set_debug_images(self, enable=True):
        L.check(_lib().rf_pipeline_set_debug_images(self.h, int(enable)))

    def last_refinement(self, k, with_virtual=False):
        """FrameDebug::virtual_depth / refined_depth of the last IntegrateFront:
        (frame_index, virtual or None, refined) or None."""
        has = C.c_int32()
        idx = C.c_uint64()
        virt = np.zeros((k.height, k.width), np.float32) if with_virtual else None
        ref = np.zeros((k.height, k.width), np.float32)
        L.check(_lib().rf_pipeline_last_refinement(self.h, _p(virt) if with_virtual else None, _p(ref),
                                                   C.byref(idx), C.byref(has)))
        return (idx.value, virt, ref) if has.value else None

    def last_mask_image(self, k):
        out = np.zeros((k.height, k.width), dtype=np.uint8)
        has = C.c_int32()
        L.check(_lib().rf_pipeline_last_mask(self.h, _p(out), C.byref(has)))
        return out if has.value else None

    def last_residuals(self, k):
        sq = np.zeros((k.height, k.width), dtype=np.float32)
        v = np.zeros((k.height, k.width), dtype=np.uint8)
        L.check(_lib().rf_pipeline_last_residuals(self.h, _p(sq), _p(v)))
        return sq, v

    def last_counters(self):
        c = L.rf_frame_counters()
        L.check(_lib().rf_pipeline_last_counters(self.h, C.byref(c)))
        return {k: getattr(c, k) for k, _ in L.rf_frame_counters._fields_}


# ------------------------------------------------------------------ evaluation (evaluation.hpp:12-50)
def _traj(tr):
    """(timestamps[n], poses[n,12]) (Pipeline.trajectory()) or a list of (timestamp, pose12)."""
    if isinstance(tr, tuple) and len(tr) == 2 and np.ndim(tr[1]) == 2:
        ts, poses = tr
    else:
        ts = [t for t, _ in tr]
        poses = [np.asarray(p, np.float64).reshape(12) for _, p in tr]
    return _f64(np.asarray(ts, np.float64).reshape(-1)), _f64(np.asarray(poses, np.float64).reshape(-1, 12))


def ate_rmse(estimated, ground_truth, max_dt=0.02):
    """AteRmse (evaluation.cpp:26-62) -> (rmse, alignment pose12, pairs).
    Fewer than 3 associated pairs raise RfError (a RuntimeError)."""
    et, ep = _traj(estimated)
    gt, gp = _traj(ground_truth)
    rmse, n = C.c_double(), C.c_uint64()
    al = np.zeros(12)
    L.check(_lib().rf_ate_rmse(_p(et), _p(ep), C.c_uint64(len(et)), _p(gt), _p(gp), C.c_uint64(len(gt)),
                               C.c_double(max_dt), C.byref(rmse), _p(al), C.byref(n)))
    return rmse.value, al, n.value


def rpe_over_time(estimated, ground_truth, delta=1.0, max_dt=0.02):
    """RpeOverTime (evaluation.cpp:64-92) -> (timestamps, translation errors)."""
    et, ep = _traj(estimated)
    gt, gp = _traj(ground_truth)
    cap = max(len(et), 1)
    ts, err, n = np.zeros(cap), np.zeros(cap), C.c_uint64()
    L.check(_lib().rf_rpe_over_time(_p(et), _p(ep), C.c_uint64(len(et)), _p(gt), _p(gp), C.c_uint64(len(gt)),
                                    C.c_double(delta), C.c_double(max_dt), _p(ts), _p(err), C.c_uint64(cap),
                                    C.byref(n)))
    return ts[:n.value].copy(), err[:n.value].copy()


def nearest_distances(queries, reference, device=0):
    """NearestDistances (evaluation.cpp:203-217) on the GPU. f32 xyz clouds as
    numpy arrays (-> numpy f64) or CUDA torch tensors (-> CUDA f64 tensor)."""
    if _is_cuda(queries) or _is_cuda(reference):
        import torch
        q = queries.reshape(-1, 3).to(torch.float32).contiguous()
        r = reference.reshape(-1, 3).to(torch.float32).contiguous()
        if r.device != q.device:
            raise ValueError("queries and reference must be on the same device")
        out = torch.empty(q.shape[0], dtype=torch.float64, device=q.device)
        _producer_done(q)  # the conversions above ran on torch's stream
        L.check(_lib().rf_nearest_distances(C.c_void_p(q.data_ptr()), C.c_uint64(q.shape[0]),
                                            C.c_void_p(r.data_ptr()), C.c_uint64(r.shape[0]),
                                            L.RF_MEMORY_DEVICE, q.device.index or 0, C.c_void_p(out.data_ptr())))
        return out
    q = np.ascontiguousarray(np.asarray(queries, np.float32).reshape(-1, 3))
    r = np.ascontiguousarray(np.asarray(reference, np.float32).reshape(-1, 3))
    out = np.zeros(len(q))
    L.check(_lib().rf_nearest_distances(_p(q), C.c_uint64(len(q)), _p(r), C.c_uint64(len(r)), L.RF_MEMORY_HOST,
                                        device, _p(out)))
    return out


def distance_cdf(distances, bin_edges, device=0):
    """DistanceCdf (evaluation.cpp:219-236): cumulative percentage at or below
    each (ascending) edge; distances numpy or a CUDA tensor."""
    e = _f64(np.asarray(bin_edges, np.float64).reshape(-1))
    out = np.zeros(len(e))
    if _is_cuda(distances):
        d = distances.reshape(-1).double().contiguous()
        _producer_done(d)
        L.check(_lib().rf_distance_cdf(C.c_void_p(d.data_ptr()), C.c_uint64(d.numel()), L.RF_MEMORY_DEVICE,
                                       d.device.index or 0, _p(e), C.c_uint64(len(e)), _p(out)))
        return out
    d = _f64(np.asarray(distances, np.float64).reshape(-1))
    L.check(_lib().rf_distance_cdf(_p(d) if len(d) else None, C.c_uint64(len(d)), L.RF_MEMORY_HOST, device,
                                   _p(e) if len(e) else None, C.c_uint64(len(e)), _p(out) if len(out) else None))
    return out
