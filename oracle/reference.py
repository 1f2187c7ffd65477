"""ORACLE — test infrastructure only.

ctypes wrapper over ``_ref/libtsdfslam_ref.so``: the REFERENCE's own,
unmodified sources (/root/reference/proj/src) compiled by ``make ref`` against
the Eigen / doctest / libpng stand-ins in ``ref_shim/`` (see ref_capi.cpp).
It pins the restatement (oracle.py) to the reference code
(tests/test_reference_build.py) and is bench.py's reference arm when present
("kind": "reference"). Same structs and calling conventions as oracle.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from . import oracle as O

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libtsdfslam_ref.so")
REF_SOURCES = "/root/reference/proj"
_lib = None


def buildable() -> bool:
    return os.path.isdir(os.path.join(REF_SOURCES, "src"))


def build() -> str | None:
    """make ref (only where /root/reference exists; the GPU box uses the prebuilt library)."""
    if buildable():
        subprocess.check_call(["make", "-s", "-j8", "-C", _HERE, "ref"])
        # the reference's own test sources against the B200 host layer (needs the CUDA library)
        if os.path.exists(os.path.join(os.path.dirname(_HERE), "paper_1905_02082_b200", "librefusion_b200.so")):
            subprocess.check_call(["make", "-s", "-j8", "-C", _HERE, "refsuite"])
    return LIB_PATH if os.path.exists(LIB_PATH) else None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} not built (make -C oracle ref)")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.r_last_error.restype = C.c_char_p
        for name in ("r_scene_parse", "r_pipe_create"):
            getattr(L, name).restype = vp
        for name in ("r_scene_num_frames", "r_pipe_num_blocks"):
            getattr(L, name).restype = C.c_uint64
            getattr(L, name).argtypes = [vp]
        L.r_scene_parse.argtypes = [C.c_char_p]
        for name in ("r_scene_free", "r_pipe_destroy", "r_pipe_finalize"):
            getattr(L, name).argtypes = [vp]
        L.r_pipe_save.argtypes = [vp, C.c_char_p]
        L.r_pipe_write_ply.argtypes = [vp, C.c_char_p, C.c_int]
        _lib = L
    return _lib


def _check(code):
    if code == 0:
        return
    msg = lib().r_last_error().decode()
    if code == O.LOST:
        raise O.TrackingLost(code, msg)
    if code == O.RESOURCE:
        raise O.ResourceLimit(code, msg)
    if code == O.INVALID:
        raise ValueError(msg)
    raise O.OracleError(code, msg)


class Scene:
    """SceneScript::Parse + RenderFrame of the reference (synth.cpp)."""

    def __init__(self, text: str):
        self.s = C.c_void_p(lib().r_scene_parse(text.encode()))
        if not self.s.value:
            raise ValueError(lib().r_last_error().decode())
        self.k = O.OIntr()
        lib().r_scene_intrinsics(self.s, C.byref(self.k))

    def __del__(self):
        if getattr(self, "s", None) is not None and self.s.value:
            lib().r_scene_free(self.s)
            self.s = None

    def __len__(self):
        return lib().r_scene_num_frames(self.s)

    def render(self, i):
        h, w = self.k.height, self.k.width
        depth = np.zeros((h, w), np.float32)
        rgb = np.zeros((h, w, 3), np.uint8)
        td = np.zeros((h, w), np.float32)
        labels = np.zeros((h, w), np.uint8)
        _check(lib().r_render(self.s, C.c_uint64(i), O._p(depth), O._p(rgb), O._p(td), O._p(labels)))
        return dict(depth=depth, rgb=rgb, true_depth=td, labels=labels)


class Pipeline:
    """tsdfslam::Pipeline of the reference (pipeline.hpp:51-86)."""

    def __init__(self, cfg: O.OPipeCfg | None = None):
        self.cfg = cfg or O.pipe_cfg()
        self.p = C.c_void_p(lib().r_pipe_create(C.byref(self.cfg)))
        if not self.p.value:
            raise ValueError(lib().r_last_error().decode())

    def __del__(self):
        if getattr(self, "p", None) is not None and self.p.value:
            lib().r_pipe_destroy(self.p)
            self.p = None

    def process_frame(self, depth, rgb, k, timestamp=0.0):
        st = O.OStats()
        pose = np.zeros(12)
        _check(lib().r_pipe_process(self.p, C.c_double(timestamp), O._p(O._f32(depth)),
                                    O._p(None if rgb is None else O._u8(rgb)), C.byref(k), C.byref(st), O._p(pose)))
        return {f: getattr(st, f) for f, _ in O.OStats._fields_}, pose

    def finalize(self):
        _check(lib().r_pipe_finalize(self.p))

    def num_blocks(self):
        return lib().r_pipe_num_blocks(self.p)

    def export(self, with_voxels=True):
        n = self.num_blocks()
        coords = np.zeros((n, 3), np.int32)
        vox = np.zeros((n, 512), dtype=O.VOXEL_DTYPE) if with_voxels else None
        lib().r_pipe_export(self.p, O._p(coords), O._p(vox))
        return coords, vox

    def save(self, path):
        _check(lib().r_pipe_save(self.p, str(path).encode()))

    def write_ply(self, path, min_weight=2):
        _check(lib().r_pipe_write_ply(self.p, str(path).encode(), int(min_weight)))
