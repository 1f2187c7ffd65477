"""The C++ host layer (include/refusion_b200.hpp), which mirrors the
reference's tsdfslam classes over the C ABI: it compiles warning-free against
the header (CPU), and on the GPU a C++ caller driving Pipeline / RunSequence /
ExtractMesh reproduces the Python-ABI results bit for bit and the oracle's
poses within 1e-4, with the reference's exception types."""
import os
import shutil
import struct
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1905_02082_b200")
SRC = os.path.join(ROOT, "tests", "cpp", "host_layer_demo.cpp")
CXX = shutil.which("g++", path="/usr/bin") or shutil.which("g++")


def compile_demo(out):
    cmd = [CXX, "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"), SRC,
           "-L", LIBDIR, "-lrefusion_b200", f"-Wl,-rpath,{LIBDIR}", "-o", out]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_host_layer_compiles(tmp_path):
    if not os.path.exists(os.path.join(LIBDIR, "librefusion_b200.so")):
        pytest.skip("CUDA library not built")
    compile_demo(str(tmp_path / "demo"))
    # The header alone also compiles as C++17-free-standing include (no Eigen).
    probe = tmp_path / "probe.cpp"
    probe.write_text('#include "refusion_b200.hpp"\nint main() { tsdfslam_b200::PipelineConfig c; c.Sync();'
                     ' return c.refinement.window == 10 ? 0 : 1; }\n')
    subprocess.run([CXX, "-std=c++20", "-Wall", "-Wextra", "-Werror", "-pedantic", "-fsyntax-only", "-I",
                    os.path.join(ROOT, "include"), str(probe)], check=True)


def test_host_containers(tmp_path):
    """CoordHashMap / HashCoord, FrameWindow and RefineDepth: host-side code of the
    layer, checked against an ordered map and the reference's rules (no GPU)."""
    if not os.path.exists(os.path.join(LIBDIR, "librefusion_b200.so")):
        pytest.skip("CUDA library not built")
    exe = str(tmp_path / "containers")
    subprocess.run([CXX, "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "host_containers.cpp"), "-L", LIBDIR, "-lrefusion_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "host containers ok" in r.stdout, r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("refine,debug", [(False, True), (True, True), (False, False)])
def test_host_layer_pipeline_matches(tmp_path, refine, debug):
    from oracle import oracle as O
    from paper_1905_02082_b200 import api as G
    from paper_1905_02082_b200 import scenes
    from tests.test_gpu_parity import frame, pose_error

    exe = str(tmp_path / "demo")
    compile_demo(exe)
    s = O.Scene(scenes.room_script(with_mover=True, frames=8))
    frames = [s.render(i) for i in range(len(s))]
    k = s.k
    with open(tmp_path / "in.bin", "wb") as f:
        f.write(struct.pack("<3i4d", k.width, k.height, len(frames), k.fx, k.fy, k.cx, k.cy))
        for fr in frames:
            f.write(struct.pack("<d", fr["timestamp"]))
            f.write(np.ascontiguousarray(fr["depth"], np.float32).tobytes())
            f.write(np.ascontiguousarray(fr["rgb"], np.uint8).tobytes())
    args = [exe, str(tmp_path / "in.bin"), str(tmp_path / "out.bin")] + (["refine"] if refine else []) + \
        ([] if debug else ["nodebug"])
    r = subprocess.run(args, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    data = (tmp_path / "out.bin").read_bytes()
    n = struct.unpack_from("<i", data)[0]
    assert n == len(frames)
    rec = np.frombuffer(data, dtype=np.dtype([("t", "<f8"), ("pose", "<f8", 12), ("lost", "<i4"), ("regs", "<i4"),
                                              ("iters", "<i4"), ("masked", "<u8")]), count=n, offset=4)
    off = 4 + rec.nbytes
    nv, nf, nb = struct.unpack_from("<3Q", data, off)
    flags = struct.unpack_from("<3i", data, off + 24)
    calls, masks, refined = struct.unpack_from("<3Q", data, off + 36)
    assert flags == (1, 1, 1), "exception mapping"
    # one record per registered frame, plus one per IntegrateFront (window 3: all but the first frame)
    if debug:
        assert calls == (n - 1) + ((n - 1) if refine else 0) and refined == ((n - 1) if refine else 0)
    else:
        assert calls == 0

    gp = G.Pipeline(G.pipeline_config(refine=refine, window=3))
    op = O.Pipeline(O.pipe_cfg(refine=refine, window=3, reg=O.reg_cfg(threads=8)))
    for i, fr in enumerate(frames):
        sg, pg = gp.process_frame(frame(k, fr["depth"], fr["rgb"], fr["timestamp"]))
        so, po = op.process_frame(fr["depth"], fr["rgb"], k, fr["timestamp"])
        assert np.array_equal(rec["pose"][i], pg), i
        assert rec["regs"][i] == sg["registrations"] and rec["iters"][i] == sg["iterations"]
        assert rec["masked"][i] == sg["masked_pixels"]
        assert max(pose_error(po, rec["pose"][i])) <= 1e-4
    gp.finalize()
    v, c, f = gp.volume().extract_mesh(2)
    assert (nv, nf) == (len(v), len(f)) and nb == gp.volume().num_blocks()
    assert nf > 1000
