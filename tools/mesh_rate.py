"""ExtractMesh timing on a C4-sized model (1280x720 frames fused into the
pipeline's volume): repeated calls, wall clock of rf_volume_extract_mesh
(device extraction, no host copy) and of the full host copy."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import oracle as O  # noqa: E402
from paper_1905_02082_b200 import _lib as L  # noqa: E402
from paper_1905_02082_b200 import api as G  # noqa: E402
from paper_1905_02082_b200 import scenes  # noqa: E402


def main(frames=int(sys.argv[1]) if len(sys.argv) > 1 else 40):
    s = O.Scene(scenes.config_script("C4"))
    k = s.k
    gk = G.intrinsics(k.fx, k.fy, k.cx, k.cy, k.width, k.height, k.depth_scale)
    p = G.Pipeline(G.pipeline_config(refine=False))
    fr = []
    for i in range(frames):
        f = s.render(i)
        fr.append(G.Frame(f["depth"], f["rgb"], gk, f["timestamp"]))
    p.process_frames(fr)
    vol = p.volume()
    lib = L.load()
    for rep in range(4):
        m = C.c_void_p()
        t0 = time.perf_counter()
        L.check(lib.rf_volume_extract_mesh(vol.h, 2, C.byref(m)))
        t1 = time.perf_counter()
        nv, nf = C.c_uint64(), C.c_uint64()
        L.check(lib.rf_mesh_counts(m, C.byref(nv), C.byref(nf)))
        lib.rf_mesh_destroy(m)
        t2 = time.perf_counter()
        v, c, f = vol.extract_mesh(2)
        t3 = time.perf_counter()
        print(f"rep {rep}: extract {1e3 * (t1 - t0):.2f} ms (device), with host copy {1e3 * (t3 - t2):.2f} ms; "
              f"{nv.value} vertices, {nf.value} faces, {vol.num_blocks()} bricks", flush=True)


if __name__ == "__main__":
    main()
