"""Where the e2e (host frames, wall clock) vs value (device frames, events)
gap comes from: the same batch call timed four ways."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_02082_b200 import _lib as L, api, scenes, synth  # noqa: E402


def main(n=200, warm=10):
    scene = synth.parse(scenes.config_script("C2"))
    k = scene.intrinsics
    F = len(scene)
    d = torch.empty((F, k.height, k.width), dtype=torch.float32, device="cuda")
    c = torch.empty((F, k.height, k.width, 3), dtype=torch.uint8, device="cuda")
    lab = torch.empty((F, k.height, k.width), dtype=torch.uint8, device="cuda")
    for i in range(F):
        synth.render(scene, i, d[i], c[i], lab[i])
    torch.cuda.synchronize()
    dh, ch = d.cpu().pin_memory(), c.cpu().pin_memory()
    lib = L.load()

    def frames(dev, start, m):
        arr = (L.rf_frame * m)()
        for j in range(m):
            f = L.rf_frame()
            f.intrinsics = k
            s = (start + j) % F
            if dev:
                f.depth, f.rgb, f.memory = d[s].data_ptr(), c[s].data_ptr(), L.RF_MEMORY_DEVICE
            else:
                f.depth, f.rgb, f.memory = dh[s].data_ptr(), ch[s].data_ptr(), L.RF_MEMORY_HOST
            f.timestamp = (start + j) / 30.0
            arr[j] = f
        return arr

    for dev in (True, False):
        p = api.Pipeline(api.pipeline_config(refine=False))
        L.check(lib.rf_pipeline_process_frames(p.h, frames(dev, 0, warm), C.c_uint64(warm), None, None))
        sptr = C.c_void_p()
        L.check(lib.rf_pipeline_stream(p.h, C.byref(sptr)))
        stream = torch.cuda.ExternalStream(sptr.value)
        arr = frames(dev, warm, n)
        st = (L.rf_frame_stats * n)()
        poses = (C.c_double * (12 * n))()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(stream)
        L.check(lib.rf_pipeline_process_frames(p.h, arr, C.c_uint64(n), st, poses))
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        ev = e0.elapsed_time(e1) / 1e3
        host_ms = sum(st[i].runtime_ms for i in range(n))
        print(f"{'device' if dev else 'host  '} frames: wall {n / wall:.1f} fps, events {n / ev:.1f} fps, "
              f"host finish {host_ms / n * 1e3:.1f} us/frame")


if __name__ == "__main__":
    main()
