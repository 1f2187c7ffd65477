"""Frames/s of the pipeline on BASELINE.json's other configs (not bench lines;
bench.py measures C2): C1 static room, C3 0.5 cm voxels with the 2^22 hash and
4M bricks, C4 1280x720 (K scaled) + final ExtractMesh. Frames rendered on the
GPU, resident in HBM; RunSequence through rf_pipeline_process_frames, timed
with CUDA events on the pipeline's stream; refine off (acceptance config)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_02082_b200 import _lib as L, api, scenes, synth  # noqa: E402


def rate(name, script, vcfg=None, frames=200, warm=10, mesh=False):
    scene = synth.parse(script)
    k = scene.intrinsics
    F = len(scene)
    d = torch.empty((F, k.height, k.width), dtype=torch.float32, device="cuda")
    c = torch.empty((F, k.height, k.width, 3), dtype=torch.uint8, device="cuda")
    lab = torch.empty((F, k.height, k.width), dtype=torch.uint8, device="cuda")
    for i in range(F):
        synth.render(scene, i, d[i], c[i], lab[i])
    torch.cuda.synchronize()
    p = api.Pipeline(api.pipeline_config(refine=False, volume=vcfg))
    lib = L.load()
    arr = (L.rf_frame * frames)()
    for j in range(frames):
        f = L.rf_frame()
        f.intrinsics = k
        f.depth, f.rgb, f.memory = d[j % F].data_ptr(), c[j % F].data_ptr(), L.RF_MEMORY_DEVICE
        f.timestamp = j / 30.0
        arr[j] = f
    L.check(lib.rf_pipeline_process_frames(p.h, arr, C.c_uint64(warm), None, None))
    sptr = C.c_void_p()
    L.check(lib.rf_pipeline_stream(p.h, C.byref(sptr)))
    stream = torch.cuda.ExternalStream(sptr.value)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    L.check(lib.rf_pipeline_process_frames(p.h, C.byref(arr, warm * C.sizeof(L.rf_frame)), C.c_uint64(frames - warm),
                                           None, None))
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (frames - warm)
    line = f"{name}: {1000.0 / ms:.1f} frames/s ({ms:.3f} ms/frame, {k.width}x{k.height}, " \
           f"{p.volume().num_blocks()} bricks, {p.tracking_losses()} losses)"
    if mesh:
        p.volume().extract_mesh(2)  # first call loads the mesh kernels' modules (lazy loading)
        torch.cuda.synchronize()
        e0.record(stream)
        v, _, fc = p.volume().extract_mesh(2)
        e1.record(stream)
        torch.cuda.synchronize()
        line += f"; ExtractMesh {len(v)} vertices / {len(fc)} faces in {e0.elapsed_time(e1):.1f} ms (incl. D2H)"
    print(line, flush=True)


def main():
    rate("C1 static room (RoomScript path, 50 frames)", scenes.config_script("C1"), frames=50)
    rate("C2 room + 2 boxes", scenes.config_script("C2"))
    rate("C3 0.5 cm, 2^22 hash", scenes.bench_script(dynamic=True, frames=200, seed=43),
         vcfg=api.volume_config(voxel_size=0.005, max_blocks=4_000_000, hash_capacity=1 << 22))
    rate("C4 1280x720", scenes.bench_script(dynamic=True, width=1280, height=720, frames=200, seed=44), mesh=True)


if __name__ == "__main__":
    main()
