#!/usr/bin/env python
"""bench.py — ReFusion per-frame hot path on B200.

metric : frames/s of Pipeline::ProcessFrame (track + mask + carve + allocate +
         integrate, pipeline.cpp:57-131) at 640x480 with 1 cm voxels.
workload: BASELINE.json configs[1] ("C2", the default): the acceptance room
         with two moving boxes, 200 frames at 30 Hz, replayed forwards then
         backwards (a continuous ping-pong sequence) so any step count keeps
         tracking. --config C1|C3|C4 runs the other BASELINE.json workloads
         (C3: large room at 0.5 cm with a 2^22 hash; C4: 1280x720 with the
         mesh export timed after the run).
         Frames are synthetic, rendered on the GPU before timing.
One step = one ProcessFrame on one frame.

Arms:
  default          : our CUDA path through the C ABI. `value` = frames/s with
                     the frames already resident in HBM (CUDA events on the
                     pipeline's stream, max over ranks); `e2e` = the same through
                     rf_pipeline_process_frame with pinned HOST buffers (H2D of
                     depth+RGB and the D2H of stats+pose inside the timed loop).
  --impl reference : the reference itself on the host CPU: /root/reference's
                     unmodified C++ sources built into oracle/_ref against the
                     Eigen / doctest / libpng stand-ins of oracle/ref_shim
                     (`make -C oracle ref`; the library travels to the GPU box),
                     all host threads. Falls back to the oracle restatement
                     (bit-identical to it, tests/test_reference_build.py) when
                     oracle/_ref was not built.
The default line carries a `parity` block: the GPU arm's per-frame poses and
counts (registrations, LM iterations, masked pixels) against the cpu_baseline
leg's over the frames both processed (same bytes, same order).
Multi-GPU (torchrun): independent sequences per GPU (replicas, no collective).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frames/sec (track+integrate, 640x480, 1cm voxels) per B200 + HBM roofline frac"
UNIT = "frames/s"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4"],
                    help="BASELINE.json workload (C2 is the headline)")
    return ap.parse_args()


def seq_index(step, n):
    """Ping-pong through the n rendered frames: 0..n-1, n-2..1, 0.."""
    period = 2 * n - 2
    i = step % period
    return i if i < n else period - i


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """SM clock and throttle reasons sampled through NVML every 0.5 ms while
    the timed region runs (one sample is always taken on entry and on exit,
    so even a 20 ms region has samples)."""

    NAMES = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.h = None
        self.stop = threading.Event()

    def _sample(self):
        import pynvml as N
        try:
            sm = N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)
            mx = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            rs = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            self.rows.append((sm, mx, rs))
        except Exception:
            pass

    def _run(self):
        while not self.stop.wait(0.0005):
            self._sample()

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.index]) if vis and vis.split(",")[self.index].isdigit() else self.index
            self.h = N.nvmlDeviceGetHandleByIndex(idx)
            self._sample()
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception:
            self.h = None
        return self

    def __exit__(self, *exc):
        if self.h is not None:
            self.stop.set()
            self.thread.join(timeout=2)
            self._sample()

    def summary(self):
        sm = sorted(r[0] for r in self.rows)
        reasons = sorted({n for r in self.rows for n, bit in self.NAMES.items() if r[2] & bit})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(r[1] for r in self.rows) if sm else None,
                "reasons": reasons, "samples": len(sm), "source": "nvml, 0.5 ms polling inside the timed region"}


# ----------------------------------------------------------------------------- workload
DATA = ("synthetic: the {cfg} scene script rendered by RenderFrame (synth.cpp:136-203, oracle restatement, "
        "mt19937 depth noise 0.001*z^2, seed {seed}); identical bytes in both arms")


def render_sequence(script: str, count: int | None = None):
    """The workload generator, outside every timed region: the first `count`
    frames (default all) of a scene script through RenderFrame on the host
    cores (frames are independent: each seeds its own mt19937, synth.cpp:185).
    Returns (intrinsics, depth [F,H,W] f32, rgb [F,H,W,3] u8, timestamps)."""
    from concurrent.futures import ThreadPoolExecutor

    import numpy as np

    from oracle import oracle as O

    scene = O.Scene(script)
    k = scene.k
    F = len(scene) if count is None else min(count, len(scene))
    depth = np.empty((F, k.height, k.width), dtype=np.float32)
    rgb = np.empty((F, k.height, k.width, 3), dtype=np.uint8)
    ts = np.empty(F)

    def one(i):
        f = scene.render(i)
        depth[i], rgb[i], ts[i] = f["depth"], f["rgb"], f["timestamp"]

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:  # ctypes releases the GIL
        list(ex.map(one, range(F)))
    return k, depth, rgb, ts


WORKLOADS = {
    "C1": "C1: synthetic static room (acceptance RoomScript), {W}x{H} RGB-D, 1 cm voxels",
    "C2": "C2: synthetic room with 2 moving boxes, {W}x{H} RGB-D, 1 cm voxels",
    "C3": "C3: synthetic large scene (12 x 4 x 12 m room + props), {W}x{H} RGB-D, 0.5 cm voxels, 2^22-entry hash",
    "C4": "C4: synthetic room with 2 moving boxes, {W}x{H} RGB-D (K 1050/639.5/359.5), 1 cm voxels, 3 levels, "
          "mesh export after the run",
}
L2_NOTE = {
    "C3": "bricks (~1e5-1e6, 0.5-4 GB) exceed the 126 MB L2: fuse/alloc stream from HBM",
    "C4": "bricks L2-resident; frames (6.4 MB each) stream from HBM",
}


def workload_config(name, W, H, F):
    """The `config` object of both arms (identical by construction)."""
    from paper_1905_02082_b200 import scenes

    return {"workload": WORKLOADS[name].format(W=W, H=H) + f", {F}-frame sequence (ping-pong past its end), "
                                                            "refine_depth off",
            "resolution": [W, H], "voxel_size": scenes.BENCH_CONFIGS[name]["voxel"], "frames_in_sequence": F,
            "l2": L2_NOTE.get(name, "bricks (~20k, 80 MB) L2-resident by design; the frames (430 MB) exceed L2")}


def volume_params(name):
    """VolumeConfig of a workload: (voxel_size, max_blocks, hash_capacity)."""
    from paper_1905_02082_b200 import scenes

    c = scenes.BENCH_CONFIGS[name]
    return c["voxel"], c.get("max_blocks", 1000000), c.get("hash_capacity", 0)


def parity_block(gpu, cpu):
    """Per-frame comparison of the GPU arm's steps with the cpu_baseline leg
    over the frames both processed (step s = frame seq_index(s) of the same
    sequence from the same bootstrap): pose difference (translation, m;
    rotation angle, rad) and count mismatches."""
    import numpy as np

    n = min(len(gpu), len(cpu))
    worst_t = worst_r = 0.0
    mism = {"registrations": 0, "iterations": 0, "masked_pixels": 0, "tracking_lost": 0}
    max_masked = 0
    for s in range(1, n):  # step 0 is the identity bootstrap in both
        (gs, gp), (cs, cp) = gpu[s], cpu[s]
        worst_t = max(worst_t, float(np.abs(gp[9:] - cp[9:]).max()))
        Rd = gp[:9].reshape(3, 3) @ cp[:9].reshape(3, 3).T
        axis = np.array([Rd[2, 1] - Rd[1, 2], Rd[0, 2] - Rd[2, 0], Rd[1, 0] - Rd[0, 1]])  # 2 sin(theta) * axis
        worst_r = max(worst_r, float(np.arctan2(0.5 * np.linalg.norm(axis), 0.5 * (np.trace(Rd) - 1.0))))
        for key in mism:
            if int(gs[key]) != int(cs[key]):
                mism[key] += 1
        max_masked = max(max_masked, abs(int(gs["masked_pixels"]) - int(cs["masked_pixels"])))
    return {"frames_compared": max(0, n - 1), "worst_pose_m": worst_t, "worst_pose_rad": worst_r,
            "mismatched_frames": mism, "max_masked_pixel_diff": max_masked,
            "bar": "pose <= 1e-4 m / 1e-4 rad (north_star)"}


# ----------------------------------------------------------------------------- ours
def run_ours(args):
    import numpy as np
    import torch

    from oracle import oracle as O
    from paper_1905_02082_b200 import _lib as L
    from paper_1905_02082_b200 import api, replicas, scenes

    name = args.config
    R = replicas.env()
    rank, world, local = R.rank, R.world, R.local
    torch.cuda.set_device(local)
    R = replicas.init("nccl")
    lib = L.load()
    cfgd = scenes.BENCH_CONFIGS[name]
    seed = replicas.sequence_seed(cfgd["seed"], R)  # independent sequence per replica
    script = scenes.config_script(name, seed=seed)
    F = cfgd["frames"]
    ok, depth_np, rgb_np, _ = render_sequence(script, min(F, args.warmup + args.steps))  # the frames the run uses
    k = api.intrinsics(ok.fx, ok.fy, ok.cx, ok.cy, ok.width, ok.height, ok.depth_scale)
    Fr, H, W = depth_np.shape
    depth_h = torch.from_numpy(depth_np).pin_memory()
    rgb_h = torch.from_numpy(rgb_np).pin_memory()
    depth = depth_h.to("cuda")
    rgb = rgb_h.to("cuda")
    torch.cuda.synchronize()

    voxel, max_blocks, cap = volume_params(name)
    cfg = api.pipeline_config(refine=False, volume=api.volume_config(voxel_size=voxel, max_blocks=max_blocks,
                                                                     hash_capacity=cap))

    def make_frames(dev_resident):
        frames = []
        for i in range(Fr):
            f = L.rf_frame()
            f.intrinsics = k
            if dev_resident:
                f.depth, f.rgb, f.memory = depth[i].data_ptr(), rgb[i].data_ptr(), L.RF_MEMORY_DEVICE
            else:
                f.depth, f.rgb, f.memory = depth_h[i].data_ptr(), rgb_h[i].data_ptr(), L.RF_MEMORY_HOST
            frames.append(f)
        return frames

    def run_steps(p, frames, start, n, stats, pose):
        for st in range(start, start + n):
            f = frames[seq_index(st, F)]
            f.timestamp = st / 30.0
            L.check(lib.rf_pipeline_process_frame(p.h, C.byref(f), C.byref(stats), pose))

    def barrier():
        replicas.barrier(R)
        torch.cuda.synchronize()

    stats = L.rf_frame_stats()
    pose = (C.c_double * 12)()

    def batch(frames, start, n):  # the timed steps as one rf_pipeline_process_frames call's input
        arr = (L.rf_frame * n)()
        for j in range(n):
            arr[j] = frames[seq_index(start + j, F)]
            arr[j].timestamp = (start + j) / 30.0
        return arr

    # ---- value: frames resident in HBM, device time on the pipeline's stream;
    # RunSequence through rf_pipeline_process_frames (frames enqueued back to back)
    pv = api.Pipeline(cfg, device=local)
    dev_frames = make_frames(True)
    # warm-up through the same batched call as the timed steps
    wst = (L.rf_frame_stats * max(1, args.warmup))()
    wposes = (C.c_double * (12 * max(1, args.warmup)))()
    L.check(lib.rf_pipeline_process_frames(pv.h, batch(dev_frames, 0, args.warmup), C.c_uint64(args.warmup),
                                           wst, wposes))
    sptr = C.c_void_p()
    L.check(lib.rf_pipeline_stream(pv.h, C.byref(sptr)))
    stream = torch.cuda.ExternalStream(sptr.value)
    launches0 = C.c_uint64()
    L.check(lib.rf_pipeline_stage_times(pv.h, None, None, C.byref(launches0)))
    timed = batch(dev_frames, args.warmup, args.steps)
    st_arr = (L.rf_frame_stats * args.steps)()
    poses = (C.c_double * (12 * args.steps))()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        L.check(lib.rf_pipeline_process_frames(pv.h, timed, C.c_uint64(args.steps), st_arr, poses))
        ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches1 = C.c_uint64()
    L.check(lib.rf_pipeline_stage_times(pv.h, None, None, C.byref(launches1)))
    gpu_launches = launches1.value - launches0.value
    agg = {"lost": sum(x.tracking_lost for x in st_arr), "iters": sum(x.iterations for x in st_arr),
           "regs": sum(x.registrations for x in st_arr), "masked": sum(x.masked_pixels for x in st_arr)}
    num_blocks = pv.volume().num_blocks()
    gpu_steps = []  # (stats, pose) per step of the value run, warm-up included (parity block)
    for j in range(args.warmup + args.steps):
        sa, pa, jj = (wst, wposes, j) if j < args.warmup else (st_arr, poses, j - args.warmup)
        gpu_steps.append(({"registrations": sa[jj].registrations, "iterations": sa[jj].iterations,
                           "masked_pixels": sa[jj].masked_pixels, "tracking_lost": sa[jj].tracking_lost},
                          np.array(pa[12 * jj:12 * jj + 12])))
    mesh = None
    if name == "C4":  # ExtractMesh of the run's model (mesh.cpp:149-181), timed apart from the frames
        vol = pv.volume()
        for _ in range(2):
            vol.extract_mesh()  # module loading, CUB temp sizing, the scratch buffer
        times = []
        for _ in range(5):
            t0 = time.perf_counter()
            v_, c_, f_ = vol.extract_mesh()
            times.append(1e3 * (time.perf_counter() - t0))
        mesh = {"ms_median": round(sorted(times)[2], 3), "ms_runs": [round(t, 3) for t in times],
                "vertices": len(v_), "faces": len(f_), "bricks": num_blocks,
                "includes": "device extraction + D2H of vertices, colours and faces (host wall clock)"}

    # ---- per-stage device times and work counters (roofline): the same steps
    # frame by frame with CUDA events between the kernels
    pp = api.Pipeline(cfg, device=local)
    run_steps(pp, dev_frames, 0, args.warmup, stats, pose)
    L.check(lib.rf_pipeline_set_profiling(pp.h, 1))
    run_steps(pp, dev_frames, args.warmup, args.steps, stats, pose)
    stage = (C.c_double * 4)()
    nprof = C.c_uint64()
    L.check(lib.rf_pipeline_stage_times(pp.h, stage, C.byref(nprof), None))
    sums = L.rf_frame_counters()
    L.check(lib.rf_pipeline_profile_counters(pp.h, C.byref(sums)))
    agg.update(pixel_passes=sums.pixel_passes, visible=sums.visible_bricks, dda=sums.dda_visits,
               new=sums.new_blocks, ff_rounds=sums.floodfill_rounds, passes=sums.passes)
    del pp

    # ---- e2e: pinned host frames through the same public call, wall clock
    # (each step's H2D copy and its result read-back inside the timed region)
    pe = api.Pipeline(cfg, device=local)
    host_frames = make_frames(False)
    L.check(lib.rf_pipeline_process_frames(pe.h, batch(host_frames, 0, args.warmup), C.c_uint64(args.warmup),
                                           None, None))
    timed_h = batch(host_frames, args.warmup, args.steps)
    barrier()
    t0 = time.perf_counter()
    L.check(lib.rf_pipeline_process_frames(pe.h, timed_h, C.c_uint64(args.steps), st_arr, poses))
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    del pe

    # ---- max over ranks
    sec, e2e_sec = replicas.max_over_ranks(R, [ms / 1000.0, e2e_s])
    value = replicas.job_rate(R, args.steps, sec)
    e2e = replicas.job_rate(R, args.steps, e2e_sec)

    if rank != 0:
        replicas.finish(R)
        return

    # ---- rooflines (SURVEY §8d bytes model): every kernel, the dominant one first
    n = args.steps
    P0 = W * H
    stage_ms = [stage[i] / max(1, nprof.value) for i in range(4)]
    bytes_per_frame = {
        # B_track = sum_passes 9*P_l + 4096*U (U ~ the frame's visible bricks)
        "track": 9.0 * agg["pixel_passes"] / n + 4096.0 * agg["visible"] / n,
        # B_alloc = 5*P0 + 16*R_visits + 4096*N_new
        "allocate": 5.0 * P0 + 16.0 * agg["dda"] / n + 4096.0 * agg["new"] / n,
        # cull reads 16 B of coordinates per allocated brick
        "cull": 16.0 * num_blocks,
        # B_carve+int = 2*4096*|visible| + 7*P0 (depth + colour gathers)
        "fuse": 2.0 * 4096.0 * agg["visible"] / n + 7.0 * P0,
    }
    names = ["track", "allocate", "cull", "fuse"]
    dom = max(range(4), key=lambda i: stage_ms[i])
    peak, peak_kind = measured_peaks()
    achieved = {nm: bytes_per_frame[nm] / (stage_ms[i] / 1e3) / 1e9 for i, nm in enumerate(names)}
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(names[dom])
    except Exception:
        pass
    # k_track is bound by its chain of dependent passes, not by bytes: the
    # latency model puts the measured grid all-reduce floor and the LM step of
    # every pass against the kernel's time (the rest is the pixel phases).
    us_red, cyc = C.c_double(), (C.c_double * 3)()
    L.check(lib.rf_diag_grid_barrier(local, 500, 1, C.byref(us_red)))
    L.check(lib.rf_diag_lm_step(local, 200, cyc))
    sm_mhz = clocks.summary().get("sm_mhz") or 1965.0
    passes = agg["passes"] / max(1, nprof.value)
    fixed_us = passes * (us_red.value + cyc[2] / sm_mhz)

    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": n,
        "warmup": args.warmup, "ms_per_step": round(sec * 1e3 / n, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": DATA.format(cfg=name, seed=seed),
        "config": workload_config(name, W, H, F),
        "parallelism": f"replicas x{world} (independent sequences, no collective)",
        "api": "rf_pipeline_process_frames (RunSequence: up to 64 frames enqueued back to back)",
        "e2e": {"value": round(e2e, 2), "unit": UNIT, "h2d_bytes_per_step": P0 * 4 + P0 * 3,
                "d2h_bytes_per_step": 192 + 32},
        "gpu_launches": int(gpu_launches),
        "roofline": {"bound": "hbm", "kernel": names[dom], "achieved": round(achieved[names[dom]], 2), "peak": peak,
                     "peak_source": peak_kind, "unit": "GB/s", "frac": round(achieved[names[dom]] / peak, 5),
                     "traffic": traffic, "bytes_per_launch": round(bytes_per_frame[names[dom]]),
                     "launch_ms": round(stage_ms[dom], 5)},
        "roofline_by_kernel": {nm: {"launch_ms": round(stage_ms[i], 5), "bytes_per_launch": round(bytes_per_frame[nm]),
                                    "achieved_gbs": round(achieved[nm], 1), "frac": round(achieved[nm] / peak, 4)}
                               for i, nm in enumerate(names)},
        "latency_model": {"kernel": "track", "passes_per_frame": round(passes, 2),
                          "allreduce_us": round(us_red.value, 3), "lm_step_us": round(cyc[2] / sm_mhz, 3),
                          "fixed_us_per_frame": round(fixed_us, 1),
                          "frac_of_track": round(fixed_us / (stage_ms[0] * 1e3), 3),
                          "note": "passes x (grid all-reduce floor + one-thread LM step), measured in-process; the "
                                  "remainder of k_track is the pixel phases, mask and pyramid"},
        "stages_ms_per_frame": {nm: round(stage_ms[i], 5) for i, nm in enumerate(names)},
        "workload_stats": {"lm_iterations_per_frame": agg["iters"] / n, "registrations_per_frame": agg["regs"] / n,
                           "masked_pixels_per_frame": agg["masked"] / n, "lost_frames": agg["lost"],
                           "visible_bricks_per_frame": agg["visible"] / n, "bricks": num_blocks,
                           "pixel_passes_per_frame": agg["pixel_passes"] / n,
                           "floodfill_rounds_per_frame": agg["ff_rounds"] / n},
        "clocks": clocks.summary(),
    }
    if mesh:
        line["mesh_export"] = mesh
    if world == 1 and not args.no_cpu_baseline:
        scene = O.Scene(script)
        cache = {}

        def frame(st):  # the bench's bytes, rendered on demand past the GPU run's frames
            j = seq_index(st, F)
            if j < Fr:
                return depth_np[j], rgb_np[j]
            if j not in cache:
                r = scene.render(j)
                cache[j] = (r["depth"], r["rgb"])
            return cache[j]

        line["cpu_baseline"], cpu_steps = cpu_baseline(frame, ok, args.cpu_sample_seconds, name)
        line["parity"] = parity_block(gpu_steps, cpu_steps)
    print(json.dumps(line), flush=True)
    replicas.finish(R)


def cpu_impl():
    """(module, kind): the reference build when present, else the oracle port."""
    from oracle import oracle as O
    from oracle import reference as Rf

    if Rf.available():
        return Rf, "reference"
    return O, "port"


def oracle_rate(frame, k, budget_s, threads, vol):
    """Oracle pipeline over a frame sample: bootstrap on frame 0 (untimed, as
    the reference's fps excludes frame 0), then time frames until budget_s.
    Returns the rate and every step's (stats, pose) for the parity block."""
    from oracle import oracle as O

    impl, _ = cpu_impl()
    p = impl.Pipeline(O.pipe_cfg(refine=False, threads=threads, reg=O.reg_cfg(threads=threads),
                                 volume=O.vol_cfg(voxel_size=vol[0], max_blocks=vol[1])))
    d, c = frame(0)
    st, pose = p.process_frame(d, c, k, 0.0)
    steps = [(st, pose)]
    spent, n = 0.0, 0
    while spent < budget_s or n < 2:
        i = n + 1
        d, c = frame(i)
        t0 = time.perf_counter()
        st, pose = p.process_frame(d, c, k, i / 30.0)
        spent += time.perf_counter() - t0
        steps.append((st, pose))
        n += 1
    return n / spent, n, spent, steps


def cpu_baseline(frame, k, budget_s, name):
    threads = os.cpu_count() or 1
    rate, n, spent, steps = oracle_rate(frame, k, budget_s, threads, volume_params(name))
    _, kind = cpu_impl()
    what = "the reference's Pipeline::ProcessFrame (oracle/_ref build)" if kind == "reference" else \
        "the oracle restatement of ProcessFrame"
    return ({"value": round(rate, 4), "unit": UNIT, "cores": threads, "kind": kind,
             "sample": f"{what} on steps 1..{n} of the same {name} sequence and the same frame bytes as the GPU arm "
                       f"({spent:.1f} s, {threads} threads for integrate/carve and registration)"},
            steps)


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    from paper_1905_02082_b200 import replicas

    R = replicas.env()
    rank, world = R.rank, R.world
    if rank != 0:  # rank 0 alone times the host CPU path; the others exit 0
        return
    from oracle import oracle as O
    from paper_1905_02082_b200 import scenes

    name = args.config
    seed = scenes.BENCH_CONFIGS[name]["seed"]
    F = scenes.BENCH_CONFIGS[name]["frames"]
    k, depth_np, rgb_np, _ = render_sequence(scenes.config_script(name, seed=seed),
                                             min(F, args.warmup + args.steps))  # the GPU arm's bytes
    Fr, H, W = depth_np.shape

    def frame(i):
        j = seq_index(i, F)
        return {"depth": depth_np[j], "rgb": rgb_np[j]}

    threads = os.cpu_count() or 1
    vox, mb, _ = volume_params(name)
    impl, kind = cpu_impl()
    p = impl.Pipeline(O.pipe_cfg(refine=False, threads=threads, reg=O.reg_cfg(threads=threads),
                                 volume=O.vol_cfg(voxel_size=vox, max_blocks=mb)))
    for i in range(args.warmup):
        f = frame(i)
        p.process_frame(f["depth"], f["rgb"], k, i / 30.0)
    t0 = time.perf_counter()
    for i in range(args.warmup, args.warmup + args.steps):
        f = frame(i)
        p.process_frame(f["depth"], f["rgb"], k, i / 30.0)
    sec = time.perf_counter() - t0
    value = args.steps / sec
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(sec * 1e3 / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "impl": "reference",
        "data": DATA.format(cfg=name, seed=seed),
        "config": workload_config(name, W, H, F),
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{'reference (oracle/_ref build)' if kind == 'reference' else 'oracle'} "
                                   f"ProcessFrame, steps {args.warmup}..{args.warmup + args.steps - 1} of the "
                                   f"{name} sequence, {threads} threads"},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
