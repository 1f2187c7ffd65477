"""Block order and snapshot bytes on the CUDA path.

The reference numbers blocks in allocation order: AllocateForFrame walks the
pixels in raster order and each pixel's segment cell by cell, and
AllocateBlock appends the first unseen key (tsdf_volume.cpp:64-77, 93-113).
blocks(), Save (tsdf_volume.cpp:375-403) and so the snapshot bytes follow
that order. The CUDA path assigns pool indices by each key's first visit
(hash_insert_ordered + assign_new), so:
  * the pool order equals the oracle's allocation order (lockstep);
  * Save files are byte-identical to the oracle's and across reruns
    (test_pipeline.cpp:119-156);
  * an allocation that exceeds max_blocks keeps exactly the reference's
    first-come bricks and hash occupancy, then raises ResourceLimitError;
  * a batch of frames stops at the overflowing frame (nothing of it is
    integrated, nothing after it runs), like the reference's exception.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1905_02082_b200 import api as G
from paper_1905_02082_b200 import scenes
from tests import helpers as H
from tests.test_gpu_parity import frame, gcfg, pair, pose_error, wavy_frame

pytestmark = pytest.mark.gpu


def assert_consistent(gv):
    """rf_diag_volume_check: table, pool and link records agree (the lock-free
    inserts, the ranked assignment and the concurrent link writers left no
    inconsistency)."""
    errs = gv.check()
    assert all(v == 0 for v in errs.values()), errs


def assert_same_pool(ov, gv, occupancy=True):
    oc, ovox = ov.export()
    gc, gvox = gv.export()
    assert oc.shape == gc.shape, f"{len(oc)} vs {len(gc)} blocks"
    assert (oc == gc).all(), "pool order differs"
    assert ovox.tobytes() == gvox.tobytes(), "voxels differ"
    if occupancy:
        assert (ov.hash_occupancy(gv.hash_capacity()) == gv.hash_occupancy()).all()
    assert_consistent(gv)


def lockstep(n=8, mover=True, vc=None):
    s = O.Scene(scenes.room_script(with_mover=mover, frames=n))
    vc = vc or O.vol_cfg()
    op = O.Pipeline(O.pipe_cfg(refine=False, volume=vc, reg=O.reg_cfg(threads=8)))
    gv = G.TsdfVolume(gcfg(vc))
    for i in range(len(s)):
        f = s.render(i)
        _, pose = op.process_frame(f["depth"], f["rgb"], s.k, f["timestamp"])
        fr = frame(s.k, f["depth"], f["rgb"])
        if i == 0:
            gv.allocate_for_frame(fr, pose)
            gv.integrate(fr, pose)
            continue
        mask = op.last_mask(s.k)
        gv.carve(fr, pose)
        gv.allocate_for_frame(fr, pose, mask)
        gv.integrate(fr, pose, mask)
    return op, gv


def test_lockstep_pool_order_and_save_bytes(tmp_path):
    op, gv = lockstep()
    ov = op.volume()
    assert_same_pool(ov, gv)
    ov.save(tmp_path / "oracle.bin")
    gv.save(str(tmp_path / "gpu.bin"))
    a, b = (tmp_path / "oracle.bin").read_bytes(), (tmp_path / "gpu.bin").read_bytes()
    assert len(a) == len(b) > 100000 and a == b


def test_save_load_cross_bytes(tmp_path):
    """GPU Save -> oracle Load -> oracle Save, and oracle Save -> GPU Load ->
    GPU Save reproduce the same bytes (Load re-allocates in file order)."""
    op, gv = lockstep(n=4)
    gv.save(str(tmp_path / "g.bin"))
    O.Volume.load(tmp_path / "g.bin").save(tmp_path / "g_o.bin")
    op.volume().save(tmp_path / "o.bin")
    G.TsdfVolume.load(str(tmp_path / "o.bin")).save(str(tmp_path / "o_g.bin"))
    ref = (tmp_path / "o.bin").read_bytes()
    for name in ("g.bin", "g_o.bin", "o_g.bin"):
        assert (tmp_path / name).read_bytes() == ref, name


def test_write_ply_bytes(tmp_path):
    """ExtractMesh + WritePly (mesh.cpp:149-225) of identical volumes: identical files."""
    op, gv = lockstep(n=6)
    op.volume().write_ply(tmp_path / "o.ply")
    gv.extract_mesh(ply_path=tmp_path / "g.ply")
    a, b = (tmp_path / "o.ply").read_bytes(), (tmp_path / "g.ply").read_bytes()
    assert len(a) > 10000 and a == b
    # an empty mesh has no colour properties (WritePly's `colored`, mesh.cpp:197)
    ev, eg = pair(O.vol_cfg())
    ev.write_ply(tmp_path / "oe.ply")
    eg.extract_mesh(ply_path=tmp_path / "ge.ply")
    assert (tmp_path / "oe.ply").read_bytes() == (tmp_path / "ge.ply").read_bytes()


def test_allocate_blocks_order_and_created():
    """AllocateBlock in argument order: created flags (duplicates and existing
    keys return false) and pool order equal the serial reference."""
    ov, gv = pair(O.vol_cfg(voxel_size=0.02, max_blocks=1000))
    rng = np.random.default_rng(3)
    first = rng.integers(-6, 6, (40, 3)).astype(np.int32)
    created_o = [ov.allocate_block(c) for c in first]
    created_g = gv.allocate_blocks(first)
    assert [int(x) for x in created_o] == [int(x) for x in created_g]
    more = np.concatenate([rng.integers(-8, 8, (60, 3)), first[:5]]).astype(np.int32)
    created_o = [ov.allocate_block(c) for c in more]
    created_g = gv.allocate_blocks(more)
    assert [int(x) for x in created_o] == [int(x) for x in created_g]
    assert_same_pool(ov, gv)


@pytest.mark.parametrize("budget", [7, 150, 300])
def test_overflow_keeps_reference_prefix(budget):
    """An AllocateForFrame that runs out of blocks throws after allocating the
    raster-order prefix (tsdf_volume.cpp:66-69); the table holds exactly those
    keys, and a later allocation continues from there."""
    k = O.small_intrinsics(64, 48, 50.0)
    ov, gv = pair(O.vol_cfg(voxel_size=0.01, max_blocks=budget))
    for i in range(3):
        d, rgb = wavy_frame(k, i)
        pose = H.small_pose((0.01 * i, 0.0, 0.0), (0, 1, 0), 0.05 * i)
        raised = []
        for vol, fr in ((ov, d), (gv, frame(k, d))):
            try:
                vol.allocate_for_frame(fr, k, pose) if vol is ov else vol.allocate_for_frame(fr, pose)
                raised.append(False)
            except (O.ResourceLimit, G.ResourceLimitError):
                raised.append(True)
        assert raised[0] == raised[1], i
        assert ov.num_blocks() == gv.num_blocks() <= budget
        assert_same_pool(ov, gv)
        if not raised[0]:
            ov.integrate(d, rgb, k, pose)
            gv.integrate(frame(k, d, rgb), pose)
            assert_same_pool(ov, gv)
    assert ov.num_blocks() == budget  # every budget above overflows by the third frame (385 blocks needed)


def pipeline_frames(n=8):
    s = O.Scene(scenes.room_script(with_mover=True, width=160, height=120, frames=n))
    return s, [s.render(i) for i in range(n)]


@pytest.mark.parametrize("batched", [False, True])
def test_pipeline_overflow_stops_at_the_frame(batched):
    """ResourceLimitError inside ProcessFrame: the failing frame's registration
    is in the trajectory, it is carved but not integrated, frame_count and
    stats stop there (pipeline.cpp:101-130) -- and in a batch nothing after it
    runs. Compared with the oracle pipeline on the same frames."""
    s, frames = pipeline_frames()
    vc = O.vol_cfg(voxel_size=0.02, max_blocks=200000)
    # the budget lands inside one frame's allocation: find it with the oracle
    op = O.Pipeline(O.pipe_cfg(refine=False, volume=vc, reg=O.reg_cfg(threads=8)))
    counts = []
    for f in frames:
        op.process_frame(f["depth"], f["rgb"], s.k, f["timestamp"])
        counts.append(op.volume().num_blocks())
    j = 3
    budget = (counts[j - 1] + counts[j]) // 2
    assert counts[j - 1] < budget < counts[j]
    vc = O.vol_cfg(voxel_size=0.02, max_blocks=budget)
    op = O.Pipeline(O.pipe_cfg(refine=False, volume=vc, reg=O.reg_cfg(threads=8)))
    gp = G.Pipeline(G.pipeline_config(refine=False, volume=gcfg(vc)))
    gfr = [frame(s.k, f["depth"], f["rgb"], f["timestamp"]) for f in frames]
    for i in range(j):
        op.process_frame(frames[i]["depth"], frames[i]["rgb"], s.k, frames[i]["timestamp"])
    with pytest.raises(O.ResourceLimit):
        op.process_frame(frames[j]["depth"], frames[j]["rgb"], s.k, frames[j]["timestamp"])
    if batched:
        with pytest.raises(G.ResourceLimitError):
            gp.process_frames(gfr)  # frames j+1.. must leave no trace
    else:
        for i in range(j):
            gp.process_frame(gfr[i])
        with pytest.raises(G.ResourceLimitError):
            gp.process_frame(gfr[j])
    ts_g, poses_g = gp.trajectory()
    assert len(ts_g) == j + 1  # the failing frame's registration is recorded (pipeline.cpp:101-102)
    assert len(op.trajectory) == j  # (the Python mirror records successful calls only)
    assert max(max(pose_error(po, pg)) for (_, po), pg in zip(op.trajectory, poses_g)) <= 1e-4
    ov = op.volume()
    assert ov.num_blocks() == gp.volume().num_blocks() == budget
    oc, _ = ov.export(False)
    gc, _ = gp.volume().export(False)
    assert (np.sort(oc.view("i4,i4,i4"), axis=0) == np.sort(gc.view("i4,i4,i4"), axis=0)).all()
    assert (ov.hash_occupancy(gp.volume().hash_capacity()) == gp.volume().hash_occupancy()).all()
    assert_consistent(gp.volume())
    # the pipeline keeps working after the exception (the next frame throws again: no room)
    with pytest.raises(G.ResourceLimitError):
        gp.process_frame(gfr[j + 1])


def test_pipeline_rerun_snapshot_bytes(tmp_path):
    """test_pipeline.cpp:119-156: reruns give identical trajectories, stats
    and snapshot bytes; single and batched submission too."""
    s, frames = pipeline_frames(12)
    cfg = G.pipeline_config(refine=True, window=3, volume=G.volume_config(voxel_size=0.02, max_blocks=200000))
    paths = []
    trajs = []
    for run in range(3):
        gp = G.Pipeline(cfg if run < 2 else G.pipeline_config(refine=False, volume=cfg.volume))
        gfr = [frame(s.k, f["depth"], f["rgb"], f["timestamp"]) for f in frames]
        if run == 2:
            gp.process_frames(gfr)
        else:
            for f in gfr:
                gp.process_frame(f)
        gp.finalize()
        trajs.append(gp.trajectory()[1])
        p = str(tmp_path / f"run{run}.bin")
        gp.volume().save(p)
        paths.append(p)
    assert np.array_equal(trajs[0], trajs[1])
    assert_consistent(gp.volume())
    assert open(paths[0], "rb").read() == open(paths[1], "rb").read()
    # the refine-off batched run differs in content, but is itself rerun-stable
    gp = G.Pipeline(G.pipeline_config(refine=False, volume=cfg.volume))
    gp.process_frames([frame(s.k, f["depth"], f["rgb"], f["timestamp"]) for f in frames])
    gp.volume().save(str(tmp_path / "again.bin"))
    assert open(paths[2], "rb").read() == (tmp_path / "again.bin").read_bytes()
