"""Fingerprint of the CUDA pipeline's trajectory on the first 40 C2 frames
(SHA-1 of the pose bytes): two library builds that print the same digest
track bit-identically (RF_LIB_PATH selects a variant). Used to check that a
kernel change which should not alter arithmetic (e.g. the default-off
extensions, a reordered but equivalent computation) does not."""
import hashlib, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from oracle import oracle as O
from paper_1905_02082_b200 import api as G, scenes
from tests.test_gpu_parity import frame
s = O.Scene(scenes.config_script("C2"))
gp = G.Pipeline(G.pipeline_config(refine=False))
for i in range(40):
    f = s.render(i)
    gp.process_frame(frame(s.k, f["depth"], f["rgb"], f["timestamp"]))
ts, poses = gp.trajectory()
print("traj", hashlib.sha1(np.ascontiguousarray(poses).tobytes()).hexdigest())
