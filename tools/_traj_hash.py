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
