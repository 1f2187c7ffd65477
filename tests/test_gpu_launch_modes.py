"""The per-frame kernels launch with programmatic dependent launch
(griddepcontrol) by default; RF_PDL=0 launches them with plain stream
serialisation. Both must give bit-identical poses, stats and volumes (the
launch attribute only changes when a kernel may start, never what it reads).
Host frames (staged through the upload stream) and device frames must agree
too."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import hashlib, json, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_1905_02082_b200 import api as G, scenes, synth
scene = synth.parse(scenes.config_script("C2"))
k = scene.intrinsics
n = 40
d = torch.empty((n, k.height, k.width), dtype=torch.float32, device="cuda")
c = torch.empty((n, k.height, k.width, 3), dtype=torch.uint8, device="cuda")
lab = torch.empty((n, k.height, k.width), dtype=torch.uint8, device="cuda")
for i in range(n):
    synth.render(scene, i, d[i], c[i], lab[i])
torch.cuda.synchronize()
out = {}
for mode in ("device", "host"):
    p = G.Pipeline(G.pipeline_config(refine=False))
    if mode == "device":
        frames = [G.Frame(depth=d[i], rgb=c[i], intrinsics=k, timestamp=i / 30.0) for i in range(n)]
    else:
        frames = [G.Frame(depth=d[i].cpu().numpy(), rgb=c[i].cpu().numpy(), intrinsics=k, timestamp=i / 30.0)
                  for i in range(n)]
    stats, poses = p.process_frames(frames)
    coords, vox = p.volume().export()
    order = np.lexsort(coords.T[::-1])
    out[mode] = {
        "poses": hashlib.sha256(np.ascontiguousarray(poses).tobytes()).hexdigest(),
        "iterations": [int(s["iterations"]) for s in stats],
        "masked": [int(s["masked_pixels"]) for s in stats],
        "volume": hashlib.sha256(coords[order].tobytes() + vox[order].tobytes()).hexdigest(),
    }
print(json.dumps(out))
"""


def run(pdl):
    env = dict(os.environ, RF_PDL=pdl)
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_pdl_and_plain_launches_identical():
    a, b = run("1"), run("0")
    assert a == b
    assert a["device"] == a["host"]
    assert sum(a["device"]["masked"]) > 0 and min(a["device"]["iterations"][1:]) > 0
