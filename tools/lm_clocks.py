"""Reads trace record 251 of an RF_TRACE_FILE written by the RF_LM_CLOCKS
diagnostics build: LM-thread cycle counters of CTA 0 per frame (accept-path
judge, solve, ExpMap + compose, whole LM section; reject-path pre-solve)."""
import sys

import numpy as np

raw = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 256, 8)[3:]  # frames past the first three
r = raw[:, 251, :].astype(np.float64).sum(0)
print("accept-path solves %.0f: judge %.0f, lm_solve %.0f, expmap+compose %.0f cycles each" %
      (r[0], r[1] / max(r[0], 1), r[2] / max(r[0], 1), r[3] / max(r[0], 1)))
print("LM sections %.0f: %.0f cycles each (all paths)" % (r[7], r[4] / max(r[7], 1)))
print("pre-solves %.0f: %.0f cycles each (lm_solve + expmap + compose)" % (r[5], r[6] / max(r[5], 1)))
q = raw[:, 250, :].astype(np.float64).sum(0)
n = max(r[7], 1)
print("per LM iteration on CTA 0's LM thread (cycles): LM-section end -> reconverged %.0f, -> barrier release %.0f, "
      "-> go read %.0f, -> (back-edge) pass entry %.0f, -> prologue done %.0f, own pixels %.0f, all-reduce %.0f, "
      "all-reduce end -> LM section %.0f" % (q[7] / n, q[0] / n, q[6] / n, q[5] / n, q[1] / n, q[2] / n, q[3] / n, q[4] / n))
t = raw[:, 249, :2].astype(np.float64).sum(0)
print("thread 0 (warp 0), same span: barrier release -> pass entry %.0f cycles (%d samples)" % (t[0] / max(t[1], 1), t[1]))
