"""Cycles of one LM step on one thread (rf_diag_lm_step: LDLT solve, ExpMap + compose)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1905_02082_b200 import _lib as L  # noqa: E402

lib = L.load()
c = (C.c_double * 3)()
L.check(lib.rf_diag_lm_step(0, 2000, c))
print(f"solve {c[0]:.0f} cycles, expmap+compose {c[1]:.0f}, total {c[2]:.0f}")
