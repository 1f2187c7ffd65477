"""Prints the per-call cost of the tracking kernel's grid barrier / all-reduce."""
import ctypes as C
import sys

sys.path.insert(0, ".")
from paper_1905_02082_b200 import _lib as L  # noqa: E402

lib = L.load()
for reduce in (0, 1, 2, 3, 4):  # barrier, 30-value all-reduce, CTA-local part, 1-value all-reduce, bare exchange
    us = C.c_double()
    L.check(lib.rf_diag_grid_barrier(0, 2000, reduce, C.byref(us)))
    print(f"{L.LIB_PATH.split('/')[-1]} reduce={reduce}: {us.value:.3f} us per call")
cyc = (C.c_double * 3)()
L.check(lib.rf_diag_lm_step(0, 1000, cyc))
print(f"LM step on one thread: solve {cyc[0]:.0f} cycles, expmap+compose {cyc[1]:.0f}, total {cyc[2]:.0f}")
