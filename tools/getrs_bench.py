"""Time the stage-two getrs (chained, nrhs <= 8) at n2 = 4000 through the debug hook."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_07572_b200 import _lib  # noqa: E402

L = _lib.lib()
P = ctypes.POINTER(ctypes.c_double)
L.slablu_gpu_debug_getrs.restype = ctypes.c_int
L.slablu_gpu_debug_getrs.argtypes = [ctypes.c_int64, ctypes.c_int64, P, P, P, ctypes.c_int, ctypes.c_int, P]
rng = np.random.default_rng(0)
for n in [int(a) for a in (sys.argv[1:] or ["1000", "4000"])]:
    A = np.asfortranarray(rng.standard_normal((n, n)))
    for nrhs in (1, 8, 16, 64):
        B = np.asfortranarray(rng.standard_normal((n, nrhs)))
        X = np.zeros((n, nrhs), order="F")
        t = np.zeros(1)
        assert L.slablu_gpu_debug_getrs(n, nrhs, A.ctypes.data_as(P), B.ctypes.data_as(P), X.ctypes.data_as(P), 20, 0,
                                        t.ctypes.data_as(P)) == 0
        err = np.linalg.norm(A @ X - B) / (np.linalg.norm(A) * np.linalg.norm(X))
        gbs = 8.0 * n * n / t[0] / 1e9
        print(f"getrs n={n} nrhs={nrhs}: {t[0]*1e6:.1f} us ({gbs:.0f} GB/s of LU) backward err {err:.2e}", flush=True)
