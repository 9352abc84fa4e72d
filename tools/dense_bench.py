"""Stage-two building blocks at block size n: GEMM, getrf, inverse (device time)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_07572_b200 import _lib  # noqa: E402

L = _lib.lib()
L.slablu_gpu_debug_dense_bench.restype = ctypes.c_int
L.slablu_gpu_debug_dense_bench.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
for n in [int(a) for a in sys.argv[1:]] or [1000, 4000]:
    for rep in range(2):
        out = (ctypes.c_double * 3)()
        assert L.slablu_gpu_debug_dense_bench(n, 0, out) == 0
    g, f, i = out
    print(f"n={n}: gemm {g*1e3:.2f} ms ({2*n**3/g/1e12:.2f} TF/s), getrf {f*1e3:.2f} ms ({2/3*n**3/f/1e12:.2f} TF/s), "
          f"inverse(getrs I) {i*1e3:.2f} ms ({2*n**3/i/1e12:.2f} TF/s)", flush=True)
