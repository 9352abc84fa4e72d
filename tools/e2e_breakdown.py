"""Where the end-to-end (host API) time goes beyond the device-timed factorization (cfg3)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2211_07572_b200 as S  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
kind, n1, n2, b, ppw, desc = bench.CONFIGS[cfg]
spec, kappa = bench.problem(cfg)
sysm = S.assemble_fd5(spec)
cfgS = S.SolverConfig(b=b, compression=S.CompressionChoice.dense)
for rep in range(3):
    t0 = time.perf_counter()
    f = S.factorize(sysm, cfgS)
    t1 = time.perf_counter()
    u = S.solve(f, sysm.rhs)
    t2 = time.perf_counter()
    st = f.refresh_stats()
    print(f"rep {rep}: factorize wall {t1 - t0:.3f} s (device {f.t_stage1 + f.t_stage2:.3f} s), "
          f"solve wall {(t2 - t1) * 1e3:.1f} ms (device {st.t_solve_last * 1e3:.1f} ms)", flush=True)
    t3 = time.perf_counter()
    u = S.solve(f, sysm.rhs)
    t4 = time.perf_counter()
    print(f"        second solve wall {(t4 - t3) * 1e3:.1f} ms", flush=True)
    t5 = time.perf_counter()
    f.close()
    print(f"        close {(time.perf_counter() - t5) * 1e3:.1f} ms", flush=True)
