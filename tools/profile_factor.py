"""Run one (or a few) factorize + solve of a bench config for profiling (ncu launch lists)."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2211_07572_b200 as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--n1", type=int, default=0)
ap.add_argument("--n2", type=int, default=0)
ap.add_argument("--b", type=int, default=0)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--solve", action="store_true")
a = ap.parse_args()
kind, n1, n2, b, ppw, desc = bench.CONFIGS[a.config]
n1, n2, b = a.n1 or n1, a.n2 or n2, a.b or b
kappa = 0.0 if ppw is None else S.kappa_from_ppw(ppw, n2)
spec = (S.poisson_log_problem(n1, n2) if kind == 0 else
        S.helmholtz_problem(n1, n2, kappa) if kind == 1 else S.helmholtz_bump_problem(n1, n2, kappa))
sysm = S.assemble_fd5(spec)
for r in range(a.reps):
    t0 = time.perf_counter()
    f = S.factorize(sysm, S.SolverConfig(b=b, compression=S.CompressionChoice.dense))
    st = f.stats
    print(f"{n1}x{n2} b={b}: T={f.t_stage1 + f.t_stage2:.4f}s chain={st.t_chain:.4f} schur={st.t_schur:.4f} "
          f"asm={st.t_assemble:.4f} stage2={f.t_stage2:.4f} launches={st.gpu_launches} wall={time.perf_counter()-t0:.3f}",
          flush=True)
    if a.solve:
        for k in range(2):  # second call is warm
            u = S.solve(f, sysm.rhs)
            st = f.refresh_stats()
            import numpy as np
            r = np.linalg.norm(sysm.matvec(u).ravel() - sysm.rhs.ravel()) / np.linalg.norm(sysm.rhs)
            print(f"  solve[{k}]: {st.t_solve_last*1e3:.2f} ms (strip sweeps {st.t_solve_strips*1e3:.2f} ms) "
                  f"relres={r:.2e}", flush=True)
    f.close()
