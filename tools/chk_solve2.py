"""Solve-kernel A/B check: the version-2 cluster sweeps (solve2.cu) against the round-1 kernel
(SLB_SOLVE_V1=1) and the residual, on a few geometries.  Usage: python tools/chk_solve2.py [big]"""
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(case):
    import paper_2211_07572_b200 as S
    kind, n1, n2, b, ppw, nrhs = case
    kappa = S.kappa_from_ppw(ppw, n2) if ppw else 0.0
    spec = S.helmholtz_bump_problem(n1, n2, kappa) if kind == 2 else S.helmholtz_problem(n1, n2, kappa)
    sysm = S.assemble_fd5(spec)
    fact = S.factorize(sysm, S.SolverConfig(b=b, refine=0, compression=S.CompressionChoice.dense))
    f = np.column_stack([sysm.rhs] + [S.gaussian_matrix(sysm.dim(), 1, 7 + c)[:, 0] for c in range(nrhs - 1)])
    u = S.solve(fact, f)
    u = S.solve(fact, f)
    st = fact.refresh_stats()
    res = np.linalg.norm(sysm.matvec(u) - f) / np.linalg.norm(f)
    red = fact.reduce_rhs(f)
    np.save("/tmp/chk_u.npy", u)
    np.save("/tmp/chk_red.npy", red)
    return res, st.t_solve_last, st.t_solve_strips


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--one":
        case = eval(sys.argv[2])
        res, t, ts = run(case)
        print(f"RESULT {res:.3e} {t * 1e3:.3f} {ts * 1e3:.3f}", flush=True)
        sys.exit(0)
    cases = [(2, 64, 48, 7, 10.0, 1), (1, 120, 96, 11, 10.0, 3), (2, 200, 200, 20, 10.0, 8), (2, 1000, 1000, 60, 10.0, 1)]
    if len(sys.argv) > 1 and sys.argv[1] == "big":
        cases.append((2, 4000, 4000, 150, 10.0, 1))
    for case in cases:
        out = {}
        for v in ("1", "2"):
            env = dict(os.environ)
            if v == "1":
                env["SLB_SOLVE_V1"] = "1"
            else:
                env.pop("SLB_SOLVE_V1", None)
            t0 = time.time()
            p = subprocess.run([sys.executable, __file__, "--one", repr(case)], env=env, capture_output=True, text=True,
                               timeout=600)
            line = [x for x in p.stdout.splitlines() if x.startswith("RESULT")]
            if p.returncode != 0 or not line:
                print(f"case {case} v{v}: FAILED rc={p.returncode}\n{p.stdout[-2000:]}\n{p.stderr[-3000:]}", flush=True)
                sys.exit(1)
            out[v] = (line[0].split()[1:], np.load("/tmp/chk_u.npy"), np.load("/tmp/chk_red.npy"))
            print(f"case {case} v{v}: residual {out[v][0][0]} solve {out[v][0][1]} ms strips {out[v][0][2]} ms "
                  f"({time.time() - t0:.1f}s)", flush=True)
        du = np.linalg.norm(out["1"][1] - out["2"][1]) / np.linalg.norm(out["1"][1])
        dr = np.linalg.norm(out["1"][2] - out["2"][2]) / np.linalg.norm(out["1"][2])
        print(f"case {case}: v2 vs v1 solution {du:.3e}, reduce_rhs {dr:.3e}", flush=True)
