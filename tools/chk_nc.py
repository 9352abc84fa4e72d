"""Solve-kernel variants on the same factorization: per-column residuals of 1/2/3-column solves
(DFMA NC=1/2/4) against the DMMA variant (SLB_SOLVE_DMMA=1 in a subprocess)."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(n, b, cols, refine):
    import paper_2211_07572_b200 as S
    kappa = S.kappa_from_ppw(10.0, n)
    sysm = S.assemble_fd5(S.helmholtz_bump_problem(n, n, kappa))
    fact = S.factorize(sysm, S.SolverConfig(b=b, refine=refine))
    f = np.column_stack([sysm.rhs] + [S.gaussian_matrix(sysm.dim(), 1, 2024 + c)[:, 0] for c in range(cols - 1)])
    u = S.solve(fact, f)
    res = np.linalg.norm(sysm.matvec(u) - f, axis=0) / np.linalg.norm(f, axis=0)
    np.save("/tmp/nc_u.npy", u)
    return res


if __name__ == "__main__":
    if sys.argv[1] == "--one":
        n, b, cols, refine = (int(x) for x in sys.argv[2:6])
        print("RES", " ".join(f"{x:.3e}" for x in run(n, b, cols, refine)), flush=True)
        sys.exit(0)
    n, b = int(sys.argv[1]), int(sys.argv[2])
    for cols in (1, 2, 3):
        for refine in (0, 1):
            out = {}
            for mode in ("dfma", "dmma"):
                env = dict(os.environ)
                if mode == "dmma":
                    env["SLB_SOLVE_DMMA"] = "1"
                p = subprocess.run([sys.executable, __file__, "--one", str(n), str(b), str(cols), str(refine)], env=env,
                                   capture_output=True, text=True, timeout=900)
                line = [x for x in p.stdout.splitlines() if x.startswith("RES")]
                out[mode] = (line[0] if line else "FAILED " + p.stderr[-500:], np.load("/tmp/nc_u.npy"))
            d = np.linalg.norm(out["dfma"][1] - out["dmma"][1]) / np.linalg.norm(out["dmma"][1])
            print(f"n={n} cols={cols} refine={refine}: dfma {out['dfma'][0]} | dmma {out['dmma'][0]} | diff {d:.2e}",
                  flush=True)
