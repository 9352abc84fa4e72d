import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_07572_b200 as S
n, b, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
kappa = S.kappa_from_ppw(10.0, n)
sysm = S.assemble_fd5(S.helmholtz_bump_problem(n, n, kappa))
fact = S.factorize(sysm, S.SolverConfig(b=b, refine=0))
for cols in (1, 2, 3):
    f = np.column_stack([sysm.rhs] + [S.gaussian_matrix(sysm.dim(), 1, 2024 + c)[:, 0] for c in range(cols - 1)])
    ref = S.solve(fact, f)
    bad = []
    for r in range(reps):
        u = S.solve(fact, f)
        dd = np.abs(u - ref)
        if dd.max() > 0:
            idx = np.argwhere(dd > 0)
            bad.append((r, float(dd.max()), len(idx), idx[:3].tolist()))
    print(f"cols={cols}: {len(bad)} of {reps} differ: {bad[:4]}", flush=True)
