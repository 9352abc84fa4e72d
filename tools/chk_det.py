"""Determinism probe of the solve stages (staged ABI) for 1/2/3 columns, repeated."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_07572_b200 as S  # noqa: E402

n, b, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
kappa = S.kappa_from_ppw(10.0, n)
sysm = S.assemble_fd5(S.helmholtz_bump_problem(n, n, kappa))
fact = S.factorize(sysm, S.SolverConfig(b=b, refine=0))
for cols in (1, 2, 3):
    f = np.column_stack([sysm.rhs] + [S.gaussian_matrix(sysm.dim(), 1, 2024 + c)[:, 0] for c in range(cols - 1)])
    reds = [fact.reduce_rhs(f) for _ in range(reps)]
    uis = [fact.sweep_solve(reds[0]) for _ in range(reps)]
    us = [fact.recover(f, uis[0]) for _ in range(reps)]
    d = lambda xs: [float(np.abs(x - xs[0]).max()) for x in xs]
    print(f"cols={cols} reduce {d(reds)} sweep {d(uis)} recover {d(us)}", flush=True)
