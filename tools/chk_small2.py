import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_07572_b200 as S
n, b = int(sys.argv[1]), int(sys.argv[2])
kappa = S.kappa_from_ppw(10.0, n)
sysm = S.assemble_fd5(S.helmholtz_bump_problem(n, n, kappa))
fact = S.factorize(sysm, S.SolverConfig(b=b, refine=0))
f = np.column_stack([sysm.rhs, S.gaussian_matrix(sysm.dim(), 1, 2024)[:, 0]])
u = S.solve(fact, f)
print("res", np.linalg.norm(sysm.matvec(u) - f, axis=0) / np.linalg.norm(f, axis=0))
