"""Unrefined relative residual at cfg2 (1000^2 Helmholtz 10 ppw, b=60, dense)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2211_07572_b200 as S
n = 1000
sysm = S.assemble_fd5(S.helmholtz_problem(n, n, S.kappa_from_ppw(10.0, n)))
f = S.factorize(sysm, S.SolverConfig(b=60, compression=S.CompressionChoice.dense, refine=0))
u = S.solve(f, sysm.rhs)[:, 0]
res = np.linalg.norm(sysm.matvec(u).ravel() - sysm.rhs) / np.linalg.norm(sysm.rhs)
print(os.environ.get("TAG", ""), f"relerr_res unrefined {res:.3e}")
