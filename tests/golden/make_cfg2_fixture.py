"""Generates tests/golden/cfg2_oracle_fixture.npz (run here, on the CPU; ~5 min).

configs[1] of BASELINE.json: helmholtz_problem(1000, 1000, kappa_from_ppw(10, 1000)),
b = 60, dense mode.  The oracle (oracle/slablu_oracle.cpp, the reference's dense path
restated on OpenBLAS) factors and solves it; then the oracle solution is refined with
residuals computed in extended precision (numpy longdouble, 64-bit mantissa):

    u_{k+1} = u_k + A^{-1}_oracle (f - A u_k)       (residual in long double)

which converges to the exact discrete solution u* because cond(A) * eps << 1.  The
fixture stores, on every 97th unknown, u_oracle and u*, plus full-vector norms, so the
GPU test can hold the engine to the oracle's own distance from u* (SURVEY.md §7 hard
part 6: arbitration when conditioning blocks a 1e-10 comparison of two solvers).
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import oracle as O  # noqa: E402


def spmv_ld(sys_o, u):
    rows = np.repeat(np.arange(sys_o.dim), np.diff(sys_o.row_ptr))
    prod = sys_o.values.astype(np.longdouble) * u[sys_o.col_idx]
    out = np.zeros(sys_o.dim, np.longdouble)
    np.add.at(out, rows, prod)
    return out


def main():
    n, b = 1000, 60
    O.set_blas_threads(os.cpu_count() or 1)
    kappa = O.kappa_from_ppw(10.0, n)
    sys_o = O.assemble_canned(O.HELMHOLTZ, n, n, kappa)
    t = time.time()
    fact = O.factorize(sys_o, b=b, threads=os.cpu_count() or 1)
    print(f"oracle factorize {time.time() - t:.1f} s", flush=True)
    f = sys_o.rhs.astype(np.longdouble)
    u_o = fact.solve(sys_o.rhs)[:, 0]
    u = u_o.astype(np.longdouble)
    hist = []
    for it in range(4):
        r = f - spmv_ld(sys_o, u)
        hist.append(float(np.sqrt(np.sum(r * r)) / np.sqrt(np.sum(f * f))))
        du = fact.solve(r.astype(np.float64))[:, 0]
        u = u + du.astype(np.longdouble)
        print(f"refinement {it}: residual {hist[-1]:.3e}, |du|/|u| {np.linalg.norm(du) / float(np.sqrt(np.sum(u*u))):.3e}",
              flush=True)
    r = f - spmv_ld(sys_o, u)
    hist.append(float(np.sqrt(np.sum(r * r)) / np.sqrt(np.sum(f * f))))
    u_star = u.astype(np.float64)
    idx = np.arange(0, n * n, 97, dtype=np.int64)
    err = np.linalg.norm(u_o - u_star) / np.linalg.norm(u_star)
    print(f"oracle |u_o - u*|/|u*| = {err:.3e}; residual history {hist}")
    np.savez_compressed(os.path.join(HERE, "cfg2_oracle_fixture.npz"), n=n, b=b, kappa=kappa,
                        nnz=sys_o.values.size, idx=idx, u_oracle_sub=u_o[idx], u_star_sub=u_star[idx],
                        u_star_norm=np.linalg.norm(u_star), oracle_err_full=err,
                        residual_history=np.array(hist))


if __name__ == "__main__":
    main()
