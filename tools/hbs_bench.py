"""HBS compression at scale: t_hbs / hbs_max_rank / residual for a few problems (GPU)."""
import sys
import time
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2211_07572_b200 as S  # noqa: E402

cases = {
    "poisson1000_b60": (lambda: S.poisson_log_problem(1000, 1000), 60),
    "helm1000_10ppw": (lambda: S.helmholtz_bump_problem(1000, 1000, S.kappa_from_ppw(10, 1000)), 0),
    "poisson2000": (lambda: S.poisson_log_problem(2000, 2000), 0),
    "helm2000_10ppw": (lambda: S.helmholtz_bump_problem(2000, 2000, S.kappa_from_ppw(10, 2000)), 0),
    "helm4000_10ppw_b150": (lambda: S.helmholtz_bump_problem(4000, 4000, S.kappa_from_ppw(10, 4000)), 150),
}
for name in (sys.argv[1:] or list(cases)):
    mk, b = cases[name]
    spec = mk()
    sysm = S.assemble_fd5(spec)
    for comp in (S.CompressionChoice.dense, S.CompressionChoice.hbs):
        t0 = time.perf_counter()
        try:
            fact = S.factorize(sysm, S.SolverConfig(b=b, compression=comp, refine=0))
        except S.CompressionError as e:
            print(f"{name} {comp.name}: CompressionError {e} (residual {e.residual_estimate:.2e})", flush=True)
            continue
        wall = time.perf_counter() - t0
        u = S.solve(fact, sysm.rhs)
        rep = S.error_report(sysm, u, None) if False else None
        st = fact.stats
        print(f"{name} {comp.name}: b={fact.b} t_stage1 {fact.t_stage1:.3f} s (hbs {st.t_hbs:.3f} s) "
              f"t_stage2 {fact.t_stage2:.3f} s wall {wall:.1f} s hbs_max_rank {fact.hbs_max_rank}", flush=True)
        del fact
