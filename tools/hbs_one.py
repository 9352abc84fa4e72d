import sys, os
sys.path.insert(0, '/root/repo') if os.path.exists('/root/repo') else None
import paper_2211_07572_b200 as S
sysm = S.assemble_fd5(S.helmholtz_bump_problem(1000, 1000, S.kappa_from_ppw(10, 1000)))
f = S.factorize(sysm, S.SolverConfig(b=60, compression=S.CompressionChoice.hbs, refine=0))
print("t_hbs", f.stats.t_hbs, "rank", f.hbs_max_rank)
