import sys, torch
sys.path.insert(0, "/root/repo")
import bench, paper_2211_07572_b200 as S
for cfg in ["cfg2"]:
    spec, kappa = bench.problem(cfg)
    kind, n1, n2, b, ppw, desc = bench.CONFIGS[cfg]
    sysm = S.assemble_fd5(spec)
    dev = torch.device("cuda", 0)
    rp, ci, v = (torch.from_numpy(a).to(dev) for a in (sysm.row_ptr, sysm.col_idx, sysm.values))
    for refine in [1, 0, 0, 1]:
        try:
            f = S.factorize_device(n1, n2, rp, ci, v, S.SolverConfig(b=b, compression=S.CompressionChoice.dense, refine=refine))
            print(cfg, "refine", refine, "ok", f.t_stage1 + f.t_stage2, flush=True); f.close()
        except Exception as e:
            print(cfg, "refine", refine, "FAIL", e, flush=True)
