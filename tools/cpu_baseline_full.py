"""Full (not extrapolated) CPU-baseline runs of the reference path at cfg1 and cfg2, dense mode
(BASELINE.md section 3), beside the GPU engine on the same inputs.

The oracle port (oracle/, the reference's dense path restated on the image's OpenBLAS) factors
and solves each config end to end with 1 BLAS thread (the reference's default, threads = 1) and
with every host core; the GPU engine runs the same system.  Prints one JSON object.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import paper_2211_07572_b200 as S  # noqa: E402

CONFIGS = {
    "cfg1": (0, 255, 255, 31, None),
    "cfg2": (1, 1000, 1000, 60, 10.0),
}


def run(cfg, threads_list):
    kind, n1, n2, b, ppw = CONFIGS[cfg]
    kappa = 0.0 if ppw is None else O.kappa_from_ppw(ppw, n2)
    osys = O.assemble_canned(kind, n1, n2, kappa)
    out = {"config": cfg, "N": n1 * n2, "b": b, "cpu": [], "gpu": None}
    u_cpu = None
    for th in threads_list:
        O.set_blas_threads(th)
        t0 = time.perf_counter()
        f = O.factorize(osys, b=b, threads=th)
        tf = time.perf_counter() - t0
        t0 = time.perf_counter()
        u = f.solve(osys.rhs)
        ts = time.perf_counter() - t0
        u_cpu = u[:, 0]
        out["cpu"].append({"threads": th, "T_factor_s": f.t_stage1 + f.t_stage2, "wall_factor_s": tf,
                           "T_solve_s": ts, "dof_s": n1 * n2 / (f.t_stage1 + f.t_stage2)})
        print(json.dumps(out["cpu"][-1]), file=sys.stderr, flush=True)
        del f
    spec = (S.poisson_log_problem(n1, n2) if kind == 0 else S.helmholtz_problem(n1, n2, kappa))
    gsys = S.assemble_fd5(spec)
    cfgS = S.SolverConfig(b=b, compression=S.CompressionChoice.dense)
    S.factorize(gsys, cfgS)  # warm-up
    fact = S.factorize(gsys, cfgS)
    import torch
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    u = S.solve(fact, gsys.rhs)[:, 0]
    ts = time.perf_counter() - t0
    T = fact.t_stage1 + fact.t_stage2
    out["gpu"] = {"T_factor_s": T, "T_solve_s_wall": ts, "dof_s": n1 * n2 / T,
                  "rel_diff_vs_cpu": float(np.linalg.norm(u - u_cpu) / np.linalg.norm(u_cpu))}
    out["speedup_factor"] = out["cpu"][0]["T_factor_s"] / T
    return out


if __name__ == "__main__":
    nproc = os.cpu_count() or 1
    res = {"host_cores": nproc, "runs": [run(c, [1, nproc]) for c in (sys.argv[1:] or ["cfg1", "cfg2"])]}
    print(json.dumps(res, indent=1))
