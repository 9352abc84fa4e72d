#!/usr/bin/env python
"""Benchmark of the B200-native SlabLU engine on BASELINE.json's metric.

metric: factorization DOF/s (N / T_factor) of the dense SlabLU path on
configs[2] = 4000x4000 variable-coefficient (bump) Helmholtz, b = 150,
kappa = kappa_from_ppw(10, 4000) (N = 16M), plus solve ms/RHS.

A "step" is one factorization of that operator.  `value` is timed on the
device (CUDA events inside the engine, CSR already resident in HBM);
`e2e` times the public host API (pinned host CSR -> factorize -> solve one
RHS -> host solution).  Inputs and factors (~100 GB) exceed the 126 MB L2,
so no L2 flush is needed between steps.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config cfg3]

--impl reference times the reference's CPU path (the oracle port, all host
threads) on a bounded sample of the same workload and prints the same JSON
line with "impl": "reference".
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (kind, n1, n2, b, ppw or None for poisson, description)
    "cfg1": (0, 255, 255, 31, None, "5-point FD Poisson 255x255, b=31"),
    "cfg2": (1, 1000, 1000, 60, 10.0, "5-point FD Helmholtz 1000x1000, 10 ppw, b=60 (dense)"),
    "cfg3": (2, 4000, 4000, 150, 10.0, "5-point FD bump Helmholtz 4000x4000 (N=16M), 10 ppw, b=150 (dense)"),
    "cfg4": (1, 2000, 2000, 100, 10.0, "5-point FD Helmholtz 2000x2000 (rectangle stand-in), 10 ppw, b=100, 64 RHS"),
}
# DRAM bytes of one Schur-sweep launch (ncu --set full capture of the current kernel,
# profiles/ncu_schur_cfg3_r02.txt)
SCHUR_DRAM_BYTES = {"cfg3": 1.912814e12 + 0.521009e12}
FP64_PEAK_TFLOPS = 37.067  # measured DMMA peak on this pool's B200 (profiles/fp64_peak_r01.json)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def geometry(n1, n2, b):
    """Strip widths and interface count exactly as partition.hpp:70-91."""
    ints, col, t, nifc = [], 0, 1, 0
    while col < n1:
        ifc = t * (b + 1) - 1
        stop = min(ifc, n1)
        if stop > col:
            ints.append(stop - col)
        col = stop
        if col == ifc and col < n1:
            nifc += 1
            col += 1
        t += 1
    return ints, nifc


def algorithmic_flops(n1, n2, b):
    """F_factor = sum 2 w^3 n2 + sum 3 c w^2 n2^2 + ((k-1) 14/3 + 2/3) n2^3."""
    widths, k = geometry(n1, n2, b)
    band = sum(2.0 * w ** 3 * n2 for w in widths)
    schur = 0.0
    for s, w in enumerate(widths):
        c = (1 if s > 0 else 0) + (1 if s < k else 0)
        schur += 3.0 * c * w * w * n2 * n2
    sweep = ((k - 1) * 14.0 / 3.0 + 2.0 / 3.0) * n2 ** 3
    return band, schur, sweep


def solve_bytes(n1, n2, b, nrhs):
    widths, k = geometry(n1, n2, b)
    band = sum((3 * w + 1) * w * n2 for w in widths)
    return 8.0 * (2 * band + (4 * k - 3) * n2 * n2) + nrhs * 8.0 * 3 * n1 * n2


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self):
        self.rows, self.proc = [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200", "-i", os.environ.get("LOCAL_RANK", "0")],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sms.append(float(r[1]))
                mx = float(r[2])
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                pass
        return {"sm_mhz": float(np.median(sms)) if sms else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sms)}


def problem(cfg):
    import paper_2211_07572_b200 as S
    kind, n1, n2, b, ppw, _ = CONFIGS[cfg]
    kappa = 0.0 if ppw is None else S.kappa_from_ppw(ppw, n2)
    spec = (S.poisson_log_problem(n1, n2) if kind == 0 else
            S.helmholtz_problem(n1, n2, kappa) if kind == 1 else S.helmholtz_bump_problem(n1, n2, kappa))
    return spec, kappa


_CPU_CACHE = {}


def cpu_sample(cfg, threads):
    """Bounded CPU-baseline sample of the reference path (oracle port), extrapolated to T_factor.
    The system is assembled once per process and the dgbtrs sample size calibrated once, so a step
    is one full-strip dgbtrf, one dgbtrs sample and one stage-two step (a few seconds)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    kind, n1, n2, b, ppw, _ = CONFIGS[cfg]
    O.set_blas_threads(threads)
    if cfg not in _CPU_CACHE:
        kappa = 0.0 if ppw is None else O.kappa_from_ppw(ppw, n2)
        _CPU_CACHE[cfg] = {"sys": O.assemble_canned(kind, n1, n2, kappa), "nrhs": None}
    cache = _CPU_CACHE[cfg]
    sysm = cache["sys"]
    widths, k = geometry(n1, n2, b)
    full = max(range(len(widths)), key=lambda s: widths[s] if 0 < s < k else -1)
    if cache["nrhs"] is None:  # calibrate once: a dgbtrs sample of >= 0.5 s
        nrhs = 8
        t_trf, t_trs = O.time_slab_sample(sysm, b, full, nrhs)
        while t_trs < 0.5 and nrhs < n2:
            nrhs = min(n2, nrhs * 4)
            t_trf, t_trs = O.time_slab_sample(sysm, b, full, nrhs)
        cache["nrhs"] = nrhs
    else:
        nrhs = cache["nrhs"]
        t_trf, t_trs = O.time_slab_sample(sysm, b, full, nrhs)
    per_col = t_trs / nrhs
    w_full = widths[full]
    t1 = 0.0
    for s, w in enumerate(widths):
        calls = (2 if (s > 0 and s < k) else 1) + (2 if (s > 0 and s < k) else 0)  # build_reduced dgbtrs calls
        scale = (w / w_full)
        t1 += t_trf * scale + calls * n2 * per_col * scale  # band ops ~ n w^2, per column ~ n w
    t_step = O.time_sweep_step(n2) if k > 1 else 0.0
    t2 = max(k - 1, 0) * t_step + (t_step / 4.0 if k > 0 else 0.0)
    T = t1 + t2
    return {"T_factor_s": T, "dof_s": n1 * n2 / T, "sample": (
        f"oracle port (OpenBLAS {threads} threads): one full strip (w={w_full}) dgbtrf + dgbtrs with {nrhs} of "
        f"{n2} identity RHS, and one stage-two step at n2={n2}; extrapolated over {len(widths)} strips "
        f"x build_reduced call counts and {k - 1} sweep steps"), "t_trf": t_trf, "t_trs_per_rhs": per_col,
        "t_sweep_step": t_step}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    kind, n1, n2, b, ppw, desc = CONFIGS[args.config]
    vals = []
    t0 = time.perf_counter()
    for step in range(args.warmup + args.steps):
        r = cpu_sample(args.config, threads)
        if step >= args.warmup:
            vals.append(r["dof_s"])
        if time.perf_counter() - t0 > 900:  # safety cap; a step is a few seconds (assembly cached)
            break
    v = float(np.median(vals)) if vals else r["dof_s"]
    line = {"metric": "factorization DOF/s (dense SlabLU, N=16M FD bump Helmholtz)" if args.config == "cfg3" else
            f"factorization DOF/s ({desc})", "value": v, "unit": "DOF/s", "n_gpus": args.gpus, "steps": len(vals),
            "warmup": args.warmup, "ms_per_step": n1 * n2 / v * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (deterministic canned problem)",
            "config": {"workload": desc, "n1": n1, "n2": n2, "b": b, "N": n1 * n2}, "impl": "reference",
            "cpu_baseline": {"value": v, "unit": "DOF/s", "cores": threads, "kind": "port", "sample": r["sample"]},
            "e2e": {"value": v, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import paper_2211_07572_b200 as S

    rank, world = 0, 1  # N > 1 runs run_ours_sharded
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    kind, n1, n2, b, ppw, desc = CONFIGS[args.config]
    spec, kappa = problem(args.config)
    t_asm = time.perf_counter()
    sysm = S.assemble_fd5(spec)
    log(f"[bench] assembled {desc}: N={sysm.dim()}, nnz={len(sysm.values)} in {time.perf_counter() - t_asm:.1f}s")
    N = sysm.dim()
    cfgS = S.SolverConfig(b=b, compression=S.CompressionChoice.dense, device=local)
    dev = torch.device("cuda", local)
    d_rp = torch.from_numpy(sysm.row_ptr).to(dev)
    d_ci = torch.from_numpy(sysm.col_idx).to(dev)
    d_v = torch.from_numpy(sysm.values).to(dev)
    # pinned host inputs for the end-to-end leg
    h_rp = torch.from_numpy(sysm.row_ptr).pin_memory()
    h_ci = torch.from_numpy(sysm.col_idx).pin_memory()
    h_v = torch.from_numpy(sysm.values).pin_memory()
    h_f = torch.from_numpy(sysm.rhs).pin_memory()
    h_u = torch.empty(N, dtype=torch.float64).pin_memory()
    sysp = S.SparseSystem(h_rp.numpy(), h_ci.numpy(), h_v.numpy(), h_f.numpy(), n1, n2, sysm.h)

    def barrier():
        torch.cuda.synchronize()

    for w in range(args.warmup):
        f = S.factorize_device(n1, n2, d_rp, d_ci, d_v, cfgS)
        log(f"[bench] warmup {w}: T_factor {f.t_stage1 + f.t_stage2:.3f}s (chain {f.stats.t_chain:.3f}, "
            f"schur {f.stats.t_schur:.3f}, asm {f.stats.t_assemble:.3f}, stage2 {f.t_stage2:.3f})")
        f.close()
    # working set vs the 126 MB L2: the factor operators alone are 32 Wp^2 n2 bytes per strip
    widths, _ = geometry(n1, n2, b)
    wp = -(-max(widths) // 8) * 8
    factor_bytes = len(widths) * 32 * wp * wp * n2
    flush = factor_bytes < 4 * 126e6
    l2buf = torch.empty(64 << 20, dtype=torch.float64, device=dev) if flush else None  # 512 MB
    clocks = ClockSampler()
    clocks.start()
    barrier()
    t_fac, t_schur, t_chain, t_st2, launches = [], [], [], [], []
    wall0 = time.perf_counter()
    fact = None
    for s in range(args.steps):
        if fact is not None:
            fact.close()
        if l2buf is not None:  # evict the previous step's data (not timed: engine events)
            l2buf.fill_(float(s))
            torch.cuda.synchronize()
        fact = S.factorize_device(n1, n2, d_rp, d_ci, d_v, cfgS)
        t_fac.append(fact.t_stage1 + fact.t_stage2)
        t_schur.append(fact.stats.t_schur)
        t_chain.append(fact.stats.t_chain)
        t_st2.append(fact.t_stage2)
        launches.append(fact.stats.gpu_launches)
    barrier()
    wall = time.perf_counter() - wall0
    # solve: 1 RHS (device-resident), unrefined (the reference's computation: reduce_rhs, sweep
    # solve, recover_interiors) and with one refinement step (SolverConfig.refine = 1, the default),
    # then a block of RHS for ms/RHS (64 at cfg4, as BASELINE.json configs[3] asks)
    d_f = torch.from_numpy(sysm.rhs).to(dev).reshape(1, N)
    d_u = torch.empty_like(d_f)
    d_u0 = torch.empty_like(d_f)

    def timed_solve(f_, u_, refine, reps=3):
        fact.set_refine(refine)
        S.solve_device(fact, f_, u_)  # warm (first-call allocations)
        ts = []
        for _ in range(reps):
            S.solve_device(fact, f_, u_)
            ts.append(fact.refresh_stats().t_solve_last)
        return float(np.median(ts)), fact.refresh_stats().t_solve_strips

    t_solve1, t_solve1_strips = timed_solve(d_f, d_u, 1)
    t_solve0, t_solve0_strips = timed_solve(d_f, d_u0, 0)
    nrhs = 64 if args.config in ("cfg4", "cfg2", "cfg1") else 8
    d_F = torch.randn(nrhs, N, dtype=torch.float64, device=dev)
    d_U = torch.empty_like(d_F)
    t_solveB, _ = timed_solve(d_F, d_U, 0, reps=2)
    t_solveB1, _ = timed_solve(d_F, d_U, 1, reps=2)
    fact.set_refine(cfgS.refine)
    clk = clocks.stop()
    # parity of this run (size-independent): residuals of the 1-RHS solves
    u = d_u.reshape(N).cpu().numpy()
    res = float(np.linalg.norm(sysm.matvec(u) - sysm.rhs) / np.linalg.norm(sysm.rhs))
    u0 = d_u0.reshape(N).cpu().numpy()
    res0 = float(np.linalg.norm(sysm.matvec(u0) - sysm.rhs) / np.linalg.norm(sysm.rhs))
    fact.close()
    # end-to-end leg: pinned host CSR -> factorize -> solve -> host u
    t_e2e = []
    for s in range(max(1, min(args.steps, 2))):
        barrier()
        t0 = time.perf_counter()
        fe = S.factorize(sysp, cfgS)
        u_h = S.solve(fe, h_f.numpy())
        h_u.numpy()[:] = u_h[:, 0]
        barrier()
        t_e2e.append(time.perf_counter() - t0)
        fe.close()
    h2d = sysm.row_ptr.nbytes + sysm.col_idx.nbytes + sysm.values.nbytes + sysm.rhs.nbytes
    d2h = N * 8
    T = float(np.mean(t_fac))
    te = float(np.mean(t_e2e))
    band, schur, sweep = algorithmic_flops(n1, n2, b)
    T_schur = float(np.mean(t_schur))
    cpu = None
    if rank == 0 and not args.no_cpu:
        try:
            cpu = cpu_sample(args.config, os.cpu_count() or 1)
        except Exception as e:  # reported, not fatal
            log(f"[bench] cpu baseline failed: {e}")
    if rank != 0:
        return
    line = {
        "metric": "factorization DOF/s (dense SlabLU, N=16M FD bump Helmholtz)" if args.config == "cfg3"
        else f"factorization DOF/s ({desc})",
        "value": world * N / T, "unit": "DOF/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": T * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (deterministic canned problem, inputs resident in HBM; factors > L2 so no flush needed)",
        "config": {"workload": desc, "n1": n1, "n2": n2, "b": b, "kappa": kappa, "N": N,
                   "parallelism": "single-gpu",
                   "l2": (f"L2 flushed between steps (512 MB write); factor operators {factor_bytes / 1e6:.0f} MB"
                          if flush else f"no flush needed: factor operators {factor_bytes / 1e9:.1f} GB >> 126 MB L2")},
        "T_factor_s": T, "T_stage1_s": T - float(np.mean(t_st2)), "T_stage2_s": float(np.mean(t_st2)),
        "phases_s": {"chain": float(np.mean(t_chain)), "schur": T_schur},
        "solve_ms_per_rhs": t_solve0 * 1e3, "solve_ms_per_rhs_refined": t_solve1 * 1e3,
        "solve_ms_per_rhs_batched": t_solveB / nrhs * 1e3, "solve_ms_per_rhs_batched_refined": t_solveB1 / nrhs * 1e3,
        "solve_batch": nrhs, "solve_strip_sweeps_ms": t_solve0_strips * 1e3,
        "solve_note": ("solve_ms_per_rhs = one pass (reduce_rhs, sweep solve, recover_interiors: the reference's "
                       "computation); _refined adds one step of iterative refinement (SolverConfig.refine=1, the "
                       "default): a residual and a second pass"),
        "relerr_res": res, "relerr_res_unrefined": res0,
        "gpu_launches": int(np.mean(launches)),
        "e2e": {"value": world * N / te, "unit": "DOF/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": d2h,
                "seconds": te},
        "roofline": {"bound": "tensor", "kernel": "schur_kernel (slab Schur sweeps)",
                     "achieved": schur / T_schur / 1e12, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": schur / T_schur / 1e12 / FP64_PEAK_TFLOPS,
                     "traffic": SCHUR_DRAM_BYTES.get(args.config),
                     "traffic_unit": "bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum, ncu --set full)",
                     "algorithmic_flops_per_launch": schur,
                     "peak_source": "FP64 DMMA measured on this pool (profiles/fp64_peak_r01.json); "
                                    "MEASURED_PEAKS.json has no FP64 entry",
                     "factor_frac": (band + schur + sweep) / T / 1e12 / FP64_PEAK_TFLOPS,
                     "solve_frac_of_hbm": solve_bytes(n1, n2, b, 1) / t_solve0 / 1e9 / 6553.3,
                     "solve_frac_of_hbm_refined": (2 * solve_bytes(n1, n2, b, 1) + 20.0 * len(sysm.values) + 24.0 * N)
                     / t_solve1 / 1e9 / 6553.3,
                     "solve_frac_of_hbm_batched": solve_bytes(n1, n2, b, nrhs) / t_solveB / 1e9 / 6553.3},
        "clocks": clk, "wall_s": wall,
    }
    if cpu is not None:
        line["cpu_baseline"] = {"value": cpu["dof_s"], "unit": "DOF/s", "cores": os.cpu_count(), "kind": "port",
                                "sample": cpu["sample"], "T_factor_s": cpu["T_factor_s"]}
    print(json.dumps(line), flush=True)


def run_ours_sharded(args):
    """N > 1: strong scaling of ONE cfg factorization over N GPUs: rank r factors
    its contiguous strips (stage one, no communication), then stage two and the solve are pipelined
    over the ranks with NCCL send/recv of one n2 x n2 (n2 x nrhs) message per rank boundary."""
    import torch
    import torch.distributed as dist
    import paper_2211_07572_b200 as S
    from paper_2211_07572_b200 import distributed as D

    for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29533"), ("RANK", "0"), ("WORLD_SIZE", "1")):
        os.environ.setdefault(k, v)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    kind, n1, n2, b, ppw, desc = CONFIGS[args.config]
    spec, kappa = problem(args.config)
    sysm = S.assemble_fd5(spec)
    N = sysm.dim()
    dev = torch.device("cuda", local)
    cfgS = S.SolverConfig(b=b, compression=S.CompressionChoice.dense, device=local)
    d_rp = torch.from_numpy(sysm.row_ptr).to(dev)
    d_ci = torch.from_numpy(sysm.col_idx).to(dev)
    d_v = torch.from_numpy(sysm.values).to(dev)
    ex = D.TorchExchange()

    def step():
        sh = D.Shard(n1, n2, d_rp, d_ci, d_v, cfgS, rank, world)
        D.factorize_dist(sh, ex)
        return sh

    def timed(fn):
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) * 1e-3], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return out, float(t[0])

    for w in range(args.warmup):
        sh, t = timed(step)
        log(f"[bench r{rank}] warmup {w}: {t:.3f}s (stage1 {sh.stats.t_stage1:.3f}, sweep {sh.refresh_stats().t_stage2:.3f})")
        sh.close()
    clocks = ClockSampler()
    clocks.start()
    ts, sh = [], None
    log(f"[bench r{rank}] timed steps")
    for s in range(args.steps):
        if sh is not None:
            sh.close()
        sh, t = timed(step)
        ts.append(t)
    st = sh.refresh_stats()
    log(f"[bench r{rank}] solve")
    d_f = torch.from_numpy(sysm.rhs).to(dev).reshape(1, N)
    for _ in range(2):  # second solve is the timed one (first-call allocations)
        d_u, t_solve = timed(lambda: D.solve_dist_refined(sh, d_f, ex, refine=1))
    clk = clocks.stop()
    res = float(np.linalg.norm(sysm.matvec(d_u.reshape(N).cpu().numpy()) - sysm.rhs) / np.linalg.norm(sysm.rhs))
    t_schur = st.t_schur
    sh.close()
    # end to end: pinned host CSR -> device, sharded factorize, pipelined solve, solution -> host
    h_rp = torch.from_numpy(sysm.row_ptr).pin_memory()
    h_ci = torch.from_numpy(sysm.col_idx).pin_memory()
    h_v = torch.from_numpy(sysm.values).pin_memory()
    h_f = torch.from_numpy(sysm.rhs).pin_memory()
    h_u = torch.empty(N, dtype=torch.float64).pin_memory()

    def e2e():
        rp, ci, v = h_rp.to(dev, non_blocking=True), h_ci.to(dev, non_blocking=True), h_v.to(dev, non_blocking=True)
        f = h_f.to(dev, non_blocking=True).reshape(1, N)
        torch.cuda.current_stream().synchronize()  # the engine reads the inputs on its own stream
        s2 = D.Shard(n1, n2, rp, ci, v, cfgS, rank, world)
        D.factorize_dist(s2, ex)
        u = D.solve_dist_refined(s2, f, ex, refine=1)
        h_u.copy_(u.reshape(N))
        s2.close()

    log(f"[bench r{rank}] e2e")
    _, te = timed(e2e)
    T = float(np.mean(ts))
    if rank == 0:
        band, schur, sweep = algorithmic_flops(n1, n2, b)
        plan = D.shard_plan(n1, n2, b, 0, world)
        widths, k = geometry(n1, n2, b)
        local_schur = schur * (plan.s_end - plan.s_begin) / len(widths)
        h2d = sysm.row_ptr.nbytes + sysm.col_idx.nbytes + sysm.values.nbytes + sysm.rhs.nbytes
        line = {
            "metric": "factorization DOF/s (dense SlabLU, N=16M FD bump Helmholtz)" if args.config == "cfg3"
            else f"factorization DOF/s ({desc})",
            "value": N / T, "unit": "DOF/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": T * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (deterministic canned problem, CSR resident in HBM on every rank; factors > L2)",
            "config": {"workload": desc, "n1": n1, "n2": n2, "b": b, "kappa": kappa, "N": N,
                       "parallelism": f"strip-sharded x{world} (stage two / solve pipelined, NCCL send/recv)",
                       "l2": "inputs+factors >> 126 MB L2"},
            "T_factor_s": T, "solve_ms_per_rhs": t_solve * 1e3, "relerr_res": res,
            "gpu_launches": int(st.gpu_launches),
            "e2e": {"value": N / te, "unit": "DOF/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": N * 8,
                    "seconds": te},
            "roofline": {"bound": "tensor", "kernel": "schur_kernel (slab Schur sweeps, rank 0 shard)",
                         "achieved": local_schur / t_schur / 1e12, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": local_schur / t_schur / 1e12 / FP64_PEAK_TFLOPS, "traffic": None},
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--sharded", action="store_true", help="use the strip-sharded multi-GPU path even at N=1")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif int(os.environ.get("WORLD_SIZE", "1")) > 1 or args.sharded:
        run_ours_sharded(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
