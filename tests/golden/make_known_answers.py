"""Extract the reference's known-answer values for the SlabLU hot path.

Run in the build container (needs /root/reference, read-only):
    python tests/golden/make_known_answers.py
Writes tests/golden/reference_known_answers.json.  Each value is read from
the reference test source at the cited file:line (the script fails if the
literal is not found there), so the fixture's provenance is checkable.
"""
import json
import os
import re
import sys

REF = "/root/reference/proj/tests"

# (key, file, line, regex with one or more float groups, description)
SPECS = [
    ("poisson_relerr_true_slablu_b4_n16", "test_driver.cpp", 248, r"Approx\(([-0-9.e]+)\)", "run_problem poisson_log 16x16, b=4, rel tol 1e-4"),
    ("poisson_relerr_true_slablu_b4_n32", "test_driver.cpp", 250, r"Approx\(([-0-9.e]+)\)", "run_problem poisson_log 32x32, b=4, rel tol 1e-4"),
    ("poisson_relerr_true_slablu_b4_n64", "test_driver.cpp", 252, r"Approx\(([-0-9.e]+)\)", "run_problem poisson_log 64x64, b=4, rel tol 1e-4"),
    ("poisson_relerr_true_dense_n16", "test_problem.cpp", 175, r"Approx\(([-0-9.e]+)\)", "dense LU poisson_log 16x16, rel tol 1e-5"),
    ("poisson_relerr_true_dense_n32", "test_problem.cpp", 176, r"Approx\(([-0-9.e]+)\)", "dense LU poisson_log 32x32, rel tol 1e-5"),
    ("poisson_relerr_true_dense_n64", "test_problem.cpp", 177, r"Approx\(([-0-9.e]+)\)", "dense LU poisson_log 64x64, rel tol 1e-5"),
    ("kappa_from_ppw_250_512", "test_problem.cpp", 222, r"Approx\(([-0-9.e]+)\)", "kappa_from_ppw(250, 512), rel 1e-6"),
    ("bessel_j0_table", "test_problem.cpp", 211, r"\{([-0-9.e]+), ([-0-9.e]+)\},\s+\{([-0-9.e]+), ([-0-9.e]+)\}", "J0 table rows 1-2 (t, value), abs 1e-13"),
    ("bessel_j0_table_2", "test_problem.cpp", 212, r"\{([-0-9.e]+), ([-0-9.e]+)\},\s+\{([-0-9.e]+), ([-0-9.e]+)\}", "J0 table rows 3-4"),
    ("bessel_j0_table_3", "test_problem.cpp", 213, r"\{([-0-9.e]+), ([-0-9.e]+)\},\s*\{([-0-9.e]+), ([-0-9.e]+)\}", "J0 table rows 5-6"),
    ("helmholtz_true_0p9_0p5_k1", "test_problem.cpp", 195, r"^\s+([0-9.]+)\)", "true_solution_helmholtz(0.9, 0.5, 1.0), abs 1e-14"),
    ("dirichlet_fold_corner", "test_problem.cpp", 105, r"== ([0-9.]+)\)", "corner rhs with g=x+y, load 7, h=0.25"),
    ("dirichlet_fold_interior", "test_problem.cpp", 107, r"== ([0-9.]+)\)", "interior rhs keeps the body load"),
    ("hand9x9_diag_off", "test_problem.cpp", 76, r"d = ([-0-9.]+), o = ([-0-9.]+);", "9x9 hand matrix, h=0.25: diag, off"),
    ("choose_b_c0p5", "test_driver.cpp", 57, r"choose_b\((\d+), (\d+), config\) == (\d+)", "c=0.5: n1, n2, b"),
    ("choose_b_c0p6", "test_driver.cpp", 59, r"choose_b\((\d+), (\d+), config\) == (\d+)", "c=0.6"),
    ("choose_b_c0p54", "test_driver.cpp", 61, r"choose_b\((\d+), (\d+), config\) == (\d+)", "c=0.54"),
    ("choose_b_clamp_hi", "test_driver.cpp", 64, r"choose_b\((\d+), (\d+), config\) == (\d+)", "c=0.6 clamp n1/2"),
    ("choose_b_clamp_lo", "test_driver.cpp", 66, r"choose_b\((\d+), (\d+), config\) == (\d+)", "c=0.05 clamp 10"),
    ("choose_b_explicit", "test_driver.cpp", 68, r"choose_b\((\d+), (\d+), config\) == (\d+)", "explicit b=17 wins"),
    ("partition_1000_50_ifc", "test_partition.cpp", 78, r"interface_count\(\) == (\d+)", "partition(1000,1000,50) interfaces"),
    ("partition_1000_50_int", "test_partition.cpp", 79, r"interior_count\(\) == (\d+)", "interiors"),
    ("partition_1000_50_lastw", "test_partition.cpp", 80, r"width == (\d+)", "last strip width"),
]


def main():
    out = {"source": "/root/reference/proj/tests (reference known-answer tests)", "values": {}}
    for key, fname, line, rx, desc in SPECS:
        path = os.path.join(REF, fname)
        lines = open(path).read().split("\n")
        text = lines[line - 1]
        m = re.search(rx, text)
        if not m:
            sys.exit(f"{fname}:{line}: pattern {rx!r} not found in {text!r}")
        vals = [float(g) for g in m.groups()]
        out["values"][key] = {"values": vals, "cite": f"proj/tests/{fname}:{line}", "what": desc}
    dst = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_known_answers.json")
    json.dump(out, open(dst, "w"), indent=1)
    print(f"wrote {dst} ({len(out['values'])} entries)")


if __name__ == "__main__":
    main()
