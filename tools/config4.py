"""BASELINE config 4 end to end at BASELINE scale: the 3-D convection-diffusion matrix at s = 80
(N = 512,000, nnz = 3,545,600), DB + CM reordering, drop-off with an explicit tolerance, SaP-C,
BiCGStab(2) to rel_tol 1e-10, the manufactured solution's 1% error gate (benchmark.hpp:47).

* host stage: the reference's db_reorder / cm_reorder (oracle/_ref, pinned to one core) -> T_DB, T_CM;
* device: paper_1509_07919_b200.sparse.solve_reordered -> T_Drop, T_Asmbl, T_LU, T_BC, T_SPK, T_LUrdcd,
  T_Kry (CUDA events), k_after, iterations (warm run: setup + solve twice, the second reported);
* CPU baseline: the reference's whole solve_sparse on the same matrix, tolerance and P (1 core).

    python tools/config4.py [--s 80] [--tols 0.3735,0.37] [--p 148] [--out profiles/config4_r02.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--s", type=int, default=80)
    ap.add_argument("--tols", default="0.3735,0.37")
    ap.add_argument("--p", type=int, default=148)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import oracle as O
    import paper_1509_07919_b200 as S
    from paper_1509_07919_b200.sparse import solve_reordered
    n, rp, ci, v = O.convection_diffusion_3d(a.s)
    xs = O.manufactured_solution(n)
    b = O.csr_matvec(n, rp, ci, v, xs)
    saved = os.sched_getaffinity(0)
    os.sched_setaffinity(0, {min(saved)})
    hs = O.ref_host_stage(n, rp, ci, v, b)
    os.sched_setaffinity(0, saved)
    out = {"workload": f"BASELINE config 4: 3-D 7-point upwind convection-diffusion s={a.s} (N={n}, "
                       f"nnz={int(rp[-1])}), DB+CM (reference host stage), drop-off, SaP-C P={a.p}, "
                       "BiCGStab(2) rel_tol 1e-10, b = A x* (manufactured parabola)",
           "host_stage": {"t_db": hs["t_db"], "t_cm": hs["t_cm"], "kind": "reference (oracle/_ref), 1 core"},
           "runs": []}
    for ti, tol in enumerate([float(t) for t in a.tols.split(",")]):
        x, st, rep = solve_reordered(hs["rp"], hs["ci"], hs["v"], hs["rhs"], hs["cm_perm"], hs["col_scale"], a.p,
                                     tol, precond=S.PrecondKind.coupled, repeat=2)
        err = float(np.linalg.norm(x - xs) / np.linalg.norm(xs))
        run = {"drop_tol": tol, "k_after": rep["k_after"], "partitions": rep["partitions"],
               "iterations": st.iterations, "converged": st.converged,
               "final_relative_residual": st.final_relative_residual, "relative_error_vs_xstar": err,
               "gpu": {q: rep[q] for q in ("t_drop", "t_asmbl", "t_lu", "t_factor_kernel", "t_bc", "t_spk",
                                           "t_lurdcd", "t_kry")},
               "gpu_device_total_s": sum(rep[q] for q in ("t_drop", "t_asmbl", "t_lu", "t_bc", "t_spk", "t_lurdcd",
                                                          "t_kry")),
               "gpu_wall_setup_solve_s": rep["wall_setup_solve"]}
        if not a.no_cpu and O.has_ref() and ti == 0:  # the CPU reference only at the first (narrowest-K) tolerance
            os.sched_setaffinity(0, {min(saved)})
            t0 = time.perf_counter()
            xr, so = O.ref_solve_sparse(n, rp, ci, v, b, a.p, 0, use_db=True, use_cm=True, drop_tol=tol)
            wall = time.perf_counter() - t0
            os.sched_setaffinity(0, saved)
            rr = so["report"]
            run["cpu_reference"] = {"wall_s": wall, "t_db": rr[0], "t_cm": rr[1], "t_drop": rr[2], "t_asmbl": rr[3],
                                    "t_bc": rr[4], "t_lu": rr[5], "t_spk": rr[6], "t_lurdcd": rr[7], "t_kry": rr[8],
                                    "k_after": so["k_after"], "iterations": so["iterations"],
                                    "converged": so["converged"], "cores": 1}
            run["parity"] = {"k_after_equal": so["k_after"] == rep["k_after"],
                             "iterations_diff": st.iterations - so["iterations"],
                             "x_rel_diff": float(np.linalg.norm(x - xr) / np.linalg.norm(xr))}
        out["runs"].append(run)
        print(json.dumps(run), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
