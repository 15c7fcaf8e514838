"""Device time-to-solution across the BASELINE configs that fit one GPU (1, 3's K and d sweeps, 5 at P=8..512),
band resident in HBM, CUDA events on the solver's stream. Prints a table (profiles/configs_<tag>.txt).

    python tools/bench_configs.py TAG [--quick]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1509_07919_b200 as S  # noqa: E402

PEAK = 37.05e12
HBM = 6452.8e9


def f_lu(m, k):
    kk = min(k, max(m - 1, 0))
    return (m - kk) * (2 * kk * kk + kk) + (kk - 1) * kk * (4 * kk + 1) / 6.0


def run(n, k, d, p, pre, reps=3):
    band_h, rhs_h = S.random_banded(n, k, d, 1)
    band = torch.from_numpy(band_h).cuda()
    rhs = torch.from_numpy(rhs_h).cuda()
    del band_h
    kind = S.PrecondKind.coupled if pre == "C" else S.PrecondKind.decoupled
    s = S.Solver(p=p, precond=kind)
    stream = torch.cuda.Stream()
    s.set_stream(stream)
    best = None
    with torch.cuda.stream(stream):
        for i in range(reps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            s.setup(band, n, k)
            x, st = s.solve(rhs)
            e1.record(stream)
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) * 1e-3
            r = s.report()
            if i > 0 and (best is None or t < best[0]):
                best = (t, r, st)
    s.close()
    t, r, st = best
    lay = S.make_partition_layout(n, p, k)
    flops = sum(f_lu(m, k) for m in lay.sizes) * (2 if pre == "C" else 1)
    band_bytes = 8.0 * n * (2 * k + 1)
    t_roof = max(flops / PEAK, (2 if pre == "C" else 1) * 2 * band_bytes / HBM)
    return {"t": t, "t_lu_kernel": r["t_factor_kernel"], "t_kry": r["t_kry"], "it": st.iterations,
            "res": st.final_relative_residual, "conv": st.converged, "flops": flops,
            "lu_tf": flops / r["t_factor_kernel"] / 1e12, "lu_frac_roof": t_roof / r["t_factor_kernel"]}


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "dev"
    quick = "--quick" in sys.argv
    rows = []
    cases = [("1", 10000, 10, 1.0, 4, "D"), ("1", 10000, 10, 1.0, 4, "C")]
    for k in ([10, 50, 200] if quick else [10, 20, 50, 100, 200, 500]):
        for pre in ("C", "D"):
            cases.append(("3 K-sweep", 200000, k, 1.0, 50, pre))
    for d in ([0.06, 1.2] if quick else [0.06, 0.1, 0.2, 0.5, 1.2]):
        cases.append(("3 d-sweep", 200000, 200, d, 50, "C"))
    for p in ([8, 512] if quick else [8, 64, 512]):
        cases.append(("5", 2000000, 128, 1.0, p, "C"))
    hdr = (f"{'cfg':10s} {'N':>8s} {'K':>4s} {'d':>5s} {'P':>4s} {'pre':>3s} {'t_solve ms':>10s} {'LU ms':>8s} "
           f"{'LU TF/s':>8s} {'LU/roof':>7s} {'Kry ms':>8s} {'iters':>6s} {'rel.res':>9s}")
    print(hdr, flush=True)
    out = [hdr]
    for cfg, n, k, d, p, pre in cases:
        t0 = time.time()
        try:
            r = run(n, k, d, p, pre)
            line = (f"{cfg:10s} {n:8d} {k:4d} {d:5.2f} {p:4d} {pre:>3s} {r['t'] * 1e3:10.3f} {r['t_lu_kernel'] * 1e3:8.3f} "
                    f"{r['lu_tf']:8.2f} {r['lu_frac_roof']:7.3f} {r['t_kry'] * 1e3:8.3f} {r['it']:6.2f} {r['res']:9.2e}"
                    + ("" if r["conv"] else "  NOT CONVERGED"))
        except Exception as e:  # report and continue
            line = f"{cfg:10s} {n:8d} {k:4d} {d:5.2f} {p:4d} {pre:>3s} ERROR {type(e).__name__}: {e}"
        print(line, f"  ({time.time() - t0:.0f}s)", flush=True)
        out.append(line)
        torch.cuda.empty_cache()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"configs_{tag}.txt"), "w") as f:
        f.write("device time-to-solution (setup + BiCGStab(2) to rel_tol 1e-10), band resident, best of 3, one B200\n"
                "LU/roof = max(F/37.05 TF/s, factor bytes/HBM) / LU kernel time\n" + "\n".join(out) + "\n")


if __name__ == "__main__":
    main()
