"""Time the LU kernel variants (env switches in lu.cu launch_band_lu_ws) on config 2: t_factor_kernel per variant."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        import paper_1509_07919_b200 as S
        n, k, p = 200000, 200, 50
        band, _ = S.random_banded(n, k, 1.0, 1)
        s = S.Solver(p=p, precond=S.PrecondKind.coupled)
        ts = []
        for _ in range(4):
            s.setup(band, n, k)
            ts.append(s.report()["t_factor_kernel"])
        print(f"{os.environ.get('VARIANT', 'default'):12s} t_factor_kernel ms: " + " ".join(f"{t * 1e3:.3f}" for t in ts))
        sys.exit(0)
    for v in ["default", "SAP_LU_SEQ", "SAP_LU_LA2"] + sys.argv[1:]:
        env = dict(os.environ)
        env["VARIANT"] = v
        if v != "default":
            env[v] = "1"
        subprocess.run([sys.executable, __file__, "child"], env=env)
