cat > /tmp/tipcheck.py <<'PY'
import os, sys, subprocess, numpy as np
sys.path.insert(0, os.getcwd())
def dump(out):
    import paper_1509_07919_b200 as S
    res = {}
    for i, (n, k, p, d) in enumerate([(4000, 20, 4, 1.0), (20000, 200, 5, 1.0), (12345, 64, 7, 0.3), (3001, 33, 3, 0.8), (9000, 150, 6, 0.1), (200000, 200, 50, 1.0)]):
        band, rhs = S.random_banded(n, k, d, 3 + i)
        s = S.Solver(p=p); s.setup(band, n, k)
        for t in range(min(p - 1, 3)):
            sp = s.spike(t)
            res[f"vb{i}_{t}"] = sp["vb"]; res[f"wt{i}_{t}"] = sp["wt"]; res[f"rb{i}_{t}"] = sp["rbar"]
        res[f"m{i}"] = s.apply_preconditioner(rhs)
        if i == 5: print("t_spk", s.report()["t_spk"])
        s.close()
    np.savez(out, **res)
if len(sys.argv) > 1: dump(sys.argv[1]); sys.exit()
subprocess.run([sys.executable, __file__, "/tmp/t_new.npz"], check=True)
env = dict(os.environ); env["SAP_TIPS_OLD"] = "1"
subprocess.run([sys.executable, __file__, "/tmp/t_old.npz"], check=True, env=env)
a, b = np.load("/tmp/t_new.npz"), np.load("/tmp/t_old.npz")
worst = 0.0
for key in a.files:
    d = float(np.max(np.abs(a[key] - b[key])) / max(np.max(np.abs(b[key])), 1e-300))
    worst = max(worst, d)
    if d > 1e-15: print(key, f"{d:.3e}")
print("worst normwise rel diff", worst)
PY
python /tmp/tipcheck.py
