"""Preconditioner-apply time (config 2, device band) of one or two builds of libsap_gpu.so:
    python tools/apply_time.py [LIB ...]     (SAP_GPU_LIB selects the build in a subprocess)"""
import os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys; sys.path.insert(0, %r)
import torch, paper_1509_07919_b200 as S
n, k, p = 200000, 200, 50
band, rhs = S.random_banded(n, k, 1.0, 1)
db = torch.from_numpy(band).cuda(); x = torch.from_numpy(rhs).cuda(); y = torch.empty_like(x)
for kind, name in ((1, "SaP-D (1 block solve)"), (0, "SaP-C (2 block solves + interfaces)")):
    with S.Solver(p=p, precond=kind) as s:
        s.setup(db, n, k)
        for _ in range(3): s.apply_preconditioner(x, y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): s.apply_preconditioner(x, y)
        e1.record(); torch.cuda.synchronize()
        print(f"  {name}: {e0.elapsed_time(e1) * 1e3 / 20:.1f} us per apply", flush=True)
''' % ROOT
libs = sys.argv[1:] or [os.path.join(ROOT, "paper_1509_07919_b200", "libsap_gpu.so")]
for lib in libs:
    print(lib, flush=True)
    subprocess.run([sys.executable, "-c", CODE], env=dict(os.environ, SAP_GPU_LIB=os.path.abspath(lib)), check=True)
