"""Reference (oracle/_ref) SaP-C solve at config 2 with d=0.06: iterations / residual history; run with
SAP_REF_LIB=libsapref_fma.so for the FMA-contracted build of the same unmodified reference."""
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import oracle as O
n, k, d, p = 200000, 200, 0.06, 50
band, rhs = O.ref_random_banded(n, k, d, 1)
x, s = O.ref_solve_banded(n, k, band, rhs, p, 0)
print(os.environ.get("SAP_REF_LIB", "libsapref.so"), "SaP-C iterations", s["iterations"], "residual", s["final_relative_residual"],
      [f"{v:.2e}" for v in s["residual_history"][:10]])
