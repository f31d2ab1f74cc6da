"""Isolated batched zgemm throughput on the product library (prof stats)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1410_5003_b200.qpscat import Solver
s = Solver()
rng = np.random.default_rng(0)
for (M, N, K) in [(600, 600, 600), (1024, 1024, 1024), (600, 600, 80), (568, 600, 32), (64, 600, 64)]:
    A = rng.standard_normal((M, K)) + 1j * rng.standard_normal((M, K))
    B = rng.standard_normal((K, N)) + 1j * rng.standard_normal((K, N))
    s.debug_zgemm(A, B)
    s.prof_reset(); s.prof_enable(True)
    for _ in range(5):
        s.debug_zgemm(A, B)
    s.prof_enable(False)
    st = s.prof_stats()
    for k, v in st.items():
        if k.startswith("zgemm"):
            print(M, N, K, k, f"{v['flops'] / v['ms'] / 1e9:.2f} TF/s single GEMM ({v['ms'] / v['launches']:.3f} ms)")
