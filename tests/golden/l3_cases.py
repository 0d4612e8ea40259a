"""skew_tridiag_gemm fixture cases (shared by make_golden.py and the tests):
(p, q, k, tril, alpha, beta); inputs regenerated from Philox(1000 + i)."""
import numpy as np

L3_CASES = [(37, 5, 3, False, 1.0, 1.0), (200, 100, 64, False, -1.0, 1.0), (200, 100, 64, True, -1.0, 1.0),
            (260, 130, 130, True, 0.5, 2.0), (60, 180, 17, False, 1.0, 0.0), (50, 150, 40, True, -1.0, 1.0),
            (129, 129, 1, False, 2.0, -1.0), (50, 20, 1, True, 0.0, 3.0), (300, 140, 150, True, -1.0, 1.0)]


def l3_inputs(i, p, q, k):
    rng = np.random.Generator(np.random.Philox(1000 + i))
    a = np.asfortranarray(rng.standard_normal((p, k)))
    b = np.asfortranarray(rng.standard_normal((k, q)))
    tau = rng.standard_normal(max(k - 1, 0))
    c = np.asfortranarray(rng.standard_normal((p, q)))
    return a, b, tau, c
