"""Prints ||A||_2 (the fixed-seed power iteration of configs.device_power_norm2)
of the full-size cfg5 on the device, for configs.NORM2_FROZEN."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time  # noqa: E402

import paper_2503_22631_b200 as rk  # noqa: E402
from paper_2503_22631_b200 import configs  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 512
t0 = time.time()
A = rk.SparseMatrix.q1_hex(N, False, configs.COEF_SEED, False)
t1 = time.time()
lam = configs.device_power_norm2(A)
print(f"cfg5 N={N}: norm2={lam!r} (gen {t1 - t0:.1f} s, power {time.time() - t1:.1f} s)", flush=True)
