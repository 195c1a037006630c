import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import ges_inputs as gi
import test_parity_gpu as T
from gpu_helpers import settings_pair
"""Randomised parity (beyond the hypothesis property test): random scenes through the
GPU path and the oracle (run_case: S1 state, lists, ranges bit-exact; image with R18's
both branches; every visible particle's gradients).
Usage: python tools/fuzz_parity.py SEED N [MAXP MAXW MAXH]"""
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
maxp, maxw, maxh = (int(x) for x in (sys.argv[3:6] if len(sys.argv) > 5 else (300, 300, 200)))
fails = 0
for it in range(n):
    seed = int(rng.integers(0, 2**31 - 1))
    P = int(rng.integers(1, maxp)); W = int(rng.integers(8, maxw)); H = int(rng.integers(8, maxh))
    deg = int(rng.integers(0, 4)); mu = float(rng.uniform(-3.0, 0.0))
    sc = gi.random_small_scene(seed, P=P, W=W, H=H, sh_degree=deg, kappa_max=0.98, log_scale_mu=mu)
    rho = float(rng.choice([0.0, 0.1, 0.5])); kernel = int(rng.integers(0, 2))
    gs, osx = settings_pair(rho=rho, kernel=kernel, background=(0.1, 0.2, 0.3))
    try:
        T.run_case(sc.particles, sc.cameras[0], gs, osx, gi.upstream_grad(seed, 0, W, H), max_amb_frac=0.05,
                   label=f"fuzz {it}")
    except AssertionError as e:
        fails += 1
        print("FAIL", it, seed, P, W, H, deg, mu, rho, kernel, str(e)[:200])
print("fuzz done", n, "fails", fails)
