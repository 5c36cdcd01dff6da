"""Stress the multilevel solver's dual certificate over many seeds."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MUX_SSP_CHECK", "1")
from paper_2303_13803_b200 import default_table
from paper_2303_13803_b200.scheduler import round_arrays
from paper_2303_13803_b200.synth import make_cluster
t = default_table()
n = int(os.environ.get("N", "2000")); q = int(os.environ.get("Q", "30")); R = int(os.environ.get("R", "60"))
bad = 0
import time
S0 = int(os.environ.get("S0", "0"))
for seed in range(S0, S0 + R):
    cl = make_cluster(n, n, seed=seed)
    t0 = time.time()
    try:
        round_arrays(t, cl.x, cl.share, cl.y, qbits=q)
    except Exception as e:
        bad += 1
        print("seed", seed, e, flush=True)
    if os.environ.get("TRACE"):
        print(f"seed {seed}: {1e3 * (time.time() - t0):.1f} ms", flush=True)
print(f"N={n} q={q} serial={os.environ.get('MUX_SSP_SERIAL','0')}: {bad}/{R} failures", flush=True)
