"""W1 matrix timing (§8(f)2): 500 agents x 2048 samples each (C3-like
agent count), device kernel vs the C restatement on one host core."""
import sys, time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import paper_2508_06948_b200 as kx
import oracle_ffi as O
rng = np.random.default_rng(3)
A, S = 500, 2048
sets = [np.sort(rng.gamma(2.0, 3.0 + (a % 17), S)) for a in range(A)]
kx.w1_matrix(sets[:4])  # warm-up
t0 = time.perf_counter(); m = kx.w1_matrix(sets); t1 = time.perf_counter()
print(f"device w1_matrix {A} agents x {S} samples: {1e3 * (t1 - t0):.1f} ms (incl. H2D/D2H)")
# CPU restatement on a sample of pairs, extrapolated to all pairs
pairs = A * (A + 1) // 2
idx = rng.integers(0, A, (300, 2))
t0 = time.perf_counter()
for i, j in idx:
    w = O.wasserstein(sets[i], sets[j])
    assert w == m[i, j]
t1 = time.perf_counter()
print(f"cpu restatement: {1e3 * (t1 - t0) / len(idx):.3f} ms/pair -> {(t1 - t0) / len(idx) * pairs:.1f} s for {pairs} pairs (1 core); sampled pairs bit-equal")
