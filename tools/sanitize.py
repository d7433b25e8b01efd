"""Small fused-path workload for compute-sanitizer (memcheck / racecheck /
synccheck): N = 2^16 (the fused cluster NTT kernels), L = 4, 2 ciphertexts —
encrypt, relinearised product, mul_lin / mul2, rotation, hoisted rotations,
rotate_sum, plaintext and constant products, one BSGS product, decrypt."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_07751_b200 import inference as inf  # noqa: E402
from paper_2409_07751_b200.backend import BackendConfig, HeBackend  # noqa: E402
from paper_2409_07751_b200.params import kan_params  # noqa: E402

p = kan_params(4)
be = HeBackend(BackendConfig(slot_count=p.slot_count, depth_budget=4), p, seed=1)
S = p.slot_count
rng = np.random.default_rng(0)
x, y = rng.uniform(-1, 1, (2, S)), rng.uniform(-1, 1, (2, S))
a, b = be.encrypt(x), be.encrypt(y)
r = [be.mul(a, b), be.mul_lin(a, b, a, 0.5), be.mul2(a, b, b, a), be.rotate(a, 3), be.mul(a, y[0]),
     be.mul(a, 0.25), be.rotate_sum([a, b], [0, 5])]
r += be.rotate_many(a, [1, 2, 7])
W = rng.normal(0, 0.1, (8, 16))
v = np.zeros((2, S))
v[:, :16] = x[:, :16]
r.append(inf.bsgs_matvec(W, be.encrypt(v), split=(4, 4)))
err = np.abs(be.decrypt(r[0]) - x * y).max()
print("ok", err)
