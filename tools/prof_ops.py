"""Profiling driver: one of each primitive at c1 shapes (N=2^16, level 36, B ciphertexts).

Run plain first, then under ncu (B200_PROFILING.md recipe).
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_07751_b200.backend import BackendConfig, make_backend  # noqa: E402
from paper_2409_07751_b200.params import kan_params  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--depth", type=int, default=36)
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
p = kan_params(args.depth)
be = make_backend(BackendConfig(slot_count=p.slot_count, depth_budget=args.depth), params=p)
x = np.random.default_rng(0).uniform(-1, 1, (args.batch, p.slot_count))
ct = be.encrypt(x)
be.ensure_rotation_keys([1])
eng = be.engine
buf = eng.alloc_u64((args.depth + 1) * args.batch * p.n)
buf.zero_()
for _ in range(args.reps):
    eng.call("hk_ntt_fwd", eng.addr(buf), 0, args.depth + 1, args.batch)
    eng.call("hk_ntt_inv", eng.addr(buf), 0, args.depth + 1, args.batch)
    be.mul(ct, ct)
    be.rotate(ct, 1)
    be.mul(ct, x[0])
    be.add(ct, ct)
eng.sync()
print("ok")
