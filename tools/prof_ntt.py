"""Profiling driver (no bench): forward + inverse NTT over [limbs][batch][N=2^16]
of uniform random residues, or one relinearised product (`mul`) / rotation
(`rot`) at level limbs-1 over `batch` ciphertexts.

  python tools/prof_ntt.py [ntt|mul|rot] [limbs] [batch]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_07751_b200.params import kan_params  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "ntt"
limbs = int(sys.argv[2]) if len(sys.argv) > 2 else 37
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 128
p = kan_params(limbs - 1)
if mode == "ntt":
    import torch
    from paper_2409_07751_b200.engine import GpuEngine
    eng = GpuEngine(p)
    buf = eng.alloc_u64(limbs * batch * p.n).view(limbs, batch * p.n)
    for i in range(limbs):
        buf[i].random_(0, int(p.q[i]))
    for _ in range(2):
        eng.call("hk_ntt_fwd", eng.addr(buf), 0, limbs, batch)
        eng.call("hk_ntt_inv", eng.addr(buf), 0, limbs, batch)
    eng.sync()
else:
    from paper_2409_07751_b200.backend import BackendConfig, HeBackend
    be = HeBackend(BackendConfig(slot_count=p.slot_count, depth_budget=limbs - 1), p, seed=1)
    x = np.random.default_rng(0).uniform(-1, 1, (batch, p.slot_count))
    a = be.encrypt(x)
    for _ in range(2):
        r = be.mul(a, a) if mode == "mul" else be.rotate(a, 3)
    be.engine.sync()
print("ok")
