"""NTT-only profiling driver (no keygen): fwd + inv over [limbs][batch][N=2^16]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_07751_b200.engine import GpuEngine  # noqa: E402
from paper_2409_07751_b200.params import kan_params  # noqa: E402

limbs, batch = int(sys.argv[1]) if len(sys.argv) > 1 else 37, int(sys.argv[2]) if len(sys.argv) > 2 else 32
p = kan_params(limbs - 1)
eng = GpuEngine(p)
buf = eng.alloc_u64(limbs * batch * p.n)
buf.zero_()
for _ in range(2):
    eng.call("hk_ntt_fwd", eng.addr(buf), 0, limbs, batch)
    eng.call("hk_ntt_inv", eng.addr(buf), 0, limbs, batch)
eng.sync()
print("ok")
