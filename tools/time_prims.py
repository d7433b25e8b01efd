"""CUDA-event timings of engine primitives at c1 shapes (N=2^16)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_07751_b200.backend import BackendConfig, make_backend  # noqa: E402
from paper_2409_07751_b200.params import kan_params  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--level", type=int, default=36)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
p = kan_params(36)
be = make_backend(BackendConfig(slot_count=p.slot_count, depth_budget=36), params=p)
eng = be.engine
B, nl, N = args.batch, args.level + 1, p.n
x = np.random.default_rng(0).uniform(-1, 1, (B, p.slot_count))
ct = be.encrypt(x, level=args.level)
ct2 = be.encrypt(-x, level=args.level)
be.ensure_rotation_keys([1])
buf = eng.alloc_u64(nl * B * N)
buf.zero_()


def timeit(name, fn, algbytes):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.reps
    print(f"{name:18s} {ms:8.3f} ms  {algbytes / ms / 1e6:8.1f} GB/s algorithmic")


limb = B * N * 8
timeit("ntt_fwd", lambda: eng.call("hk_ntt_fwd", eng.addr(buf), 0, nl, B), 2 * nl * limb)
timeit("ntt_inv", lambda: eng.call("hk_ntt_inv", eng.addr(buf), 0, nl, B), 2 * nl * limb)
timeit("add", lambda: be.add(ct, ct2), 6 * nl * limb)
timeit("mul_plain", lambda: be.mul(ct, x[0]), 4 * nl * limb)
timeit("mul_ct(relin)", lambda: be.mul(ct, ct), 6 * nl * limb)
timeit("rotate", lambda: be.rotate(ct, 1), 4 * nl * limb)
rbuf = eng.alloc_u64(2 * nl * B * N)
timeit("rescale-only", lambda: eng.call("hk_rescale", eng.addr(ct.data), ct.level, eng.addr(rbuf), B), 4 * nl * limb)
torch.cuda.synchronize()
print("ok")
