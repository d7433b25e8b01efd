"""c5 [3072,128,10] encrypted at N = 2^17 (S = 65536: 33792 packed slots do not fit
2^15): decrypted outputs vs the reference's golden (tests/golden/c5.npz) and the
exact-arithmetic twin, with phase timings and device memory (diagnostic tool)."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_07751_b200 import configs, inference as inf, model as mdl  # noqa: E402
from paper_2409_07751_b200.backend import BackendConfig, make_backend  # noqa: E402
from paper_2409_07751_b200.params import kan_params  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=2)
ap.add_argument("--passes", type=int, default=1)
args = ap.parse_args()
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
gold = np.load(os.path.join(root, "tests", "golden", "c5.npz"))
t0 = time.perf_counter()
_, model, X = configs.workload("c5", batch=args.batch)
X = X[:args.batch]
depth = inf.plan_model(model, inf.PipelineConfig()).total
p = kan_params(depth, log_n=17)
be = make_backend(BackendConfig(slot_count=p.slot_count, depth_budget=depth), params=p)
print(f"setup {time.perf_counter() - t0:.1f}s depth {depth}", flush=True)
for i in range(args.passes):
    torch.cuda.synchronize()
    t = time.perf_counter()
    ct = inf.encrypt_input(X, model, be)
    out, stats = inf.model_forward_he(model, ct, inf.PipelineConfig())
    dec = be.decrypt(out)[:, :10]
    torch.cuda.synchronize()
    print(f"pass {i}: {time.perf_counter() - t:.1f}s, max mem {torch.cuda.max_memory_allocated() / 2**30:.1f} GiB",
          flush=True)
cs = inf.PipelineConfig().comparator()
twin = np.stack([mdl.model_forward_plain(model, x, "mirrored", cs, "lazy", schedule="cheb") for x in X])
n = min(args.batch, gold["mirrored"].shape[0])
res = {"err_vs_twin": float(np.abs(dec - twin).max()),
       "err_vs_reference_mirrored": float(np.abs(dec[:n] - gold["mirrored"][:n]).max()),
       "counts": stats.to_json()["total"],
       "reference_counts": json.loads(str(gold["counts"]))}
print(json.dumps(res))
