"""One c1 forward pass over B ciphertexts (after a warm pass that builds keys
and plaintext caches) — for ncu launch lists of the real step mix."""
import argparse

import numpy as np
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_07751_b200 import configs, inference as inf  # noqa: E402
from paper_2409_07751_b200.backend import BackendConfig, make_backend  # noqa: E402
from paper_2409_07751_b200.params import kan_params  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--passes", type=int, default=2)
ap.add_argument("--config", default="c1")
ap.add_argument("--log-n", type=int, default=16)
args = ap.parse_args()
_, model, X = configs.workload(args.config, batch=args.batch)
X = X[:args.batch] if X.shape[0] >= args.batch else np.resize(X, (args.batch, X.shape[1]))
depth = inf.plan_model(model, inf.PipelineConfig()).total
p = kan_params(depth, log_n=args.log_n)
be = make_backend(BackendConfig(slot_count=p.slot_count, depth_budget=depth), params=p)
ct = inf.encrypt_input(X, model, be)
for _ in range(args.passes):
    out, _ = inf.model_forward_he(model, ct, inf.PipelineConfig())
be.engine.sync()
print("ok", be.engine.lib.hk_launch_count(be.engine.ctx))
