"""GPU busy/idle split of one c1 forward pass (torch.profiler / CUPTI kernel
records): union of kernel intervals vs the pass's device span. Tells whether
launch gaps and tails (not kernel speed) cost time."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_07751_b200 import configs, inference as inf  # noqa: E402
from paper_2409_07751_b200.backend import BackendConfig, make_backend  # noqa: E402
from paper_2409_07751_b200.params import kan_params  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--config", default="c1")
args = ap.parse_args()
_, model, X = configs.workload(args.config, batch=args.batch)
X = X[:args.batch] if X.shape[0] >= args.batch else np.resize(X, (args.batch, X.shape[1]))
depth = inf.plan_model(model, inf.PipelineConfig()).total
p = kan_params(depth)
be = make_backend(BackendConfig(slot_count=p.slot_count, depth_budget=depth), params=p)
ct = inf.encrypt_input(X, model, be)
inf.model_forward_he(model, ct, inf.PipelineConfig())  # warm: keys, caches
be.engine.sync()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    inf.model_forward_he(model, ct, inf.PipelineConfig())
    be.engine.sync()
iv = []
names = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0:
        iv.append((e.time_range.start, e.time_range.end))
        names[e.name[:40]] = names.get(e.name[:40], 0) + 1
iv.sort()
busy, cur_s, cur_e, gaps = 0.0, None, None, []
for s, e in iv:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
            gaps.append(s - cur_e)
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
span = iv[-1][1] - iv[0][0]
gaps = np.array(gaps)
print(f"kernels {len(iv)}  span {span / 1e3:.1f} ms  busy {busy / 1e3:.1f} ms  idle {100 * (1 - busy / span):.1f}%")
print(f"gaps: n={len(gaps)} mean {gaps.mean():.2f} us  p50 {np.median(gaps):.2f}  p99 {np.percentile(gaps, 99):.1f}  "
      f"sum>20us {gaps[gaps > 20].sum() / 1e3:.1f} ms")
