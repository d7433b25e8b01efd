"""Device memory over one c1 forward pass (B ciphertexts): torch-allocated bytes
after setup, after each layer's pass and the peak, plus the C workspace size."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_07751_b200 import configs, inference as inf  # noqa: E402
from paper_2409_07751_b200.backend import BackendConfig, make_backend  # noqa: E402
from paper_2409_07751_b200.params import kan_params  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
cfgname = sys.argv[2] if len(sys.argv) > 2 else "c1"
_, model, X = configs.workload(cfgname)
X = np.resize(X, (B, X.shape[1]))
depth = inf.plan_model(model, inf.PipelineConfig()).total
p = kan_params(depth)
be = make_backend(BackendConfig(slot_count=p.slot_count, depth_budget=depth), params=p)
G = 1 << 30
print(f"after context+keys: {torch.cuda.memory_allocated() / G:.2f} GiB torch")
ct = inf.encrypt_input(X, model, be)
print(f"after encrypt: {torch.cuda.memory_allocated() / G:.2f} GiB; one ct {2 * (depth + 1) * B * p.n * 8 / G:.2f} GiB")
torch.cuda.reset_peak_memory_stats()
out, _ = inf.model_forward_he(model, ct, inf.PipelineConfig())
be.engine.sync()
print(f"after pass 1: {torch.cuda.memory_allocated() / G:.2f} GiB, peak {torch.cuda.max_memory_allocated() / G:.2f} GiB, "
      f"pt cache {be._pt_cache_bytes / G:.2f} GiB ({len(be._pt_cache)} entries)")
torch.cuda.reset_peak_memory_stats()
out, _ = inf.model_forward_he(model, ct, inf.PipelineConfig())
be.engine.sync()
print(f"after pass 2: {torch.cuda.memory_allocated() / G:.2f} GiB, peak {torch.cuda.max_memory_allocated() / G:.2f} GiB")
free, total = torch.cuda.mem_get_info()
print(f"device used {(total - free) / G:.2f} GiB of {total / G:.2f} (torch reserved {torch.cuda.memory_reserved() / G:.2f})")
