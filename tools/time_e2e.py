"""Per-piece timing of the e2e path (encrypt_input / forward / decrypt) for one
c1 chunk, host-synchronised wall clock (diagnostic, not a bench number)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_07751_b200 import configs, inference as inf  # noqa: E402
from paper_2409_07751_b200.backend import BackendConfig, make_backend  # noqa: E402
from paper_2409_07751_b200.params import kan_params  # noqa: E402

_, model, X = configs.workload("c1", batch=32)
p = kan_params(36)
be = make_backend(BackendConfig(slot_count=p.slot_count, depth_budget=36), params=p)
pc = inf.PipelineConfig()
ct = inf.encrypt_input(X, model, be)
o, _ = inf.model_forward_he(model, ct, pc)
be.decrypt(o)


def t(f):
    torch.cuda.synchronize()
    a = time.perf_counter()
    r = f()
    torch.cuda.synchronize()
    return r, (time.perf_counter() - a) * 1e3


for _ in range(2):
    ct, te = t(lambda: inf.encrypt_input(X, model, be))
    o, tf = t(lambda: inf.model_forward_he(model, ct, pc)[0])
    _, td = t(lambda: be.decrypt(o))
    _, tf2 = t(lambda: inf.model_forward_he(model, ct, pc)[0])
    ms = torch.cuda.memory_stats()
    print("retries", ms.get("num_alloc_retries"), "segments", ms.get("segment.all.current"),
          "reserved GB", round(ms.get("reserved_bytes.all.current", 0) / 2**30, 1))
    print(f"encrypt {te:.1f} ms  forward {tf:.1f} ms  decrypt {td:.1f} ms  forward-again {tf2:.1f} ms")
