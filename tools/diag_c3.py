import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_07751_b200 import configs, inference as inf, model as mdl
from paper_2409_07751_b200.backend import BackendConfig, HeBackend
from paper_2409_07751_b200.engine import GpuEngine
from paper_2409_07751_b200.params import make_params
_, model, X = configs.workload("c3", batch=8)
cs = inf.PipelineConfig().comparator()
B = 8
for log_n in (9, 12, 14, 16):
    p = make_params(log_n, 54)
    be = HeBackend(BackendConfig(slot_count=p.slot_count, depth_budget=54), p, engine=GpuEngine(p))
    ct = inf.encrypt_input(X[:B], model, be)
    x = X[:B]
    for li, layer in enumerate(model.layers):
        ct = inf.layer_forward_he(layer, ct, inf.PipelineConfig())
        x = np.stack([mdl.layer_forward_plain(layer, r, "mirrored", cs, "lazy", schedule="cheb") for r in x])
        dec = be.decrypt(ct)[:, :layer.n_o]
        print(f"N=2^{log_n} layer {li}: max|he-twin| = {np.abs(dec - x).max():.3g}  per-sample {np.abs(dec - x).max(axis=1).round(8).tolist()}", flush=True)
