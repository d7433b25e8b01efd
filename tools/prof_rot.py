"""One level-36 rotation of B (argv[1], default 32) c1-shaped ciphertexts (after a warm-up rotation
that generates the key), bracketed by cudaProfilerStart/Stop so
`ncu --profile-from-start off` captures exactly the key switch's launches."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_07751_b200.backend import BackendConfig, make_backend  # noqa: E402
from paper_2409_07751_b200.params import kan_params  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
p = kan_params(36)
be = make_backend(BackendConfig(slot_count=p.slot_count, depth_budget=36), params=p)
ct = be.encrypt(np.zeros((B, p.slot_count)))
be.rotate(ct, 1)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
be.rotate(ct, 1)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
