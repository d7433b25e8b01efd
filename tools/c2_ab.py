"""c2 primitive timings only (for same-box A/B of library builds)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

out = bench.c2_microbench(0)
print(json.dumps({k: v["ms"] for k, v in out.items() if isinstance(v, dict) and "ms" in v}))
