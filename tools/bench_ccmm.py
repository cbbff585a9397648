"""CCMM row of bench.py alone (tools helper): python tools/bench_ccmm.py -> one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2509_09424_b200 import Context  # noqa: E402

cfg = synth.CONFIGS["C2"]
ctx = Context(cfg["log_n"], cfg["L"], cfg["alpha"], cfg["dnum"])
print(json.dumps(bench.bench_ccmm(ctx, cfg, torch.cuda.current_stream())))
print("launches", ctx.launch_count())
