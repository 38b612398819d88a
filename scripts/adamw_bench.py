"""AdamW step (kernels_opt.cu) throughput against the HBM roofline: one JSON line per size
(1 and 32 layers of the C4 fine-tune adapters), with and without the clip pass."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import bench_configs as bc  # noqa: E402

for layers in (1, 32):
    for clip in (0.0, 1.0):
        print(json.dumps(bc.adamw_step(layers=layers, clip=clip)), flush=True)
