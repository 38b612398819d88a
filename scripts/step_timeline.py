"""Kernel timeline of one C4 step via torch.profiler (CUPTI): busy time per kernel and the idle
gaps between consecutive device activities.  With PDL a kernel's interval starts at its early
launch (it waits in griddepcontrol.wait), so per-kernel busy times overlap and add up to more
than the span: use the gaps (device idle) here and the ncu launch list for shares."""
import json
import re
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

dev = torch.device("cuda", 0)
wl = bench.Workload(4, 0, dev)
st = torch.cuda.current_stream()
for i in range(3):
    wl.step(st)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(3):
        wl.step(st)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
t0, t1 = ev[0].time_range.start, ev[-1].time_range.end
busy = {}
gaps = []
prev_end = None
for e in ev:
    k = re.sub(r"^void ", "", e.name.replace("(anonymous namespace)::", "")).split("(")[0]
    k = re.sub(r"^.*::(?=[A-Za-z_]\w*(<|$))", "", k)[:60]   # the kernel's own name (+ template args)
    busy[k] = busy.get(k, 0) + (e.time_range.end - e.time_range.start)
    if prev_end is not None and e.time_range.start > prev_end:
        gaps.append(e.time_range.start - prev_end)
    prev_end = max(prev_end or 0, e.time_range.end)
span = t1 - t0
out = {"layers_per_step": bench.N_LAYERS, "span_us_per_step": span / 3, "busy_us_per_step": sum(busy.values()) / 3, "gap_us_per_step": sum(gaps) / 3,
       "n_gaps": len(gaps) // 3, "top": sorted(((k, round(v / 3, 1)) for k, v in busy.items()), key=lambda x: -x[1])[:14]}
print(json.dumps(out, indent=1))
