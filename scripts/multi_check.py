"""Launch counts of the C4 forward per projection group: smlm_forward_multi (shared pre-shrink) vs
per-projection smlm_forward (diagnostic for SURVEY f1 on mixed batches)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2511_00101_b200 import smlm as S  # noqa: E402

dev = torch.device("cuda", 0)
wl = bench.Workload(4, synth.CONFIGS[4].rank, dev)
layer = wl.layers[0]
st = torch.cuda.current_stream()
for grp in bench.FWD_GROUPS:
    n0 = S.smlm_launch_count()
    bench.forward_groups(S, layer, wl.b, lambda p: wl.X[bench.GROUP_OF[p]], wl.Y, wl.V, st, [grp])
    torch.cuda.synchronize()
    print(grp, "launches", S.smlm_launch_count() - n0,
          "ws_multi", layer[grp]["ws"].numel() if len(grp) > 1 else None)
