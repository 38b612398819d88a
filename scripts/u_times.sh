#!/bin/bash
# per-launch durations (ncu, serialised) of the U / pre-shrink kernels of one C4 layer step, for a library
SMLM_LIB_PATH=$PWD/${1:-paper_2511_00101_b200/libsmlm.so} /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:smlm_u_kernel --csv python scripts/prof_step.py 2>/dev/null | grep gpu__time | python3 -c "
import sys, csv
rows = list(csv.reader(sys.stdin))
t = [float(r[-1]) / 1000 for r in rows]
h = t[len(t) // 2:]
print(len(h), 'launches', round(sum(h), 1), 'us:', [round(x, 1) for x in h])"
