#!/bin/bash
# Same-box A/B of two library builds on the headline step: ab/libsmlm_prev.so vs the current
# paper_2511_00101_b200/libsmlm.so, interleaved, N pairs (default 3).  Prints value / fwd GEMM TF/s.
N=${1:-3}
for i in $(seq 1 $N); do
  for lib in ab/libsmlm_prev.so paper_2511_00101_b200/libsmlm.so; do
    SMLM_LIB_PATH=$PWD/$lib python bench.py --no-side --no-e2e --no-cpu-baseline --steps 6 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value']), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])"
  done
done
