#!/bin/bash
# Same-box A/B of two library builds, interleaved, N rounds (default 3):
#   $A (default ab/libsmlm_prev.so) vs $B (default the in-tree paper_2511_00101_b200/libsmlm.so)
# on the headline step (bench.py value, fwd GEMM TF/s, SM clock) and, with GEMM=1, on
# scripts/gemm_micro.py (forward with LoRA TF/s per shape).
N=${1:-3}
A=${A:-ab/libsmlm_prev.so}
B=${B:-paper_2511_00101_b200/libsmlm.so}
for i in $(seq 1 $N); do
  for lib in $A $B; do
    SMLM_LIB_PATH=$PWD/$lib python bench.py --no-side --no-e2e --no-cpu-baseline --steps 6 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value']), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])"
    if [ "${GEMM:-0}" = "1" ]; then
      SMLM_LIB_PATH=$PWD/$lib python scripts/gemm_micro.py 2>/dev/null | \
        python -c "import json,sys; print('$lib', ' '.join('%d/%d:%.0f(cublas %.0f)' % (d['K'], d['N'], d['smlm_lora_tflops'], d['cublas_tflops']) for d in map(json.loads, sys.stdin)))"
    fi
  done
done
