#!/bin/bash
# Profile evidence for the SMLM kernels (run under gpurun on ONE GPU).
#   1. launch list with per-launch device time (cold-cache, serialised: compare SHARES)
#   2. ncu --set full of the forward tcgen05 GEMM (gate projection), the backward GEMM
#      (gate) and the token-contraction dA/dB kernel
set -x
OUT=${1:-gpurun_out}
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$NCU --metrics gpu__time_duration.sum --clock-control none -k regex:smlm --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches_bench.json 2>&1
# launch order per step: fwd q,k,v,o,gate,up,down (index 4 = gate), then bwd down,up,gate,...
$NCU --set full --clock-control none --import-source on -k regex:smlm_gemm_kernel -s 4 -c 1 -o $OUT/prof_fwd_gate -f $CMD > /dev/null 2>&1
$NCU --set full --clock-control none --import-source on -k regex:smlm_gemm_kernel -s 9 -c 1 -o $OUT/prof_bwd_gate -f $CMD > /dev/null 2>&1
$NCU --set full --clock-control none --import-source on -k regex:smlm_tok_kernel -s 2 -c 1 -o $OUT/prof_tok -f $CMD > /dev/null 2>&1
$NCU --set full --clock-control none --import-source on -k regex:shrink_short -s 4 -c 1 -o $OUT/prof_shrink -f $CMD > /dev/null 2>&1
ls -la $OUT
