#!/bin/bash
# Profile evidence for the SMLM kernels (run under gpurun on ONE GPU; round-2 launch order, see
# scripts/prof_step.py: 8 CTA-pair GEMM launches per one-layer step).
#   1. launch list (per-launch device time, cold-cache, serialised: compare SHARES) of the bench
#   2. DRAM bytes of the forward / backward CTA-pair GEMM launches of one layer (-> ncu_traffic.json)
#   3. ncu --set full of the merged q/k/v forward GEMM, the gate/up backward GEMM, the token
#      contraction, the fused q/k/v decode launch and the prefill attention kernel
set -x
OUT=${1:-gpurun_out}
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_layer.csv \
     python scripts/prof_step.py > /dev/null 2>&1
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
     -k regex:smlm_gemm2 -s 8 -c 8 --csv --log-file $OUT/gemm_traffic.csv python scripts/prof_step.py > /dev/null 2>&1
$NCU --set full --clock-control none --import-source on -k regex:smlm_gemm2 -s 8 -c 1 -o $OUT/prof_fwd_qkv -f python scripts/prof_step.py > /dev/null 2>&1
$NCU --set full --clock-control none --import-source on -k regex:smlm_gemm2 -s 13 -c 1 -o $OUT/prof_bwd_gateup -f python scripts/prof_step.py > /dev/null 2>&1
$NCU --set full --clock-control none --import-source on -k regex:smlm_tok_kernel -s 9 -c 1 -o $OUT/prof_tok -f python scripts/prof_step.py > /dev/null 2>&1
$NCU --set full --clock-control none --import-source on -k regex:smlm_dec3 -s 2 -c 1 -o $OUT/prof_dec3_qkv -f python scripts/dec_layer_phases.py > /dev/null 2>&1
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/dec_launches.csv python scripts/bench_configs.py --c2-only > /dev/null 2>&1
$NCU --set full --clock-control none --import-source on -k regex:attn_prefill -s 2 -c 1 -o $OUT/prof_attn_prefill -f python scripts/bench_configs.py --attention > /dev/null 2>&1
ls -la $OUT
