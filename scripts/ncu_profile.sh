#!/bin/bash
# Profile evidence for the SMLM kernels (run under gpurun on ONE GPU).
#   1. launch list of one bench step with per-launch device time (cold-cache, serialised:
#      compare SHARES, not absolutes)
#   2. DRAM bytes of every forward CTA-pair GEMM launch of one step (-> profiles/ncu_traffic.json)
#   3. ncu --set full of the forward GEMM (gate), the backward dX GEMM (gate), the token
#      contraction, the U pass and the forward pre-shrink
set -x
OUT=${1:-gpurun_out}
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-side"
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > /dev/null 2>&1
# smlm_gemm2_kernel launches per step: 7 forward (q,k,v,o,gate,up,down) then 7 backward
# (down,up,gate,o,v,k,q); the first step is the warm-up, so the timed step's forward is 14..20
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
     -k regex:smlm_gemm2_kernel -s 14 -c 7 --csv --log-file $OUT/fwd_traffic.csv $CMD > /dev/null 2>&1
$NCU --set full --clock-control none --import-source on -k regex:smlm_gemm2_kernel -s 18 -c 1 -o $OUT/prof_fwd_gate -f $CMD > /dev/null 2>&1
$NCU --set full --clock-control none --import-source on -k regex:smlm_gemm2_kernel -s 23 -c 1 -o $OUT/prof_bwd_gate -f $CMD > /dev/null 2>&1
$NCU --set full --clock-control none --import-source on -k regex:smlm_tok_kernel -s 9 -c 1 -o $OUT/prof_tok -f $CMD > /dev/null 2>&1
# smlm_u_kernel per step: 7 forward pre-shrinks (q,k,v,o,gate,up,down) then 7 backward U passes
# (down,up,gate,...); the timed step starts at launch 14 -> gate pre-shrink = 18, gate U = 23
$NCU --set full --clock-control none --import-source on -k regex:smlm_u_kernel -s 23 -c 1 -o $OUT/prof_u -f $CMD > /dev/null 2>&1
$NCU --set full --clock-control none --import-source on -k regex:smlm_u_kernel -s 18 -c 1 -o $OUT/prof_preshrink -f $CMD > /dev/null 2>&1
ls -la $OUT
# decode path (kernels_dec3.cu): one q projection call and one fused q/k/v call at C2 shapes
$NCU --set full --clock-control none --import-source on -k regex:smlm_dec3 -s 2 -c 1 -o $OUT/prof_dec3_q -f env PROJ=q N=3 python scripts/run_c2_once.py > /dev/null 2>&1
$NCU --set full --clock-control none --import-source on -k regex:smlm_dec3 -s 2 -c 1 -o $OUT/prof_dec3_qkv -f python scripts/dec_layer_phases.py > /dev/null 2>&1
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/dec_launches.csv python scripts/bench_configs.py --c2-only > /dev/null 2>&1
# AdamW step (kernels_opt.cu): duration + DRAM bytes of both passes at the 32-layer size
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:adamw -c 8 --csv --log-file $OUT/adamw_launches.csv python scripts/adamw_bench.py > /dev/null 2>&1
