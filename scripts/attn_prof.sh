set -x
NCU=ncu
mkdir -p gpurun_out/attn
timeout 300 python scripts/bench_configs.py --attention > gpurun_out/attn/att.json 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:attn_prefill -s 2 -c 1 -o gpurun_out/attn/prof_attn_prefill2 -f python scripts/bench_configs.py --attention > gpurun_out/attn/ncu.log 2>&1
ls -la gpurun_out/attn
