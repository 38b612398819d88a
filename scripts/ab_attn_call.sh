# attention A/B call: parity tests of the attention branch, same-box A/B (scripts/ab_attn.sh),
# measure-build phase counters of the two-tile prefill kernel
timeout 300 python -m pytest tests/test_gpu_attention.py -q -x > gpurun_out/attn_tests.txt 2>&1; tail -2 gpurun_out/attn_tests.txt
bash scripts/ab_attn.sh > gpurun_out/ab_attn.txt 2>&1; cat gpurun_out/ab_attn.txt
SMLM_MEASURE_LIB=1 SMLM_ATTN_DEBUG=1 timeout 300 python scripts/bench_configs.py --attention 2>&1 | grep "cta 0 \|cta 64 " | head -4
