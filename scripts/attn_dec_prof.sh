# ncu launch list (time, DRAM bytes) of the attention branch's kernels on the C4 batch
# (bench_configs.attention_step with one timed iteration: 4 prefill calls, then 4 decode calls)
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:attn_ --csv --log-file gpurun_out/attn_launches.csv \
  python -c "import sys; sys.path.insert(0, 'scripts'); sys.path.insert(0, '.'); import bench_configs as b; print(b.attention_step(iters=1))" > gpurun_out/attn_launches.log 2>&1
