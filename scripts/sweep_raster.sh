# Raster-group budgets of the CTA-pair GEMMs (measure build: SMLM_RASTER_MB forward X band,
# SMLM_RASTER_BWD_MB backward dY band): DRAM bytes of the 8 GEMM launches of one C4 layer and
# the headline step, interleaved on one box.
mkdir -p gpurun_out/sw
for mb in ${FWD_MBS:-16 24 32 48 64}; do
  SMLM_MEASURE_LIB=1 SMLM_RASTER_MB=$mb ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:smlm_gemm2 -s 8 -c 8 --csv --log-file gpurun_out/sw/traffic_$mb.csv python scripts/prof_step.py > /dev/null 2>&1
done
for mb in ${BWD_MBS:-}; do
  SMLM_MEASURE_LIB=1 SMLM_RASTER_BWD_MB=$mb ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:smlm_gemm2 -s 8 -c 8 --csv --log-file gpurun_out/sw/traffic_bwd_$mb.csv python scripts/prof_step.py > /dev/null 2>&1
done
for i in 1 2; do for mb in ${BENCH_BWD_MBS:-48}; do
  echo "BWD_MB=$mb $(SMLM_MEASURE_LIB=1 SMLM_RASTER_BWD_MB=$mb python bench.py --no-side --no-e2e --no-cpu-baseline --steps 8 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])")"
done; done
