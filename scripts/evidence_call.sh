# Round-end evidence on one GPU: ncu captures (scripts/ncu_profile.sh -> gpurun_out/r02prof), the
# GPU suite, smoke(), and the bench line.
bash scripts/ncu_profile.sh gpurun_out/r02prof > gpurun_out/r02prof_ncu.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
