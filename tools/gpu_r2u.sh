python -m pytest tests -m gpu -q -x > gpurun_out/r2u_pytest_gpu.log 2>&1; tail -3 gpurun_out/r2u_pytest_gpu.log
python tools/grid_perf.py > gpurun_out/r2u_grid_perf.jsonl 2> gpurun_out/r2u_grid_perf.err; tail -2 gpurun_out/r2u_grid_perf.err
