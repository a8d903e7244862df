python -m pytest tests -m gpu -q > gpurun_out/r2c_pytest_gpu.log 2>&1; tail -15 gpurun_out/r2c_pytest_gpu.log
python -m pytest tests -m "not gpu" -q > gpurun_out/r2c_pytest_cpu.log 2>&1; tail -2 gpurun_out/r2c_pytest_cpu.log
