timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -12
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_cfg2.log | cut -c1-300
