timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_cfg2.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_cfg2.log
for c in 1 2 3; do timeout 300 python tools/kbench.py --config $c --steps 10 --label r2c; done
