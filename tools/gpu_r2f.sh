timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_cfg2.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_cfg2.log | cut -c1-400
for c in 1 3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.log 2>&1; echo "bench cfg$c rc=$?"; tail -1 gpurun_out/bench_cfg$c.log | cut -c1-300; done
