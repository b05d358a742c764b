# cfg4 (order 6, n=96) on one B200 + cfg3; per-kernel split via kbench
timeout 1200 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.log 2>&1; echo "cfg4 rc=$?"; tail -1 gpurun_out/bench_cfg4.log | cut -c1-600
timeout 900 python tools/kbench.py --config 4 --steps 3 --label r2 > gpurun_out/kbench_cfg4.log 2>&1; tail -1 gpurun_out/kbench_cfg4.log
timeout 900 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3.log 2>&1; echo "cfg3 rc=$?"; tail -1 gpurun_out/bench_cfg3.log | cut -c1-300
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
