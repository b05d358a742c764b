# Round-2 evidence pass: full GPU suite, smoke, the default bench (cfg2), its
# launch list under ncu, and per-kernel times.
TAG=${1:-s3}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_cfg2_$TAG.json 2> gpurun_out/bench_cfg2_$TAG.err; echo "bench rc=$?"; cut -c1-700 gpurun_out/bench_cfg2_$TAG.json
timeout 300 python tools/kbench.py --config 2 --steps 20 --label $TAG > gpurun_out/kbench_cfg2_$TAG.jsonl 2>&1; tail -1 gpurun_out/kbench_cfg2_$TAG.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu rc=$?"
