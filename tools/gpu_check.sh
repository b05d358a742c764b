# parity tests + per-kernel timing of the BASELINE configs (used between kernel changes)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
rm -f gpurun_out/kbench.log
for c in ${CFGS:-0 1 2 3}; do timeout 300 python tools/kbench.py --config $c --steps 10 --label c$c >> gpurun_out/kbench.log 2>&1; done; cat gpurun_out/kbench.log
