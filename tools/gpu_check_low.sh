# GPU suite + per-config kernel timing after a low-order kernel change
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_low.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_low.log
for c in 2 1 0; do timeout 300 python tools/kbench.py --config $c --steps 10 --label low_c$c; done
CSB_LOW_DEFER=0 timeout 300 python tools/kbench.py --config 2 --steps 10 --label nodefer_c2
