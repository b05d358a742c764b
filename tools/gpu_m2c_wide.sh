# moms2cums with 1024-thread CTAs for big order-4 blocks (cfg3) vs 256
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_wide.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_wide.log
for c in 3 1; do
timeout 300 python tools/kbench.py --config $c --steps 6 --label wide_c$c
CSB_M2C_WIDE=0 timeout 300 python tools/kbench.py --config $c --steps 6 --label narrow_c$c
done
