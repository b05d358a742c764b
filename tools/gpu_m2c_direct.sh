# moms2cums: copies + norm terms written in phase 1 (out-of-block pass) vs a second pass
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_direct.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_direct.log
for c in 2 3 1; do
timeout 300 python tools/kbench.py --config $c --steps 6 --label direct_c$c
CSB_M2C_DIRECT=0 timeout 300 python tools/kbench.py --config $c --steps 6 --label twopass_c$c
done
