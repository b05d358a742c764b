# cfg2: chunk of 10 k4 steps (40 rows, 4 stages) vs the default 8 (32 rows, 7 stages)
timeout 300 python tools/kbench.py --config 2 --steps 6 --label hs8
CSB_HS=10 timeout 300 python tools/kbench.py --config 2 --steps 6 --label hs10
CSB_HS=10 CSB_TILE_ORDER_MIX=1 timeout 300 python tools/kbench.py --config 2 --steps 6 --label hs10mix
CSB_HS=10 timeout 600 python -m pytest tests/test_gpu_wide.py -x -q -k n40 > gpurun_out/pytest_hs10.log 2>&1; echo "pytest hs10 rc=$?"; tail -1 gpurun_out/pytest_hs10.log
