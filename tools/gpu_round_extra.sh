bash tools/gpu_round.sh
CSB_HS=8 timeout 300 python tools/kbench.py --config 1 --steps 10 --label c1_hs8
