CSB_LIB_PATH=$PWD/paper_1701_06446_b200/lib/exp/libexp${TL:-128}.so python tools/prof_step.py --config 1 --steps 1 > gpurun_out/timeline2.txt 2>&1
