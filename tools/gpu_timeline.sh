CSB_LIB_PATH=$PWD/paper_1701_06446_b200/lib/exp/libexp64.so python tools/prof_step.py --config 1 --steps 2 > gpurun_out/timeline.txt 2>&1
grep -c "^T" gpurun_out/timeline.txt
