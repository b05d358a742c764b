# A/B of experiment libraries on kbench: LIBS="nopad exp3" CFGS="1 2" bash tools/gpu_libs_ab.sh
for c in ${CFGS:-1 2}; do
  timeout 300 python tools/kbench.py --config $c --steps 10 --label "base c$c"
  for l in $LIBS; do CSB_LIB_PATH=$PWD/paper_1701_06446_b200/lib/exp/lib$l.so timeout 300 python tools/kbench.py --config $c --steps 10 --label "$l c$c"; done
done
