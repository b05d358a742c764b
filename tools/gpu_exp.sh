# timing experiments: kernel variants built with -DCSB_EXP=k under lib/exp/
for e in ${EXPS:-"" 1 2 3}; do
  if [ -n "$e" ]; then export CSB_LIB_PATH=$PWD/paper_1701_06446_b200/lib/exp/libexp$e.so; else unset CSB_LIB_PATH; fi
  for c in ${CFGS:-1 2}; do timeout 300 python tools/kbench.py --config $c --steps 10 --label "exp$e c$c"; done
done
