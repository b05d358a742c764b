# A/B of an environment switch on kbench: bash tools/gpu_ab.sh VAR
for v in 0 1; do for c in ${CFGS:-1 2}; do env $1=$v python tools/kbench.py --config $c --steps 10 --label "$1=$v c$c"; done; done
