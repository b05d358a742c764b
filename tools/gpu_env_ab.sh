# A/B of environment settings on kbench: VARS="A=1 B=2" CFGS="1 2" bash tools/gpu_env_ab.sh
for c in ${CFGS:-1 2}; do
  timeout 300 python tools/kbench.py --config $c --steps 10 --label "base c$c"
  for v in $VARS; do timeout 300 env $v python tools/kbench.py --config $c --steps 10 --label "$v c$c"; done
done
