# cfg2 (order 6) sweep of the DMMA kernel's plan/geometry switches
run() { env "$@" timeout 300 python tools/kbench.py --config 2 --steps 6 --label "$*" | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['label'], round(d['step_ms'],3), 'top', round(d['moment_top_ms'],3))"; }
run X=0
run CSB_ONES4=1
run CSB_ONES4=2
run CSB_ONES4=3
run CSB_HS=4
run CSB_HS=6
run CSB_R4_MAX=4
run CSB_R4_MAX=2
run CSB_TILE_ORDER_MIX=1
