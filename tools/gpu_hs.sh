for hs in 4 6 8; do CSB_HS=$hs python tools/kbench.py --config 1 --steps 10 --label "hs$hs"; done
