# A/B of the low-order side kernel placement at cfg2 (order 6) and cfg1
for c in 2 1; do
timeout 300 python tools/kbench.py --config $c --steps 10 --label default_c$c
CSB_LOW_DEFER=0 timeout 300 python tools/kbench.py --config $c --steps 10 --label nodefer_c$c
CSB_LOW_KERNEL=side timeout 300 python tools/kbench.py --config $c --steps 10 --label side_c$c
CSB_LOW_KERNEL=side CSB_LOW_DEFER=0 timeout 300 python tools/kbench.py --config $c --steps 10 --label side_nodefer_c$c
done
