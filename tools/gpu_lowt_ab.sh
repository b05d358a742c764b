# A/B of the low-order TMA kernel's shared-memory budget (stages per CTA)
for c in 2 1; do
for kb in 200 100 64 48; do
CSB_LOW_DEFER=0 CSB_LOWT_SMEM=$kb timeout 300 python tools/kbench.py --config $c --steps 10 --label nodefer_smem${kb}_c$c
CSB_LOWT_SMEM=$kb timeout 300 python tools/kbench.py --config $c --steps 10 --label defer_smem${kb}_c$c
done
done
