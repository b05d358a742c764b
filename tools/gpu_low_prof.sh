# mirror A/B (low kernel launched first, so the mirror scope holds no join
# wait) and one ncu --set full capture of the low-order kernel at cfg2
for c in 2; do
CSB_LOW_DEFER=0 timeout 300 python tools/kbench.py --config $c --steps 10 --label staged_nodefer_c$c
CSB_LOW_DEFER=0 CSB_MIRROR_SCATTER=1 timeout 300 python tools/kbench.py --config $c --steps 10 --label scatter_nodefer_c$c
done
timeout 900 bash tools/gpu_prof_k.sh 2 moment_lower_tma 1 low
