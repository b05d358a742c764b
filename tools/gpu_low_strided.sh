# low-order kernel: strided element ownership (conflict-free staged-row reads) vs consecutive
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_strided.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_strided.log
for rep in 1 2; do
timeout 300 python tools/kbench.py --config 2 --steps 6 --label strided_c2
CSB_LOWT_STRIDED=0 timeout 300 python tools/kbench.py --config 2 --steps 6 --label consec_c2
CSB_LOW_DEFER=0 timeout 300 python tools/kbench.py --config 2 --steps 6 --label strided_nodefer_c2
CSB_LOW_DEFER=0 CSB_LOWT_STRIDED=0 timeout 300 python tools/kbench.py --config 2 --steps 6 --label consec_nodefer_c2
done
