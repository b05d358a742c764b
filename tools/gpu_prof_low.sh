# ncu --set full of one low-order (orders 1..4) kernel launch at cfg2
python tools/prof_step.py --config 2 --steps 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:moment_lower_tma" -c 1 \
    -o gpurun_out/prof_low4_c2 python tools/prof_step.py --config 2 --steps 2 > gpurun_out/prof_ncu.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/prof_ncu.log
