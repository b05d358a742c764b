# ncu --set full of one order-6 moms2cums launch at cfg2
python tools/prof_step.py --config 2 --steps 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:moms2cums_v2<\(int\)6" -c 1 \
    -o gpurun_out/prof_m2c6_c2 python tools/prof_step.py --config 2 --steps 2 > gpurun_out/prof_ncu.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/prof_ncu.log
