# ncu --set full of one update launch of the top kernel (cfg given as $1)
CFG=${1:-1}
python tools/prof_step.py --config $CFG --steps 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:moment_top -s 1 -c 1 \
    -o gpurun_out/prof_top_c$CFG python tools/prof_step.py --config $CFG --steps 2 > gpurun_out/prof_ncu.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/prof_ncu.log
