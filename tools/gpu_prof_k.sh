# ncu --set full of one launch of kernel regex $2 at config $1 (skip $3 launches)
CFG=${1:-1}; K=${2:-moment_top}; SKIP=${3:-1}; TAG=${4:-$K}
python tools/prof_step.py --config $CFG --steps 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 \
    -o gpurun_out/prof_${TAG}_c$CFG python tools/prof_step.py --config $CFG --steps 2 > gpurun_out/prof_ncu.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/prof_ncu.log
