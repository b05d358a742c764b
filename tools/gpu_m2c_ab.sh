# A/B: moms2cums register cap for orders <= 4 (bench + kbench, cfg1/cfg0/cfg3)
timeout 600 python -m pytest tests/test_gpu_wide.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_m2c.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_m2c.log
for rep in 1 2; do
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_m2c.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bench_m2c.log').read().strip().splitlines()[-1]);print('bench', d['value'], d['e2e']['value'], d['roofline']['frac'])"
done
for c in 1 0 3; do timeout 300 python tools/kbench.py --config $c --steps 10 --label m2c4_c$c; done
