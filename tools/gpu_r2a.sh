# Round 2, first pass: full GPU suite (incl. the config-kernel parity tests
# and the gloo-backed sharded stream), a short cfg2 bench, and the
# reference's cfg2 prime/step cost on this host.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv,noheader
nproc; grep -m1 "model name" /proc/cpuinfo; free -g | head -2
timeout 1500 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; cat gpurun_out/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg2.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_cfg2.log
timeout 900 python - > gpurun_out/ref_cfg2.log 2>&1 <<'PY'
import time, os, sys
sys.path.insert(0, ".")
from oracle.oracle import Oracle, RefStream
from paper_1701_06446_b200.synth import CONFIGS, StreamGen
cfg = CONFIGS[2]; g = StreamGen(cfg); w = g.window(); b1 = g.batch(1); b2 = g.batch(2)
ref = Oracle("ref", workers=os.cpu_count())
t = time.perf_counter(); st = RefStream(ref, cfg.n, cfg.d, cfg.T, cfg.p, cfg.b, w, resync_every=0); print("prime", time.perf_counter() - t, flush=True)
for b in (b1, b2):
    t = time.perf_counter(); st.step(b); print("step", time.perf_counter() - t, flush=True)
PY
echo "ref rc=$?"; cat gpurun_out/ref_cfg2.log
