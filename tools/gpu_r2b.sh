for wb in tools/window_bench tools/window_bench_kc64 tools/window_bench_kc16 tools/window_bench_u4; do
timeout 300 $wb 6 48 4 2000 3 2 > gpurun_out/windows.log 2>&1
echo $wb
python3 -c "
import json
for ln in open('gpurun_out/windows.log'):
    if not ln.startswith('{'): print(ln.strip()); continue
    j = json.loads(ln); w = j['windows']
    print(j['d'], j['n'], 'dmma_all', w[0]['ms'], 'tail_tasks', j['tail_tasks'], 'tail_ms', j['tail_ms'], 'total', round(w[0]['ms'] + j['tail_ms'], 3), j['err'])
"
done
