"""End-to-end ingestion variants at one config (experiments)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1701_06446_b200 import capi
from paper_1701_06446_b200.synth import CONFIGS, StreamGen

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
g = StreamGen(cfg)
st = capi.Stream(cfg.n, cfg.d, cfg.T, cfg.p, cfg.b, g.window(), resync_every=0)
bs = [torch.from_numpy(g.batch(1 + k)).pin_memory() for k in range(24)]
dev = [b.cuda() for b in bs]
torch.cuda.synchronize()
for k in range(3):
    st.step(bs[k].numpy())

def timeit(name, fn, n=20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn(n)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / n
    print(f"{name:28s} {dt*1e3:8.3f} ms/step")

timeit("step_dev (report)", lambda n: [st.step_dev(dev[k].data_ptr(), cfg.p, cfg.n, report=True) for k in range(n)])
timeit("step host pinned", lambda n: [st.step(bs[k].numpy()) for k in range(n)])
def pipe(n):
    st.upload(bs[0].numpy())
    for k in range(n):
        if k + 1 < n:
            st.upload(bs[k + 1].numpy())
        st.step_uploaded()
timeit("upload pipelined", pipe)
def seq(n):
    for k in range(n):
        st.upload(bs[k].numpy())
        st.step_uploaded()
timeit("upload then step", seq)
timeit("step_dev no report", lambda n: [st.step_dev(dev[k].data_ptr(), cfg.p, cfg.n, report=False) for k in range(n)])
ts = []
st.upload(bs[0].numpy())
for k in range(12):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if k + 1 < 12:
        st.upload(bs[k + 1].numpy())
    t1 = time.perf_counter()
    st.step_uploaded()
    t2 = time.perf_counter()
    ts.append(((t1 - t0) * 1e3, (t2 - t1) * 1e3))
print("per-step (upload ms, step ms):", [(round(a, 3), round(b, 3)) for a, b in ts])
ts = []
torch.cuda.synchronize()
st.upload(bs[0].numpy())
for k in range(12):
    t0 = time.perf_counter()
    if k + 1 < 12:
        st.upload(bs[k + 1].numpy())
    t1 = time.perf_counter()
    st.step_uploaded()
    t2 = time.perf_counter()
    ts.append(((t1 - t0) * 1e3, (t2 - t1) * 1e3))
print("no-sync per-step (upload ms, step ms):", [(round(a, 3), round(b, 3)) for a, b in ts])
ts = []
torch.cuda.synchronize()
for k in range(12):
    t0 = time.perf_counter()
    st.step(bs[k].numpy())
    ts.append(round((time.perf_counter() - t0) * 1e3, 3))
print("no-sync step host:", ts)
