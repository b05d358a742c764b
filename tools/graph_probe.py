"""Step time of the host-buffer path with and without CUDA-graph replay
(csb_stream_use_graphs) at one BASELINE config.
    python tools/graph_probe.py [config=0]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1701_06446_b200 import capi
from paper_1701_06446_b200.synth import CONFIGS, StreamGen

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 0]
g = StreamGen(cfg)
heads = cfg.T // cfg.p
bs = [torch.from_numpy(g.batch(1 + k % cfg.steps)).pin_memory() for k in range(8)]
out = {"config": cfg.name, "ring_heads": heads}
for graphs in (False, True):
    st = capi.Stream(cfg.n, cfg.d, cfg.T, cfg.p, cfg.b, g.window(), resync_every=0)
    st.use_graphs(graphs)
    for k in range(2 * heads + 2):  # first visit eager, second captured
        st.step(bs[k % 8].numpy())
    n = 4 * heads
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(n):
        st.step(bs[k % 8].numpy())
    torch.cuda.synchronize()
    out["graphs" if graphs else "eager"] = {"ms_per_step": 1e3 * (time.perf_counter() - t0) / n,
                                            "replays": st.graph_replays()}
    st.close()
print(json.dumps(out))
