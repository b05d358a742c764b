"""Small driver for ncu captures: prime a BASELINE config on cuda:0 and run a
few device-resident window updates (the bench step), then exit.

    python tools/prof_step.py [--config 1] [--steps 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    import torch

    from paper_1701_06446_b200 import capi
    from paper_1701_06446_b200.synth import CONFIGS, StreamGen

    cfg = CONFIGS[args.config]
    g = StreamGen(cfg)
    st = capi.Stream(cfg.n, cfg.d, cfg.T, cfg.p, cfg.b, g.window(), resync_every=0)
    xs = [torch.from_numpy(g.batch(k + 1)).cuda() for k in range(args.steps)]
    torch.cuda.synchronize()
    for k in range(args.steps):
        rep = st.step_dev(xs[k].data_ptr(), cfg.p, cfg.n, report=True)
    torch.cuda.synchronize()
    print("ok", rep["window"], rep["nu"])


if __name__ == "__main__":
    main()
