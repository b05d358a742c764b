"""Controlled timing of the kernels of one window update (A/B experiments):
prime a BASELINE config, run warm-up + N device-resident steps with the
library's per-kernel event profiling, print per-tag averages (ms)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--label", default="")
    ap.add_argument("--p", type=int, default=0, help="override rows per step (experiments)")
    ap.add_argument("--resync", action="store_true", help="every step a full recompute (resync_every=1)")
    args = ap.parse_args()
    import torch

    from paper_1701_06446_b200 import capi
    from paper_1701_06446_b200.synth import CONFIGS, StreamGen

    cfg = CONFIGS[args.config]
    if args.p:
        import dataclasses
        cfg = dataclasses.replace(cfg, p=args.p)
    g = StreamGen(cfg)
    st = capi.Stream(cfg.n, cfg.d, cfg.T, cfg.p, cfg.b, g.window(), resync_every=1 if args.resync else 0)
    xs = [torch.from_numpy(g.batch(1 + k % cfg.steps)).cuda() for k in range(args.steps + 3)]
    for k in range(3):
        st.step_dev(xs[k].data_ptr(), cfg.p, cfg.n, report=True)
    torch.cuda.synchronize()
    capi.profile_enable(True)
    for tag in ("moment_top", "moment_tail", "mirror", "moment_low", "moms2cums", "norm_partials", "norms", "m2c_2", "m2c_3", "m2c_4", "m2c_5", "m2c_6", "step_update", "step_m2c", "step_report"):
        capi.profile_read(tag)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cs = torch.cuda.ExternalStream(st.cuda_stream())
    e0.record(cs)
    for k in range(args.steps):
        st.step_dev(xs[3 + k].data_ptr(), cfg.p, cfg.n, report=True)
    e1.record(cs)
    torch.cuda.synchronize()
    out = {"label": args.label, "config": cfg.name, "step_ms": e0.elapsed_time(e1) / args.steps}
    for tag in ("moment_top", "moment_tail", "mirror", "moment_low", "moms2cums", "norm_partials", "norms", "m2c_2", "m2c_3", "m2c_4", "m2c_5", "m2c_6", "step_update", "step_m2c", "step_report"):
        ms, n = capi.profile_read(tag)
        out[tag + "_ms"] = ms / max(1, n)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
