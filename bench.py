#!/usr/bin/env python3
"""Benchmark of the B200 sliding-window cumulant update (arXiv 1701.06446).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Workload (default): BASELINE.json configs[2] (d=6, n=48, b=4, T=50000,
p=2000) -- BASELINE's metric names no config, so the largest config it does
not assign to sharding: the order-6 update.  --config 0..4 selects another
(cfg1 and cfg3 are the order-4 ones; cfg4 needs ~55 GB of HBM).  One step =
one window update of the reference's `step()` (stream.cpp:85-108):
exchange p rows, moments_update of M1..Md, moms2cums to C1..Cd, and the
window report (nu_3..nu_d, the config's stated gauge) read back to the host.

--gpus N (N > 1) without a torchrun environment re-launches itself under
torch.distributed.run with N ranks; every rank owns a block-prefix shard of
M_d / C_d and exchanges over NCCL (allgather M_{d-1}, allreduce of the norm
partials); value = window updates/s of the one sharded stream.

value  = window updates/s with the incoming rows already resident in HBM
         (device timed with CUDA events on the engine's stream; L2 flushed
         between steps, the flush outside the events).
e2e    = the same through the C ABI with HOST buffers (csb_stream_step on
         pinned rows): H2D of the rows and D2H of the report inside the
         timed region.
roofline = the order-d/d-1 moment computation: the DMMA kernel (moment_top,
         the wide column windows) plus, where the plan uses it, the CUDA-core
         kernel of the narrowest windows (moment_tail) -- algorithmic flops
         of orders d and d-1 per step / the two kernels' event-timed average
         durations per step, against the measured FP64 peak
         (profiles/fp64_peak.json; MEASURED_PEAKS.json has no FP64 entry).
cpu_baseline = the reference itself (oracle/_ref, compiled from
         /root/reference) on the host cores: one step's two library calls
         (moments_update + moms2cums, stream.cpp:85-108) at the config's
         full size on a zero-initialised state (their cost does not depend
         on the values), all host threads.

--impl reference: the reference CPU library on the same workload, all host
threads, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from math import comb

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1701_06446_b200.synth import CONFIGS, StreamGen  # noqa: E402

METRIC = "window updates/sec (order-d sliding cumulant update, FP64)"
UNIT = "window-updates/s"


def bell_partition_flops(s: int) -> int:
    # 1 + sum_sigma sigma * S(s, sigma) over sigma >= 2
    S = [[0] * (s + 1) for _ in range(s + 1)]
    S[0][0] = 1
    for i in range(1, s + 1):
        for j in range(1, i + 1):
            S[i][j] = S[i - 1][j - 1] + j * S[i - 1][j]
    return 1 + sum(sig * S[s][sig] for sig in range(2, s + 1))


def algorithmic_flops(cfg) -> dict:
    n, d, p = cfg.n, cfg.d, cfg.p
    canon = {s: comb(n + s - 1, s) for s in range(1, d + 1)}
    f_mom = 4 * p * sum(canon.values())
    f_m2c = sum(canon[s] * bell_partition_flops(s) for s in range(2, d + 1))
    f_top = 4 * p * (canon[d] + canon[d - 1])  # the fused order-d/d-1 kernel, per launch
    return {"F_mom": f_mom, "F_m2c": f_m2c, "F_alg": f_mom + f_m2c, "F_top_launch": f_top}


def fp64_peak() -> tuple[float, str]:
    path = os.path.join(ROOT, "profiles", "fp64_peak.json")
    try:
        with open(path) as fh:
            j = json.load(fh)
        v = max(j.get("dgemm_cublas_tflops", 0.0), j.get("dfma_tflops", 0.0), j.get("dmma_tflops", 0.0))
        if v > 0:
            return v, "measured on B200 (profiles/fp64_peak.json: max of cuBLAS DGEMM, DFMA, DMMA microbenchmarks)"
    except (OSError, ValueError):
        pass
    return 37.2, "nominal 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz (no FP64 entry in MEASURED_PEAKS.json)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]
        return False

    def summary(self) -> dict:
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline_sample(cfg, batch_in, batch_out) -> dict | None:
    """The reference library (oracle/_ref) on a bounded sample of the same
    workload: the two calls one step() makes (moments_update of M1..Md with
    p rows in / p rows out, then moms2cums; stream.cpp:85-108) at full size
    on a zero-initialised series -- prime skipped, its cost is T/p steps'
    worth of accumulation and outside every step."""
    try:
        from oracle.oracle import Oracle, ref_library_path
    except Exception:
        return None
    if ref_library_path() is None:
        return None
    cores = os.cpu_count() or 1
    ref = Oracle("ref", workers=cores)
    m = ref.alloc_series(cfg.n, cfg.d, cfg.b)
    t0 = time.perf_counter()
    ref.moments_update(m, cfg.T, batch_in, batch_out, cfg.b)
    t1 = time.perf_counter()
    ref.moms2cums(m, cfg.n, cfg.b, cfg.T)
    t2 = time.perf_counter()
    dt = t2 - t0
    return {"value": 1.0 / dt, "unit": UNIT, "cores": cores, "kind": "reference",
            "cpu": cpu_model(),
            "sample": f"{cfg.name}: one step of the reference library (oracle/_ref, "
                      f"{os.path.basename(ref.path)}, workers={cores}): moments_update {t1 - t0:.2f} s + "
                      f"moms2cums {t2 - t1:.2f} s on a zero-initialised state",
            "s_per_step": dt}


def bench_config(cfg) -> dict:
    """The workload, identical in both arms' lines."""
    return {"workload": cfg.name, "d": cfg.d, "n": cfg.n, "b": cfg.b, "T": cfg.T, "p": cfg.p,
            "l2": "GPU arm: 256 MB written between steps, outside the step events"}


def run_reference_arm(args, cfg) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    try:
        from oracle.oracle import Oracle, RefStream, ref_library_path
    except Exception as e:  # pragma: no cover
        print(json.dumps({"impl": "reference", "unavailable": f"oracle import failed: {e}"}))
        return
    if ref_library_path() is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (make -C oracle ref)"}))
        return
    cores = os.cpu_count() or 1
    gen = StreamGen(cfg)
    window = gen.window()
    total = args.warmup + args.steps
    batches = [gen.batch(1 + (k % cfg.steps)) for k in range(total)]
    ref = Oracle("ref", workers=cores)
    t0 = time.perf_counter()
    st = RefStream(ref, cfg.n, cfg.d, cfg.T, cfg.p, cfg.b, window, resync_every=0)
    t_prime = time.perf_counter() - t0
    for k in range(args.warmup):
        st.step(batches[k])
    t0 = time.perf_counter()
    for k in range(args.warmup, total):
        rep = st.step(batches[k])
    dt = time.perf_counter() - t0
    st.close()
    value = args.steps / dt
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": bench_config(cfg),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "cpu": cpu_model(),
                         "sample": f"prime ({t_prime:.1f} s) + {args.warmup} warm-up + {args.steps} timed "
                                   f"step() calls of the unmodified reference library "
                                   f"({os.path.basename(ref.path)}, workers={cores})"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "last_report_nu": [float(v) for v in rep[6:6 + cfg.d - 2]],
    }))


def relaunch_under_torchrun(args) -> None:
    """--gpus N outside torchrun: one rank per GPU on this node."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd, env=env))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    cfg = CONFIGS[args.config]

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
        return

    if args.impl == "reference":
        run_reference_arm(args, cfg)
        return

    import torch

    from paper_1701_06446_b200 import capi

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    capi.check(capi.lib().csb_set_device(local if world > 1 else 0))
    dev = torch.device("cuda", local if world > 1 else 0)

    # one shared stream: every rank sees the same rows and owns a block shard
    gen = StreamGen(cfg)
    window = gen.window()
    total = args.warmup + 3 * args.steps
    batches = [gen.batch(1 + (k % cfg.steps)) for k in range(total)]

    if world > 1:
        uid = [capi.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        capi.comm_init(world, rank, uid[0])
        capi.comm_selftest(1 << 16)  # fail loudly before timing if the NCCL exchange is broken
    st = capi.Stream(cfg.n, cfg.d, cfg.T, cfg.p, cfg.b, window, resync_every=0,
                     shard_index=rank, shard_count=world)
    # steps run eagerly here: the engine would capture a CUDA graph on the second visit of a (ring head, batch
    # address) key -- a one-off cost of a few ms per key that pays back over a long stream but would land inside
    # this short timed region (at cfg2 graphs change nothing: the step is 12 ms of kernels)
    st.use_graphs(False)
    cs = torch.cuda.ExternalStream(st.cuda_stream(), device=dev)
    xdev = [torch.from_numpy(b).to(dev) for b in batches]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2
    torch.cuda.synchronize()

    for k in range(args.warmup):
        st.step_dev(xdev[k].data_ptr(), cfg.p, cfg.n, report=True)
    torch.cuda.synchronize()

    # ---- value: inputs resident in HBM -------------------------------------
    # Two timed passes of K steps each, identical apart from profiling: the
    # first records per-kernel events (the roofline's top-kernel duration),
    # the second is unprofiled and gives `value` (per-scope event records add
    # host work that can leave the GPU idle between a step's launches).
    def timed_pass(first, profiled):
        if profiled:
            capi.profile_enable(True)
            capi.profile_read("moment_top")
            capi.profile_read("moment_tail")
        l0 = capi.launch_count()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        r = None
        for k in range(args.steps):
            flush.fill_(float(k))
            torch.cuda.synchronize()
            evs[k][0].record(cs)
            r = st.step_dev(xdev[first + k].data_ptr(), cfg.p, cfg.n, report=True)
            evs[k][1].record(cs)
        torch.cuda.synchronize()
        w = time.perf_counter() - w0
        nl = capi.launch_count() - l0
        tm, tn = (capi.profile_read("moment_top") if profiled else (0.0, 0))
        if profiled:
            tt, _ = capi.profile_read("moment_tail")
            tm += tt  # both kernels of the order-d/d-1 pair
        if profiled:
            capi.profile_enable(False)
        ms = [a.elapsed_time(b) for a, b in evs]
        return ms, w, nl, tm, tn, r

    _, _, _, top_ms, top_n, _ = timed_pass(args.warmup, True)
    with ClockSampler(dev.index) as clocks:
        step_ms, wall, launches, _, _, rep = timed_pass(args.warmup + args.steps, False)
    dev_s = sum(step_ms) * 1e-3
    if dist:
        t = torch.tensor([dev_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_s = float(t.item())
    value = args.steps / dev_s  # window updates of the one (sharded) stream

    # ---- e2e: through the C ABI with host (pinned) buffers -----------------
    pinned = [torch.from_numpy(b).pin_memory() for b in batches[args.warmup + 2 * args.steps:]]
    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    torch.cuda.synchronize()
    # the library's pipelined ingestion (csb_stream_upload / csb_stream_step_uploaded, what the C++ run() loop
    # uses): step k is queued, then batch k+1's host-to-device copy is started on the copy stream and runs under
    # it, then step k's report is read back; every batch is copied inside a timed interval (batch 0 inside step
    # 0's, serialized)
    for k in range(args.steps):
        flush.fill_(float(k))
        torch.cuda.synchronize()
        ev2[k][0].record(cs)
        if k == 0:
            st.upload(pinned[0].numpy())
        st.step_uploaded(report=False)       # queued; returns at once
        if k + 1 < args.steps:
            st.upload(pinned[k + 1].numpy())  # the next batch's copy, under this step
        rep2 = st.report()                    # waits for the step, reads the report back
        ev2[k][1].record(cs)
    torch.cuda.synchronize()
    e2e_s = sum(a.elapsed_time(b) for a, b in ev2) * 1e-3
    if dist:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = args.steps / e2e_s

    flops = algorithmic_flops(cfg)
    peak, peak_src = fp64_peak()
    top_avg_s = (top_ms / max(1, top_n)) * 1e-3
    achieved = flops["F_top_launch"] / top_avg_s / 1e12 if top_n else None
    traffic = None
    tr_src = None
    for tr_path in (os.path.join(ROOT, "profiles", "r02", "moment_top_traffic_cfg2.json"),
                    os.path.join(ROOT, "profiles", "moment_top_traffic.json")):
        try:
            tr = json.load(open(tr_path))
            if tr.get("workload") == cfg.name:
                traffic = tr.get("bytes_per_launch")
                tr_src = os.path.relpath(tr_path, ROOT)
                break
        except (OSError, ValueError):
            continue
    hbm_peak = None
    try:
        hbm_peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs")
    except (OSError, ValueError):
        hbm_peak = None
    if not hbm_peak:
        hbm_peak = 6650.0  # profiling recipe fallback

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(cfg, batches[0], window[:cfg.p])

    if rank == 0:
        ms_per_step = 1e3 * dev_s / args.steps
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(cfg),
            "method": {"parallelism": (f"block-prefix shards x{world} (NCCL allgather M_d-1, allreduce "
                                       "norm partials)") if world > 1 else "single",
                       "step": f"exchange + moments_update(M1..M{cfg.d}) + moms2cums(C1..C{cfg.d}) + "
                               f"report(nu3..nu{cfg.d})"},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "kernel": (f"orders {cfg.d} and {cfg.d - 1}: moment_top_dmma_kernel (FP64 DMMA) + "
                                    "moment_tail_kernel (FP64 FMA, narrowest column windows)"),
                         "flops_per_launch": flops["F_top_launch"], "avg_launch_ms": top_avg_s * 1e3,
                         "launches": top_n, "peak_source": peak_src,
                         "timed_in": "a profiled pass of the same K steps run just before the (unprofiled) value pass",
                         "note": "FP64 path: bound is the FP64 pipe (DFMA/DMMA), not bf16 tensor",
                         "hbm": ({"traffic_bytes": traffic, "achieved_gbs": traffic / top_avg_s / 1e9,
                                  "peak_gbs": hbm_peak, "frac": traffic / top_avg_s / 1e9 / hbm_peak,
                                  "source": f"ncu dram__bytes_read+write of one launch ({tr_src})"}
                                 if traffic and top_n else None)},
            "step_flops": {"F_alg": flops["F_alg"], "F_mom": flops["F_mom"], "F_m2c": flops["F_m2c"],
                           "alg_tflops_per_s": flops["F_alg"] / (dev_s / args.steps) / 1e12},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": cfg.p * cfg.n * 8,
                    "d2h_bytes_per_step": (cfg.d + 3 * cfg.n) * 8,
                    "api": "csb_stream_upload + csb_stream_step_uploaded with pinned host rows (batch k+1's copy "
                           "under step k, as the C++ run() loop does) + report read back every step"},
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "wall_s_timed_region": wall,
            "step_ms_stats": {"min": min(step_ms), "median": statistics.median(step_ms), "max": max(step_ms)},
            "last_report": {"window": rep["window"], "nu": {str(k): v for k, v in rep["nu"].items()}},
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    st.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
