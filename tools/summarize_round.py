"""Copy the round evidence from gpurun_out/ (tools/gpu_round.sh) into
profiles/: the bench line, per-config kernel timings, the ncu launch list of
the bench command (per-kernel shares) and the ncu --set full summary of the
top kernel, plus profiles/moment_top_traffic.json (bench.py's `traffic`).

    python tools/summarize_round.py TAG      # e.g. v12 -> profiles/r01/*_v12.*
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def launches(path):
    rows = list(csv.reader(line for line in open(path) if not line.startswith("==")))
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("(anonymous namespace)::", "")
        t = float(r[vi].replace(",", ""))
        unit = r[h.index("Metric Unit")] if "Metric Unit" in h else "ns"
        us = t / 1000.0 if unit in ("nsecond", "ns") else t if unit in ("usecond", "us") else t * 1000.0
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    ks = [{"kernel": k, "launches": v[0], "total_us": round(v[1], 1), "avg_us": round(v[1] / v[0], 2),
           "share": round(v[1] / tot, 4)} for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])]
    return ks


def ncu_summary(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, v = rows[0], rows[2]
    d = dict(zip(h, v))

    def f(k):
        return float(d[k].replace(",", "")) if k in d and d[k] else None

    mb = 1e6  # ncu reports dram bytes in Mbyte here
    rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
    return {
        "kernel": d.get("Kernel Name", "").replace("(anonymous namespace)::", ""),
        "workload": "cfg1_d4_n96_b8_T20000_p1000",
        "source": "ncu --set full --clock-control none --import-source on, one update launch (tools/gpu_prof_k.sh)",
        "duration_us_under_ncu": f("gpu__time_duration.sum"),
        "dram_read_bytes": rd * mb,
        "dram_write_bytes": wr * mb,
        "bytes_per_launch": (rd + wr) * mb,
        "dmma_subpipe_active_pct": f("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
        "dmma_pipe_active_pct_elapsed": f("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        "fp64_pipe_active_pct": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "registers_per_thread": f("launch__registers_per_thread"),
        "grid": f("launch__grid_size"),
        "smem_wavefronts": f("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
        "smem_bank_conflicts": f("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
        "sm_clock_ghz": f("sm__cycles_elapsed.avg.per_second"),
    }


def main():
    tag = sys.argv[1]
    rdir = os.path.join(PROF, "r01")
    os.makedirs(rdir, exist_ok=True)
    bench = [line for line in open(os.path.join(OUT, "bench.log")) if line.startswith("{")][-1]
    open(os.path.join(rdir, f"bench_{tag}.json"), "w").write(bench)
    kb = [line for line in open(os.path.join(OUT, "kbench.log")) if line.startswith("{")]
    open(os.path.join(rdir, f"kbench_{tag}.jsonl"), "w").write("".join(kb))
    ks = launches(os.path.join(OUT, "launches.csv"))
    json.dump({"command": "python bench.py --steps 2 --warmup 3 --no-cpu-baseline (cfg1), "
                          "ncu --metrics gpu__time_duration.sum --clock-control none",
               "note": "cold-cache serialised launches incl. prime and warm-up; compare shares",
               "kernels": ks}, open(os.path.join(rdir, f"launches_bench_cfg1_{tag}.json"), "w"), indent=1)
    s = ncu_summary(os.path.join(OUT, "prof_top_c1.ncu-rep"))
    json.dump(s, open(os.path.join(rdir, f"ncu_top_cfg1_{tag}.json"), "w"), indent=1)
    json.dump(s, open(os.path.join(PROF, "moment_top_traffic.json"), "w"), indent=1)
    print(json.dumps(s, indent=1))
    for k in ks[:8]:
        print(k)


if __name__ == "__main__":
    main()
