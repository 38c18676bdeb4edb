"""Summarise an ncu report (read here, no GPU needed) into the JSON kept
under profiles/: per captured kernel the duration, DRAM bytes, throughput
percentages, occupancy, pipe utilisation and the warp-stall breakdown.

  python tools/ncu_summary.py gpurun_out/k1.ncu-rep --out profiles/k1_ncu_summary.json \
      --alg-bytes 83886080 --note "..."
"""
import argparse
import csv
import io
import json
import subprocess

KEEP = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second",
    "lts__t_sector_hit_rate.pct",
]
STALL_PREFIX = "smsp__average_warp_latency_issue_stalled_"
STALL_PREFIX2 = "smsp__average_warps_issue_stalled_"


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return float(v.replace(",", "")) * scale.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--out", required=True)
    ap.add_argument("--alg-bytes", type=int, default=None, help="algorithmic bytes per launch")
    ap.add_argument("--source", default="")
    ap.add_argument("--launch", default="")
    ap.add_argument("--note", default="")
    ap.add_argument("--lib-sha", default="", help="sha256[:16] of the libghostserve_b200.so that was profiled")
    ap.add_argument("--src-sha", default="", help="tools/srcsha.py of the sources that were profiled")
    a = ap.parse_args()
    raw = subprocess.check_output(["ncu", "-i", a.report, "--page", "raw", "--csv"]).decode()
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, body = rows[0], rows[1], rows[2:]
    caps = []
    for r in body:
        rec = dict(zip(head, r))
        u = dict(zip(head, units))
        cap = {"kernel": rec.get("Kernel Name", "")}
        for m in KEEP:
            if m in rec:
                cap[m] = [rec[m], u.get(m, "")]
        stalls = {}
        for m, v in rec.items():
            for pre in (STALL_PREFIX2, STALL_PREFIX):
                if m.startswith(pre) and m.endswith("_per_issue_active.ratio"):
                    name = m[len(pre):-len("_per_issue_active.ratio")]
                    try:
                        stalls[name] = round(float(v.replace(",", "")), 2)
                    except ValueError:
                        pass
        if stalls:
            cap["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:12])
        caps.append(cap)
    import os
    out = {"source": a.source, "launch": a.launch, "note": a.note, "file": os.path.basename(a.report),
           "lib_sha256_16": a.lib_sha, "src_sha256_16": a.src_sha, "captures": caps}
    if caps:
        c = caps[-1]
        out["kernel"] = c["kernel"]
        rd = to_bytes(*c["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in c else None
        wr = to_bytes(*c["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in c else None
        if rd is not None and wr is not None:
            out["dram_read_bytes_per_launch"] = int(rd)
            out["dram_write_bytes_per_launch"] = int(wr)
            out["dram_bytes_per_launch"] = int(rd + wr)
        if a.alg_bytes:
            out["algorithmic_bytes_per_launch"] = a.alg_bytes
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "captures"}))


if __name__ == "__main__":
    main()
