"""Summarise the ncu range captures of tools/link_capture.py (host-link legs)
into one JSON: PCIe bytes, range duration, achieved GB/s, PCIe throughput %.

  python tools/link_summary.py gpurun_out/link_encode_r2.csv gpurun_out/link_rebuild_r2.csv \
      --out profiles/r2_link_capture.json
"""
import argparse
import csv
import json


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    head = rows[0]
    vals = {}
    for r in rows[1:]:
        rec = dict(zip(head, r))
        vals[rec["Metric Name"]] = (float(rec["Metric Value"].replace(",", "")), rec["Metric Unit"])
    return vals


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csvs", nargs="+")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    out = {"method": "ncu --replay-mode app-range (cudaProfilerStart/Stop around one call; copies and kernels "
                     "together), tools/link_capture.py", "legs": {}}
    for p in a.csvs:
        v = load(p)
        leg = ("e2e_call (gs_encode_host: H2D of 8 x 80 MiB data + K1 + D2H of 2 x 80 MiB parity)" if "e2e" in p
               else "encode_step (K1 + D2H of 2 x 80 MiB parity)" if "encode" in p
               else "chunk_rebuild (H2D of parity row 0 + K2)")
        ns = v["gpu__time_duration.sum"][0]
        wr, rd = v["pcie__write_bytes.sum"][0], v["pcie__read_bytes.sum"][0]
        out["legs"][leg] = {"range_us": round(ns / 1e3, 1), "pcie_write_bytes (device->host)": int(wr),
                            "pcie_read_bytes (host->device)": int(rd),
                            "d2h_gbs": round(wr / ns, 2), "h2d_gbs": round(rd / ns, 2),
                            "pcie_throughput_pct": v["pcie__throughput.avg.pct_of_peak_sustained_elapsed"][0],
                            "dram_read_bytes": int(v["dram__bytes_read.sum"][0]),
                            "dram_write_bytes": int(v["dram__bytes_write.sum"][0])}
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
