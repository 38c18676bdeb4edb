"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) per
kernel: launches, total / mean ns, share of the listed GPU time. Cold-cache,
serialised per-launch times: compare SHARES with bench.py, not absolutes.

  python tools/launch_summary.py gpurun_out/launches_r1.csv --out profiles/r1_launches_summary.csv
"""
import argparse
import collections
import csv
import re


def short(name: str) -> str:
    m = re.match(r"(?:void )?(?:gsb::)?([A-Za-z_0-9:]+)(<.*>)?\(", name)
    base = m.group(1) if m else name[:60]
    if m and m.group(2):
        t = m.group(2)
        spec = re.search(r"(EncSpec|DecSpec)<[^>]*>", t)
        paged = re.search(r",\s*(\(bool\))?1>$", t.rstrip())
        if spec:
            base += f"<{spec.group(0)}{', paged' if paged and base == 'k_apply_special' else ''}>"
    return base


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    rows = [r for r in csv.reader(open(a.csv)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        k = short(r[ki])
        ns = float(r[vi].replace(",", ""))
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + ns)
    total = sum(t for _, t in agg.values())
    with open(a.out, "w") as f:
        f.write("kernel,launches,total_ns,mean_ns,share\n")
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"\"{k}\",{n},{int(t)},{int(t / n)},{t / total:.4f}\n")
    print(open(a.out).read())


if __name__ == "__main__":
    main()
