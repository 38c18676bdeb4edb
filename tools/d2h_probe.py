"""Sustained device->host copy rate in the shapes the C3 step uses (not the
bench): 20 steps of 160 MiB parity D2H into pinned memory as one copy per
step, as 6 pieces (2 rows x 32/32/16 MiB, the pipeline's), on one stream or
split over two streams (two DMA engines), and the single 256 MiB copy
bench.py's host_link_peaks takes as the link peak. Device-timed with events."""
import json

import torch

MiB = 1 << 20


def run(name, steps, pieces, streams):
    src = torch.empty((2, 80 * MiB), dtype=torch.uint8, device="cuda")
    dst = torch.empty((steps, 2, 80 * MiB), dtype=torch.uint8).pin_memory()
    ss = [torch.cuda.Stream() for _ in range(streams)]

    def go():
        for t in range(steps):
            i = 0
            for r in range(2):
                o = 0
                for p in pieces:
                    st = ss[i % streams]
                    with torch.cuda.stream(st):
                        dst[t, r, o:o + p].copy_(src[r, o:o + p], non_blocking=True)
                    o += p
                    i += 1

    go()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    e0.record(cur)
    for st in ss:
        st.wait_stream(cur)
    go()
    for st in ss:
        cur.wait_stream(st)
    e1.record(cur)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    return {"shape": name, "gbs": round(steps * 160 * MiB / (ms * 1e-3) / 1e9, 2), "ms_per_step": round(ms / steps, 3)}


def main():
    out = []
    out.append(run("1 stream, 2 x 80 MiB per step", 20, [80 * MiB], 1))
    out.append(run("1 stream, pipeline pieces 32/32/16 MiB", 20, [32 * MiB, 32 * MiB, 16 * MiB], 1))
    out.append(run("2 streams, pipeline pieces", 20, [32 * MiB, 32 * MiB, 16 * MiB], 2))
    out.append(run("2 streams, 2 x 80 MiB (one row per stream)", 20, [80 * MiB], 2))
    out.append(run("1 stream, 8 MiB pieces", 20, [8 * MiB] * 10, 1))
    out.append(run("2 streams, 8 MiB pieces", 20, [8 * MiB] * 10, 2))
    h = torch.empty(256 * MiB, dtype=torch.uint8).pin_memory()
    d = torch.empty(256 * MiB, dtype=torch.uint8, device="cuda")
    best = 0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h.copy_(d, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = max(best, 256 * MiB / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    out.append({"shape": "host_link_peaks: one 256 MiB copy, best of 5", "gbs": round(best, 2)})
    for r in out:
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
