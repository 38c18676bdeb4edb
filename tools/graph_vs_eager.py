"""Per-block checkpoint latency: eager Pipeline.encode_offload vs the same
call replayed from a CUDA graph (device.capture_offload).

One block = 32 requests x RS(8,2) x `slice` bytes per worker (C2 shape at
slice = 256 KiB). Prints one JSON line per slice size with the mean wall
time per block (enqueue + completion, 200 blocks back to back) and the
number of host API calls the eager path makes per block.

  python tools/graph_vs_eager.py [--slices 4096,16384,65536,262144]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_00831_b200 import coding as G, device as D  # noqa: E402


def timed(fn, iters):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(iters):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--slices", default="4096,16384,65536,262144")
    ap.add_argument("--requests", type=int, default=32)
    ap.add_argument("--iters", type=int, default=200)
    a = ap.parse_args()
    scheme = G.CodingScheme.reed_solomon(8, 2)
    for ln in [int(x) for x in a.slices.split(",")]:
        S = a.requests
        data = torch.randint(0, 256, (S, 8, ln), dtype=torch.uint8, device="cuda")
        h_par = torch.zeros((S, 2, ln), dtype=torch.uint8).pin_memory()
        pipe = D.Pipeline(0, 64 << 20)
        comp, copy = torch.cuda.Stream(), torch.cuda.Stream()

        def eager():
            pipe.encode_offload(scheme, data, h_par, compute=comp, copy=copy)
            comp.wait_stream(copy)

        for _ in range(5):
            eager()
        k0 = D.launches()
        t_eager = timed(eager, a.iters)
        kpb = (D.launches() - k0) / a.iters
        g = D.capture_offload(scheme, data, h_par, staging_bytes=64 << 20)
        for _ in range(5):
            g.replay()
        t_graph = timed(g.replay, a.iters)
        torch.cuda.synchronize()
        ok = torch.equal(h_par, D.encode(scheme, data).cpu())
        print(json.dumps({"slice_bytes": ln, "requests": S, "block_bytes": S * 8 * ln,
                          "eager_us_per_block": round(t_eager * 1e6, 2),
                          "graph_us_per_block": round(t_graph * 1e6, 2),
                          "kernels_per_block": kpb, "parity_ok": ok}), flush=True)
        pipe.close()


if __name__ == "__main__":
    main()
