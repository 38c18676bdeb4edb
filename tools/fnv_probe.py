"""GPU FNV-1a seal (gs_fnv1a64_device) vs the host seal: throughput on the
configs' parity batches, timed with CUDA events on the launching stream
(warm, median of repeats), and the host batch checksum on all cores beside it.

  C2 block : 32 chunks x RS(8,2) parity, 2 x 256 KiB each
  C3 prefill: 64 chunks x 2 x 80 MiB (10 GiB of parity)
"""
import ctypes as C
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_00831_b200 import _lib as L  # noqa: E402

OFFSET = 0xCBF29CE484222325


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C2,C3")
    want = ap.parse_args().configs.split(",")
    lib = L.lib()
    st = torch.cuda.Stream()
    res = []
    for name, chunks, ln, reps in [("C2", 32, 262144, 20), ("C3", 64, 83886080, 5)]:
        if name not in want:
            continue
        par = torch.randint(0, 256, (chunks, 2, ln), dtype=torch.uint8, device="cuda")
        ptrs = L.ptr_array([par[c, i].data_ptr() for c in range(chunks) for i in range(2)])
        out = torch.zeros(chunks, dtype=torch.int64, device="cuda")
        run = lambda: lib.gs_fnv1a64_device(ptrs, chunks, 2, ln, OFFSET, out.data_ptr(), st.cuda_stream)
        assert run() == 0, lib.gs_last_error()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            assert run() == 0
            e1.record(st)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[len(ts) // 2]
        # host seal of the same bytes (all cores), checked against the GPU
        hp = par.cpu()
        hptr = L.ptr_array([hp[c, i].data_ptr() for c in range(chunks) for i in range(2)])
        hout = (C.c_uint64 * chunks)()
        t0 = time.perf_counter()
        assert lib.gs_parity_checksum_batch(hptr, chunks, 2, ln, os.cpu_count() or 1, hout) == 0
        host_ms = (time.perf_counter() - t0) * 1e3
        dev = [int(v) & (2**64 - 1) for v in out.cpu().tolist()]
        ok = all(dev[c] == hout[c] for c in range(chunks))
        nbytes = chunks * 2 * ln
        res.append({"config": name, "chunks": chunks, "parity_bytes": nbytes, "gpu_ms": round(ms, 3),
                    "gpu_gbs": round(nbytes / ms / 1e6, 1), "host_ms": round(host_ms, 1),
                    "host_gbs": round(nbytes / host_ms / 1e6, 1), "host_threads": os.cpu_count(),
                    "launches_per_call": 10 if os.environ.get("GS_FNV_LEGACY") == "1" else 2,
                    "kernel": "legacy multi-pass" if os.environ.get("GS_FNV_LEGACY") == "1" else "k_fnv_window", "bit_exact": ok})
        print(json.dumps(res[-1]), flush=True)
        del par, hp


if __name__ == "__main__":
    main()
