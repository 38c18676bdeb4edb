"""Host-memory contention during the C3 recovery: the 5 GiB H2D of parity row 0
alone, and while host threads hash another 5 GiB of pinned host memory with
the bit-sliced FNV (what the verification's row-1 continuations do)."""
import ctypes as C
import json
import os
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_00831_b200 import _lib as L  # noqa: E402

PER, N = 83886080, 64


def main():
    lib = L.lib()
    row0 = torch.randint(0, 256, (N, PER), dtype=torch.uint8).pin_memory()
    row1 = torch.randint(0, 256, (N, PER), dtype=torch.uint8).pin_memory()
    dev = torch.empty((N, PER), dtype=torch.uint8, device="cuda")
    st = torch.cuda.Stream()

    def h2d():
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(st):
            for c in range(N):
                dev[c].copy_(row0[c], non_blocking=True)
        st.synchronize()
        return N * PER / (time.perf_counter() - t0) / 1e9

    h2d()
    alone = h2d()
    threads = int(os.environ.get("THREADS", "14"))
    ptrs = L.ptr_array([row1[c].data_ptr() for c in range(N)])
    outs = (C.c_uint64 * N)()
    res = {}

    def hash_all():
        t0 = time.perf_counter()
        lib.gs_parity_checksum_batch(ptrs, N, 1, PER, threads, outs)
        res["hash_gbs"] = N * PER / (time.perf_counter() - t0) / 1e9

    th = threading.Thread(target=hash_all)
    th.start()
    time.sleep(0.005)
    busy = h2d()
    th.join()
    t0 = time.perf_counter()
    lib.gs_parity_checksum_batch(ptrs, N, 1, PER, threads, outs)
    hash_alone = N * PER / (time.perf_counter() - t0) / 1e9
    print(json.dumps({"h2d_alone_gbs": round(alone, 2), "h2d_while_hashing_gbs": round(busy, 2),
                      "hash_threads": threads, "hash_alone_gbs": round(hash_alone, 2),
                      "hash_while_h2d_gbs": round(res["hash_gbs"], 2)}))


if __name__ == "__main__":
    main()
