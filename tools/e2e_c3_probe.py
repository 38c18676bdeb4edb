"""e2e (gs_encode_host_async, host buffers) at the C3 step geometry vs the
staging-ring size, next to the bare H2D of the same 640 MiB (the bound)."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_00831_b200 import _lib as L, coding as G, device as D  # noqa: E402
from paper_2605_00831_b200.coding import check  # noqa: E402

PER = 83886080


def main():
    lib = L.lib()
    h_in = [torch.randint(0, 256, (8, PER), dtype=torch.uint8).pin_memory() for _ in range(2)]
    h_out = torch.empty((2, PER), dtype=torch.uint8).pin_memory()
    enc = G.encoder(G.CodingScheme.reed_solomon(8, 2))
    pi = [L.ptr_array([h[j].data_ptr() for j in range(8)]) for h in h_in]
    po = L.ptr_array([h_out[i].data_ptr() for i in range(2)])
    d = torch.empty((8, PER), dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    for _ in range(3):
        d.copy_(h_in[0], non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(10):
        d.copy_(h_in[i % 2], non_blocking=True)
    torch.cuda.synchronize()
    h2d = 10 * 8 * PER / (time.perf_counter() - t0) / 1e9
    print(json.dumps({"bare_h2d_gbs": round(h2d, 2)}), flush=True)
    for mib in (256, 512, 1024, 256):
        pipe = D.Pipeline(0, mib << 20)
        for i in range(3):
            check(lib.gs_encode_host_async(pipe.handle, enc.handle, pi[i % 2], po, PER), "e2e")
        check(lib.gs_pipeline_sync(pipe.handle), "sync")
        best = 0
        for _ in range(3):
            t0 = time.perf_counter()
            for i in range(10):
                check(lib.gs_encode_host_async(pipe.handle, enc.handle, pi[i % 2], po, PER), "e2e")
            check(lib.gs_pipeline_sync(pipe.handle), "sync")
            best = max(best, 10 * 8 * PER / (time.perf_counter() - t0) / 1e9)
        print(json.dumps({"staging_mib": mib, "e2e_gbs": round(best, 2), "frac_of_bare_h2d": round(best / h2d, 3)}),
              flush=True)
        pipe.close()


if __name__ == "__main__":
    main()
