"""Host-side cost of one small pipelined call (no GPU wait): wall time per
gs_encode_offload / gs_apply_device enqueue for a 1-stripe RS(8,2) encode of
64 KiB shards, and of the bare ctypes round trip, averaged over many calls.
The GPU work is tiny, so this is what bounds eager small-block throughput.
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
from paper_2605_00831_b200 import device as D  # noqa: E402
from paper_2605_00831_b200.coding import CodingScheme, check, encoder  # noqa: E402


def per_call(fn, reps=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    t = (time.perf_counter() - t0) / reps
    torch.cuda.synchronize()
    return round(t * 1e6, 2)


def main():
    lib = L.lib()
    n, k, ln = 8, 2, 65536
    enc = encoder(CodingScheme.reed_solomon(n, k))
    data = torch.randint(0, 256, (n, ln), dtype=torch.uint8, device="cuda")
    par = torch.empty((k, ln), dtype=torch.uint8, device="cuda")
    hp = torch.empty((k, ln), dtype=torch.uint8).pin_memory()
    sl = L.ptr_array([data[j].data_ptr() for j in range(n)])
    ol = L.ptr_array([par[i].data_ptr() for i in range(k)])
    hl = L.ptr_array([hp[i].data_ptr() for i in range(k)])
    pipe = D.Pipeline(0, 64 << 20)
    st = torch.cuda.Stream()
    cs, ks = st.cuda_stream, torch.cuda.Stream().cuda_stream
    out = {
        "ctypes_noop_us": per_call(lambda: lib.gs_abi_version()),
        "apply_device_us": per_call(lambda: check(lib.gs_apply_device(enc.handle, 1, sl, ol, ln, cs))),
        "encode_offload_us": per_call(lambda: check(lib.gs_encode_offload(pipe.handle, enc.handle, 1, sl, hl, ln,
                                                                          cs, ks))),
        "torch_empty_kernel_us": per_call(lambda: par.zero_()),
    }
    print(json.dumps(out), flush=True)
    pipe.close()


if __name__ == "__main__":
    main()
