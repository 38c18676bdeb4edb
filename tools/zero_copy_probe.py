"""Probe: K1 streaming straight over the host link (no staging copies).

Pinned host buffers are device-addressable under UVA, so gs_apply_device can
take host pointers: the kernel's 16-byte loads become PCIe reads of the host
shards and its stores PCIe writes into the host parity. Compares, for the C2
e2e workload (8 x 8 MiB host shards -> 2 x 8 MiB host parity):
  * staged  : gs_encode_host (H2D pieces -> K1 -> D2H pieces, overlapped)
  * zc_dev  : K1 reads host, writes device parity (+ separate D2H)
  * zc_host : K1 reads host, writes host parity (one kernel, nothing else)
and the raw copy-engine rates. Wall clock around synchronous calls.
"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_00831_b200 import _lib as L  # noqa: E402
from paper_2605_00831_b200 import coding as G  # noqa: E402
from paper_2605_00831_b200 import device as D  # noqa: E402
from paper_2605_00831_b200.coding import check  # noqa: E402


def timeit(fn, steps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / steps


def main():
    per = int(sys.argv[1]) if len(sys.argv) > 1 else 32 * 262144
    n, k = 8, 2
    scheme = G.CodingScheme.reed_solomon(n, k)
    enc = G.encoder(scheme)
    lib = L.lib()
    h_in = torch.randint(0, 256, (n, per), dtype=torch.uint8).pin_memory()
    h_out = torch.zeros((k, per), dtype=torch.uint8).pin_memory()
    d_out = torch.empty((k, per), dtype=torch.uint8, device="cuda")
    want = D.encode(scheme, h_in.cuda()).cpu()
    pi = L.ptr_array([h_in[j].data_ptr() for j in range(n)])
    po = L.ptr_array([h_out[i].data_ptr() for i in range(k)])
    pd = L.ptr_array([d_out[i].data_ptr() for i in range(k)])
    st = torch.cuda.current_stream().cuda_stream
    pipe = D.Pipeline(0, 256 << 20)
    res = {"bytes_in": n * per, "bytes_out": k * per}

    t = timeit(lambda: check(lib.gs_encode_host(pipe.handle, enc.handle, pi, po, per), "staged"))
    res["staged_gbs"] = round(n * per / t / 1e9, 2)
    res["staged_ok"] = torch.equal(h_out, want)
    h_out.zero_()

    def zc_dev():
        check(lib.gs_apply_device(enc.handle, 1, pi, pd, per, st), "zc_dev")
        h_out.copy_(d_out, non_blocking=True)
    t = timeit(zc_dev)
    res["zc_dev_gbs"] = round(n * per / t / 1e9, 2)
    res["zc_dev_ok"] = torch.equal(h_out, want)
    h_out.zero_()

    t = timeit(lambda: check(lib.gs_apply_device(enc.handle, 1, pi, po, per, st), "zc_host"))
    torch.cuda.synchronize()
    res["zc_host_gbs"] = round(n * per / t / 1e9, 2)
    res["zc_host_ok"] = torch.equal(h_out, want)

    # kernel-only read rate of the host shards: XOR(8) -> device output
    x = G.encoder(G.CodingScheme.xor_code(n))
    t = timeit(lambda: check(lib.gs_apply_device(x.handle, 1, pi, pd, per, st), "zc_xor"))
    res["zc_read_xor_dev_gbs"] = round(n * per / t / 1e9, 2)

    da = torch.empty(n * per, dtype=torch.uint8, device="cuda")
    t = timeit(lambda: da.copy_(h_in.view(-1), non_blocking=True))
    res["copy_h2d_gbs"] = round(n * per / t / 1e9, 2)
    for v in (0, 1):
        check(lib.gs_set_kernel_variant(v))
        t = timeit(lambda: check(lib.gs_apply_device(enc.handle, 1, pi, po, per, st), "zc_host"))
        res[f"zc_host_variant{v}_gbs"] = round(n * per / t / 1e9, 2)
    check(lib.gs_set_kernel_variant(2))
    print(json.dumps(res), flush=True)
    pipe.close()


if __name__ == "__main__":
    main()
