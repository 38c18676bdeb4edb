"""Where the host-tier (ParityStore) C2 block checkpoint spends its time:
host time per block of reserve_batch / encode_offload / commit, and the
device-side D2H rate into store slabs vs into a plain pinned ring."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_00831_b200 import _lib as L  # noqa: E402
from paper_2605_00831_b200.coding import CodingScheme, check, encoder  # noqa: E402
from paper_2605_00831_b200.device import Pipeline  # noqa: E402
from paper_2605_00831_b200.parity_store import ParityStore  # noqa: E402

S, N, K, SL = 32, 8, 2, 262144


def main():
    dev = torch.device("cuda", 0)
    scheme = CodingScheme.reed_solomon(N, K)
    enc = encoder(scheme)
    ring = torch.randint(0, 256, (8, S, N, SL), dtype=torch.uint8, device=dev)
    slots = [L.ptr_array([ring[b, s, j].data_ptr() for s in range(S) for j in range(N)]) for b in range(8)]
    pipe = Pipeline(0, 64 << 20)
    comp, copy = torch.cuda.Stream(), torch.cuda.Stream()
    store = ParityStore(seal_threads=14)
    store.bind_device(0)
    blocks = 64
    res = {}
    for phase in ("warm", "timed"):
        tr = te = tc = 0.0
        t0 = time.perf_counter()
        for b in range(blocks):
            keys = [(s, b) for s in range(S)]
            a = time.perf_counter()
            acc, dst = store.reserve_batch(keys, scheme, 16, SL)
            bb = time.perf_counter()
            check(L.lib().gs_encode_offload(pipe.handle, enc.handle, S, slots[b % 8], L.ptr_array(dst), SL,
                                            comp.cuda_stream, copy.cuda_stream), "x")
            c = time.perf_counter()
            store.commit_batch(keys, copy)
            d = time.perf_counter()
            tr += bb - a
            te += c - bb
            tc += d - c
        copy.synchronize()
        t_d2h = time.perf_counter() - t0
        store.wait_sealed()
        t_all = time.perf_counter() - t0
        res[phase] = {"reserve_ms_per_block": round(tr / blocks * 1e3, 3), "encode_offload_ms": round(te / blocks * 1e3, 3),
                      "commit_ms": round(tc / blocks * 1e3, 3), "until_d2h_gbs": round(blocks * S * N * SL / t_d2h / 1e9, 1),
                      "sealed_gbs": round(blocks * S * N * SL / t_all / 1e9, 1)}
        for s in range(S):
            store.erase_request(s)
    # store destinations, but ONE commit after the whole loop (no per-block host callback)
    allkeys = []
    t0 = time.perf_counter()
    for b in range(blocks):
        keys = [(s, 1000 + b) for s in range(S)]
        acc, dst = store.reserve_batch(keys, scheme, 16, SL)
        check(L.lib().gs_encode_offload(pipe.handle, enc.handle, S, slots[b % 8], L.ptr_array(dst), SL,
                                        comp.cuda_stream, copy.cuda_stream), "x")
        allkeys += keys
    copy.synchronize()
    res["store_dsts_no_callback_gbs"] = round(blocks * S * N * SL / (time.perf_counter() - t0) / 1e9, 1)
    store.commit_batch(allkeys, copy)
    store.wait_sealed()
    # same loop into one reused pinned ring (no store)
    host = torch.empty((4, S, K, SL), dtype=torch.uint8).pin_memory()
    dsts = [L.ptr_array([host[i, s, r].data_ptr() for s in range(S) for r in range(K)]) for i in range(4)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for b in range(blocks):
        check(L.lib().gs_encode_offload(pipe.handle, enc.handle, S, slots[b % 8], dsts[b % 4], SL,
                                        comp.cuda_stream, copy.cuda_stream), "x")
    copy.synchronize()
    res["pinned_ring_gbs"] = round(blocks * S * N * SL / (time.perf_counter() - t0) / 1e9, 1)
    # footprint: a 1 GiB pinned ring (64 distinct blocks, like the store), plain
    # cudaHostAlloc vs transparent-huge-page backed + cudaHostRegister
    import ctypes
    import mmap
    big = torch.empty((blocks, S, K, SL), dtype=torch.uint8).pin_memory()
    bd = [L.ptr_array([big[i, s, r].data_ptr() for s in range(S) for r in range(K)]) for i in range(blocks)]

    def run_ring(d):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for b in range(blocks):
            check(L.lib().gs_encode_offload(pipe.handle, enc.handle, S, slots[b % 8], d[b], SL,
                                            comp.cuda_stream, copy.cuda_stream), "x")
        copy.synchronize()
        return round(blocks * S * N * SL / (time.perf_counter() - t0) / 1e9, 1)

    run_ring(bd)
    res["pinned_1gib_ring_gbs"] = run_ring(bd)
    nbytes = blocks * S * K * SL
    mm = mmap.mmap(-1, nbytes + (2 << 20))
    try:
        mm.madvise(mmap.MADV_HUGEPAGE)
    except Exception as e:   # noqa: BLE001
        res["thp_madvise_error"] = str(e)
    addr = ctypes.addressof(ctypes.c_char.from_buffer(mm))
    base = (addr + (2 << 20) - 1) & ~((2 << 20) - 1)
    ctypes.memset(base, 0, nbytes)
    rc = torch.cuda.cudart().cudaHostRegister(base, nbytes, 0)
    res["thp_register_rc"] = int(rc)
    try:
        res["thp_enabled"] = open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip()
        res["anon_huge_kb"] = [l for l in open("/proc/meminfo") if "AnonHugePages" in l][0].split()[1]
    except Exception:   # noqa: BLE001
        pass
    hd = [L.ptr_array([base + ((i * S + s) * K + r) * SL for s in range(S) for r in range(K)]) for i in range(blocks)]
    run_ring(hd)
    res["thp_1gib_ring_gbs"] = run_ring(hd)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
