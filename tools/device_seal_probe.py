"""The device-sealed C2 block checkpoint (bench.host_tier_device_sealed):
host time per block of its parts, and the rate with more buffers in flight /
without the store commit, to find what holds it below the plain offload."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_00831_b200 import _lib as L  # noqa: E402
from paper_2605_00831_b200.coding import CodingScheme, check, encoder  # noqa: E402
from paper_2605_00831_b200.parity_store import ParityStore  # noqa: E402

S, N, K, SL = 32, 8, 2, 262144


def run(R, commit=True, blocks=64, threads=14):
    dev = torch.device("cuda", 0)
    scheme = CodingScheme.reed_solomon(N, K)
    enc, lib = encoder(scheme), L.lib()
    ring = torch.randint(0, 256, (8, S, N, SL), dtype=torch.uint8, device=dev)
    slots = [L.ptr_array([ring[b, s, j].data_ptr() for s in range(S) for j in range(N)]) for b in range(8)]
    comp, copy = torch.cuda.Stream(), torch.cuda.Stream()
    store = ParityStore(seal_threads=threads)
    store.bind_device(0)
    par = torch.empty((R, S, K, SL), dtype=torch.uint8, device=dev)
    sums = [torch.zeros(S, dtype=torch.int64, device=dev) for _ in range(R)]
    rows = [L.ptr_array([par[i, s, r].data_ptr() for s in range(S) for r in range(K)]) for i in range(R)]
    free = [None] * R
    t = {"wait": 0.0, "reserve": 0.0, "k1": 0.0, "offload": 0.0, "commit": 0.0}

    def one(b):
        i = b % R
        a = time.perf_counter()
        if free[i] is not None:
            comp.wait_event(free[i])
            free[i].synchronize()
        b1 = time.perf_counter()
        keys = [(s, b) for s in range(S)]
        acc, dst = store.reserve_batch(keys, scheme, 16, SL)
        b2 = time.perf_counter()
        check(lib.gs_apply_device(enc.handle, S, slots[b % 8], rows[i], SL, comp.cuda_stream), "k1")
        b3 = time.perf_counter()
        check(lib.gs_parity_offload_sealed(rows[i], S, K, SL, L.ptr_array(dst), sums[i].data_ptr(),
                                           comp.cuda_stream, copy.cuda_stream), "device seal")
        b4 = time.perf_counter()
        if commit:
            store.commit_sealed_batch(keys, sums[i].data_ptr(), copy)
        free[i] = torch.cuda.Event()
        free[i].record(copy)
        b5 = time.perf_counter()
        for k_, v in zip(t, (b1 - a, b2 - b1, b3 - b2, b4 - b3, b5 - b4)):
            t[k_] += v

    for b in range(blocks):
        one(b)
    copy.synchronize()
    store.wait_sealed()
    for s in range(S):
        store.erase_request(s)
    for k_ in t:
        t[k_] = 0.0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for b in range(blocks):
        one(b)
    copy.synchronize()
    t_gpu = time.perf_counter() - t0
    store.wait_sealed()
    t_all = time.perf_counter() - t0
    data = blocks * S * N * SL
    store.close()
    return {"R": R, "commit": commit, "gbs_until_d2h": round(data / t_gpu / 1e9, 1),
            "gbs_sealed": round(data / t_all / 1e9, 1),
            "host_us_per_block": {k_: round(v / blocks * 1e6, 1) for k_, v in t.items()}}


def main():
    for R, commit in ((8, True), (4, True), (4, False), (16, True), (4, True), (8, True)):
        print(json.dumps(run(R, commit)), flush=True)


if __name__ == "__main__":
    main()
