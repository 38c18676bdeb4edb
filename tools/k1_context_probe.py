"""Why is K1 slower inside the checkpoint step than back to back? Times the
C2 K1 launch (32 stripes x RS(8,2) x 256 KiB) with events around each launch
in different surroundings:
  back_to_back   : eager launches, nothing else running
  with_d2h       : a second stream streams 16 MiB D2H copies continuously
  idle_gaps      : a ~300 us spin kernel between launches (GPU otherwise idle)
  gaps_and_d2h   : both (the checkpoint step's situation)
  with_h2d / with_d2d_ce / with_d2h_1m : other copy-engine traffic shapes
"""
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_00831_b200 import _lib as L  # noqa: E402
from paper_2605_00831_b200.coding import CodingScheme, check, encoder  # noqa: E402


def main():
    S, n, k, ln, B = 32, 8, 2, 262144, 8
    dev = torch.device("cuda")
    data = torch.randint(0, 256, (B, S, n, ln), dtype=torch.uint8, device=dev)
    par = torch.empty((B, S, k, ln), dtype=torch.uint8, device=dev)
    enc = encoder(CodingScheme.reed_solomon(n, k))
    lib = L.lib()
    sl = [L.ptr_array([data[b, s, j].data_ptr() for s in range(S) for j in range(n)]) for b in range(B)]
    ol = [L.ptr_array([par[b, s, i].data_ptr() for s in range(S) for i in range(k)]) for b in range(B)]
    st, cp = torch.cuda.Stream(), torch.cuda.Stream()
    h = torch.empty(16 << 20, dtype=torch.uint8).pin_memory()
    d = torch.empty(16 << 20, dtype=torch.uint8, device=dev)
    from cuda.bindings import runtime as rt
    d2 = torch.empty(16 << 20, dtype=torch.uint8, device=dev)
    # host buffer on transparent huge pages (2 MiB), then registered (pinned)
    libc = C.CDLL("libc.so.6", use_errno=True)
    libc.mmap.restype = C.c_void_p
    libc.mmap.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_long]
    libc.madvise.argtypes = [C.c_void_p, C.c_size_t, C.c_int]
    hsz = 32 << 20
    raw = libc.mmap(None, hsz + (2 << 20), 3, 0x22, -1, 0)  # PROT_READ|WRITE, MAP_PRIVATE|ANONYMOUS
    hp = (raw + (2 << 20) - 1) // (2 << 20) * (2 << 20)
    rc = libc.madvise(C.c_void_p(hp), hsz, 14)  # MADV_HUGEPAGE
    C.memset(hp, 1, hsz)
    rt.cudaHostRegister(hp, hsz, 0)
    huge_info = {"madvise_rc": rc}
    try:
        with open("/proc/meminfo") as f:
            huge_info["AnonHugePages"] = [l.split()[1] for l in f if l.startswith("AnonHugePages")][0]
    except Exception:
        pass

    def spin(us):
        # busy-wait kernel on `st` (torch._sleep takes cycles)
        torch.cuda._sleep(int(us * 1965))

    def run(mode, reps=64):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        torch.cuda.synchronize()
        ncp = reps * (20 if "gaps" in mode else 2)
        if mode in ("with_d2h", "gaps_and_d2h"):
            with torch.cuda.stream(cp):
                for _ in range(ncp):
                    h.copy_(d, non_blocking=True)
        elif mode == "with_d2h_1m":
            for _ in range(ncp * 16):
                rt.cudaMemcpyAsync(h.data_ptr(), d.data_ptr(), 1 << 20,
                                   rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, cp.cuda_stream)
        elif mode == "with_d2h_huge":
            for _ in range(ncp):
                rt.cudaMemcpyAsync(hp, d.data_ptr(), 16 << 20, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost,
                                   cp.cuda_stream)
        elif mode == "with_h2d":
            with torch.cuda.stream(cp):
                for _ in range(ncp):
                    d.copy_(h, non_blocking=True)
        elif mode == "with_d2d_ce":
            for _ in range(ncp * 8):
                rt.cudaMemcpyAsync(d2.data_ptr(), d.data_ptr(), 16 << 20,
                                   rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice, cp.cuda_stream)
        with torch.cuda.stream(st):
            for i in range(reps):
                if "gaps" in mode:
                    spin(300)
                evs[i][0].record(st)
                check(lib.gs_apply_device(enc.handle, S, sl[i % B], ol[i % B], ln, st.cuda_stream), "k1")
                evs[i][1].record(st)
        torch.cuda.synchronize()
        t = sorted(a.elapsed_time(b) * 1e3 for a, b in evs[4:])
        return {"median_us": round(t[len(t) // 2], 2), "min_us": round(t[0], 2), "max_us": round(t[-1], 2)}

    out = {}
    for mode in ("back_to_back", "with_d2h", "idle_gaps", "gaps_and_d2h", "with_d2h_1m", "with_h2d",
                 "with_d2d_ce", "with_d2h_huge"):
        run(mode, 8)
        out[mode] = run(mode)
    out["huge"] = huge_info
    # one event pair around 64 back-to-back launches (event latency amortised)
    for mode in ("alone", "with_d2h"):
        torch.cuda.synchronize()
        if mode == "with_d2h":
            with torch.cuda.stream(cp):
                for _ in range(400):
                    h.copy_(d, non_blocking=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record(st)
            for i in range(64):
                check(lib.gs_apply_device(enc.handle, S, sl[i % B], ol[i % B], ln, st.cuda_stream), "k1")
            e1.record(st)
        torch.cuda.synchronize()
        out[f"batch64_{mode}_us_per_launch"] = round(e0.elapsed_time(e1) * 1e3 / 64, 2)
    # D2H rate into each host buffer alone
    for name, ptr in (("cudaHostAlloc", h.data_ptr()), ("thp_registered", hp)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cp)
        for _ in range(20):
            rt.cudaMemcpyAsync(ptr, d.data_ptr(), 16 << 20, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, cp.cuda_stream)
        e1.record(cp)
        e1.synchronize()
        out[f"d2h_gbs_{name}"] = round(20 * (16 << 20) / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
