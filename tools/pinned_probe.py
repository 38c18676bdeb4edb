"""D2H / H2D rate into pinned host memory by allocation kind (not the bench):
cudaHostAlloc (what the bench and torch use on one-node hosts), mmap +
cudaHostRegister with 4 KiB pages, and mmap + MADV_HUGEPAGE (THP) +
cudaHostRegister. 160 MiB per step (the C3 step's parity), 20 steps, events."""
import ctypes as C
import json
import mmap
import os

import torch
from cuda.bindings import runtime as rt

MiB = 1 << 20
N = 160 * MiB
libc = C.CDLL("libc.so.6", use_errno=True)
libc.mmap.restype = C.c_void_p
libc.mmap.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_long]
libc.madvise.argtypes = [C.c_void_p, C.c_size_t, C.c_int]


def mapped(huge: bool) -> int:
    p = libc.mmap(None, N + (2 * MiB), 3, 0x22, -1, 0)  # RW, MAP_PRIVATE | MAP_ANONYMOUS
    p = (p + 2 * MiB - 1) // (2 * MiB) * (2 * MiB)
    if huge:
        libc.madvise(p, N, 14)  # MADV_HUGEPAGE
    C.memset(p, 0, N)
    err, = rt.cudaHostRegister(p, N, 0)
    assert int(err) == 0, err
    return p


def main():
    d = torch.empty(N, dtype=torch.uint8, device="cuda")
    st = torch.cuda.Stream()
    err, ha = rt.cudaHostAlloc(N, 0)
    kinds = {"cudaHostAlloc": ha, "mmap+register 4K": mapped(False), "mmap+THP+register": mapped(True)}
    for name, p in kinds.items():
        for kind, (dst, src, k) in {"d2h": (p, d.data_ptr(), rt.cudaMemcpyKind.cudaMemcpyDeviceToHost),
                                    "h2d": (d.data_ptr(), p, rt.cudaMemcpyKind.cudaMemcpyHostToDevice)}.items():
            for _ in range(3):
                rt.cudaMemcpyAsync(dst, src, N, k, st.cuda_stream)
            st.synchronize()
            best = []
            for rep in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for _ in range(20):
                    rt.cudaMemcpyAsync(dst, src, N, k, st.cuda_stream)
                e1.record(st)
                e1.synchronize()
                best.append(20 * N / (e0.elapsed_time(e1) * 1e-3) / 1e9)
            print(json.dumps({"alloc": name, "dir": kind, "gbs_runs": [round(x, 2) for x in best]}), flush=True)


if __name__ == "__main__":
    main()
