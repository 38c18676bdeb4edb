"""Host-link DMA shapes for the e2e pipeline: how fast 64 MiB of H2D moves
as one 1-D copy, as 1 MiB 1-D copies, as 2-D copies (8 rows x 1 MiB, pitch
8 MiB -- what gs_encode_host issues per piece), alone and with a concurrent
16 MiB D2H on a second stream. Device-timed with events; not the bench.
"""
import json

import torch
from cuda.bindings import runtime as rt

MiB = 1 << 20


def main():
    n, per = 8, 8 * MiB
    h = torch.empty((n, per), dtype=torch.uint8).pin_memory()
    d = torch.empty((n, per), dtype=torch.uint8, device="cuda")
    hp = torch.empty((2, per), dtype=torch.uint8).pin_memory()
    dp = torch.empty((2, per), dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost

    def one_1d():
        rt.cudaMemcpyAsync(d.data_ptr(), h.data_ptr(), n * per, H2D, s1.cuda_stream)

    def many_1d(piece):
        def f():
            for r0 in range(0, per, piece):
                for j in range(n):
                    rt.cudaMemcpyAsync(d[j].data_ptr() + r0, h[j].data_ptr() + r0, piece, H2D, s1.cuda_stream)
        return f

    def many_2d(piece):
        def f():
            for r0 in range(0, per, piece):
                rt.cudaMemcpy2DAsync(d.data_ptr() + r0, per, h.data_ptr() + r0, per, piece, n, H2D,
                                     s1.cuda_stream)
        return f

    def d2h_2d(piece):
        def f():
            for r0 in range(0, per, piece):
                rt.cudaMemcpy2DAsync(hp.data_ptr() + r0, per, dp.data_ptr() + r0, per, piece, 2, D2H,
                                     s2.cuda_stream)
        return f

    def timed(fns, reps=20):
        for f in fns:
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s1)
        s2.wait_event(e0)
        for _ in range(reps):
            for f in fns:
                f()
        s1.wait_stream(s2)
        e1.record(s1)
        e1.synchronize()
        return e0.elapsed_time(e1) / reps * 1e-3

    out = {}
    for name, f in (("h2d_1d_64MiB", one_1d), ("h2d_1d_1MiB_pieces", many_1d(MiB)),
                    ("h2d_2d_1MiB_rows", many_2d(MiB)), ("h2d_2d_256KiB_rows", many_2d(256 << 10)),
                    ("h2d_2d_2MiB_rows", many_2d(2 * MiB))):
        t = timed([f])
        out[name] = round(n * per / t / 1e9, 2)
        t = timed([f, d2h_2d(MiB)])
        out[name + "+d2h"] = round(n * per / t / 1e9, 2)
    t = timed([d2h_2d(MiB)])
    out["d2h_2d_1MiB_rows"] = round(2 * per / t / 1e9, 2)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
