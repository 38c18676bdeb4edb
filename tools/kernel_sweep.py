"""Kernel-only throughput sweep (not the bench): K1 RS(8,2) encode and K2
single-loss rebuild over growing shard sizes, both specialised variants,
next to torch's device copy of the same byte volume (the roofline
reference). Times CUDA-graph replays with events on the launch stream.

    python tools/kernel_sweep.py [--sizes 1,4,16,64,256] (MiB per shard)
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_00831_b200 import _lib as L  # noqa: E402
from paper_2605_00831_b200.coding import CodingScheme, ErasurePattern, check, decoder, encoder  # noqa: E402


def graph_time(fn, reps, stream):
    with torch.cuda.stream(stream):
        fn()
    stream.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(reps):
            fn()
    with torch.cuda.stream(stream):
        g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(3):
            g.replay()
        e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / (3 * reps) * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="0.25,1,4,16,64,256")
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--k", type=int, default=2)
    ap.add_argument("--kind", choices=["rs", "rdp", "xor"], default="rs")
    ap.add_argument("--lost", default="1", help="comma-separated lost shard indices for K2")
    ap.add_argument("--generic", action="store_true", help="runtime-coefficient (PRMT split-table) back end")
    args = ap.parse_args()
    lib = L.lib()
    dev = torch.device("cuda:0")
    st = torch.cuda.Stream()
    n, k = args.n, args.k
    scheme = {"rs": lambda: CodingScheme.reed_solomon(n, k), "rdp": lambda: CodingScheme.rdp(n),
              "xor": lambda: CodingScheme.xor_code(n)}[args.kind]()
    k = scheme.k
    lost = [int(x) for x in args.lost.split(",")]
    if args.generic:
        from paper_2605_00831_b200.coding import codec_ex
        enc = codec_ex(scheme, generic=True)
        dec = codec_ex(scheme, ErasurePattern(lost), generic=True)
    else:
        enc = encoder(scheme)
        dec = decoder(scheme, ErasurePattern(lost))
        # codecs outside the compiled registry: wait for their runtime-specialised build
        import ctypes as C
        for c in (enc, dec):
            js = C.c_int()
            lib.gs_codec_jit_status(c.handle, 1, C.byref(js))
    out = []
    for mib in [float(x) for x in args.sizes.split(",")]:
        L_ = int(mib * (1 << 20)) // 4096 * 4096
        nbuf = max(2, min(8, int((1 << 30) // (L_ * (n + k))) ))  # rotate so data > L2
        data = torch.randint(0, 256, (nbuf, n, L_), dtype=torch.uint8, device=dev)
        par = torch.empty((nbuf, k, L_), dtype=torch.uint8, device=dev)
        reb = torch.empty((nbuf, max(dec.n_out, 1), L_), dtype=torch.uint8, device=dev)
        sl = [L.ptr_array([data[b, j].data_ptr() for j in range(n)]) for b in range(nbuf)]
        ol = [L.ptr_array([par[b, i].data_ptr() for i in range(k)]) for b in range(nbuf)]
        dl = [L.ptr_array([None if j in lost else (data[b, j].data_ptr() if j < n else par[b, j - n].data_ptr())
                           for j in range(n + k)]) for b in range(nbuf)]
        rl = [L.ptr_array([reb[b, i].data_ptr() for i in range(dec.n_out)]) for b in range(nbuf)]
        dec_bytes = (len(dec.coefficients().any(axis=0).nonzero()[0]) + dec.n_out) * L_
        row = {"kind": args.kind, "n": n, "k": k, "generic": args.generic, "mib_per_shard": mib, "bytes_enc": (n + k) * L_, "bytes_dec": dec_bytes}
        for v in (0, 1):
            check(lib.gs_set_kernel_variant(v))
            cnt = [0]

            def k1():
                b = cnt[0] % nbuf
                cnt[0] += 1
                check(lib.gs_apply_device(enc.handle, 1, sl[b], ol[b], L_, st.cuda_stream))

            def k2():
                b = cnt[0] % nbuf
                cnt[0] += 1
                check(lib.gs_apply_device(dec.handle, 1, dl[b], rl[b], L_, st.cuda_stream))
            t1 = graph_time(k1, nbuf * 2, st)
            t2 = graph_time(k2, nbuf * 2, st)
            row[f"k1_v{v}_gbs"] = round((n + k) * L_ / t1 / 1e9, 1)
            row[f"k2_v{v}_gbs"] = round(dec_bytes / t2 / 1e9, 1)
            row[f"k1_v{v}_us"] = round(t1 * 1e6, 2)
        # device copy of the same byte volume (read + write), rotating over
        # buffers so the L2 cannot serve it: the attainable HBM rate at this size
        half = (n + k) * L_ // 2
        ncp = max(2, min(8, int((1 << 30) // half)))
        src = torch.empty((ncp, half), dtype=torch.uint8, device=dev)
        dst = torch.empty_like(src)
        cc = [0]

        def cp():
            b = cc[0] % ncp
            cc[0] += 1
            dst[b].copy_(src[b])
        tc = graph_time(cp, ncp * 2, st)
        row["copy_gbs"] = round((n + k) * L_ / tc / 1e9, 1)
        out.append(row)
        print(json.dumps(row), flush=True)
        del data, par, reb, src, dst
    check(lib.gs_set_kernel_variant(2))


if __name__ == "__main__":
    main()
