"""Per-config results table: C1-C4 on one B200, each with
encode incl. D2H, K1 alone, lost-shard recovery, their roofline fractions,
the reference CPU codec on this host (1 thread as shipped and all cores;
checkpoint_chunk / reconstruct_chunk per chunk) and a full-size bit-exact
check of the GPU parity against the reference's own output.

    python bench.py --configs [--configs-only C1,C3]     (one JSON line per config)

Inputs are the reference KV stream (make_ground_truth_slice, kv_seed 3)
generated on the device; the CPU legs read host copies of stripe 0. The
reference (oracle/_ref) is used as the CPU baseline and as the checker only.

Rooflines: encode incl. D2H t* = max((n+k)·L·S / HBM, k·L·S / D2H);
K1 t* = (n+k)·L·S / HBM; recovery of e shards t* = max((n+e)·L·S / HBM,
e·L·S / H2D); frac = t* / t. Throughput = n·L·S / t (tools/ghostserve.cpp:279).
"""
from __future__ import annotations

import json
import os
import platform
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# name -> (kind, n, k, (layers, kv_heads, head_dim, tp), chunk tokens, stripes, lost, request-major?)
CONFIGS = {
    "C1": dict(scheme=("rs", 4, 2), geom=(32, 8, 128, 4), m=4096, stripes=1, lost=[1],
               what="RS(4,2), 32 L x 8 H x 128 D, 4,096 tokens, bs 1, tp 4 (4 x 128 MiB slices)",
               fp=("dc3fbb698a8561cd", "8c2a59acc76fa0d0")),
    "C2": dict(scheme=("rs", 8, 2), geom=(32, 8, 128, 8), m=16, stripes=32, lost=[5], by_request=True,
               what="Llama-3-8B TP=8, RS(8,2), one 16-token decode block of 32 requests (32 x 8 x 256 KiB)",
               fp=("b6fbcffd8cdef63e", "db184baa5292394a")),
    "C3": dict(scheme=("rs", 8, 2), geom=(80, 8, 128, 8), m=2048, stripes=64, lost=[5],
               what="Llama-3-70B TP=8, 128K-token prefill = 64 chunks x 8 x 80 MiB; worker 5's full shard "
                    "rebuilt (5 GiB)", fp=("1d3b4c93d3c5ee99", "a3d31fe0a4ccc6b0")),
    "C4": dict(scheme=("rs", 6, 2), geom=(80, 6, 128, 6), m=2048, stripes=8, lost=[0, 3],
               what="RS(6,2), 80 L x 6 H x 128 D tp 6, 8 chunks x 6 x 80 MiB, two lost shards {0,3}",
               fp=None),
}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def run_configs(args) -> None:
    import numpy as np
    import torch

    from oracle import oracle as O
    from paper_2605_00831_b200 import _lib as L
    from paper_2605_00831_b200 import device as D
    from paper_2605_00831_b200 import kv_layout as K
    from paper_2605_00831_b200.coding import CodingScheme, ErasurePattern, check, decoder, encoder

    sys.path.insert(0, ROOT)
    from bench import host_link_peaks, load_peaks

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    hbm, hbm_src = load_peaks()
    link = host_link_peaks(torch, dev)
    lib = L.lib()
    ref = O.ref() if O.have_ref() else None
    port = O.port()
    threads = os.cpu_count() or 1
    comp, copy = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    pipe = D.Pipeline(0, 256 << 20)
    only = set(args.configs_only.split(",")) if args.configs_only else set(CONFIGS)

    def ev_time(fn, reps):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        comp.wait_stream(torch.cuda.current_stream())
        e0.record(comp)
        for _ in range(reps):
            fn()
        comp.wait_stream(copy)
        e1.record(comp)
        e1.synchronize()
        return e0.elapsed_time(e1) / reps * 1e-3   # seconds per call

    for name, c in CONFIGS.items():
        if name not in only:
            continue
        kind, n, k = c["scheme"]
        scheme = CodingScheme.reed_solomon(n, k)
        layers, heads, dim, tp = c["geom"]
        cfg = K.ModelConfig(layers, heads, dim, 2, tp)
        m, S, lost = c["m"], c["stripes"], c["lost"]
        e = len(lost)
        ln = K.slice_bytes(cfg, m)
        data = torch.empty((S, n, ln), dtype=torch.uint8, device=dev)
        for s in range(S):
            for j in range(n):
                req, chunk = (s, 0) if c.get("by_request") else (0, s)
                K.make_ground_truth_slice(3, req, chunk, j, cfg, m, m, out=data[s, j])
        h_par = torch.empty((S, k, ln), dtype=torch.uint8).pin_memory()
        par_dev = torch.empty((S, k, ln), dtype=torch.uint8, device=dev)
        enc = encoder(scheme)
        slots = L.ptr_array([data[s, j].data_ptr() for s in range(S) for j in range(n)])
        hout = L.ptr_array([h_par[s, i].data_ptr() for s in range(S) for i in range(k)])
        dout = L.ptr_array([par_dev[s, i].data_ptr() for s in range(S) for i in range(k)])
        big = S * n * ln >= (1 << 30)
        reps = 2 if big else 10

        # encode incl. D2H (gs_encode_offload: K1 into staging, D2H pieces on the copy stream)
        t_off = ev_time(lambda: check(lib.gs_encode_offload(pipe.handle, enc.handle, S, slots, hout, ln,
                                                            comp.cuda_stream, copy.cuda_stream), name), reps)
        t_k1 = ev_time(lambda: check(lib.gs_apply_device(enc.handle, S, slots, dout, ln, comp.cuda_stream),
                                     name), reps)
        # recovery: H2D of the e used parity rows + K2 over the survivors -> fresh buffers
        dec = decoder(scheme, ErasurePattern(lost))
        rebuilt = torch.empty((S, e, ln), dtype=torch.uint8, device=dev)
        rslots = []
        for s in range(S):
            for j in range(n + k):
                if j in lost:
                    rslots.append(None)
                elif j < n:
                    rslots.append(data[s, j].data_ptr())
                else:
                    rslots.append(h_par[s, j - n].data_ptr())
        rslots = L.ptr_array(rslots)
        routs = L.ptr_array([rebuilt[s, b].data_ptr() for s in range(S) for b in range(e)])
        t_rec = ev_time(lambda: check(lib.gs_reconstruct_upload(pipe.handle, dec.handle, S, rslots, routs, ln,
                                                                comp.cuda_stream, copy.cuda_stream), name),
                        reps)
        rec_ok = bool(torch.equal(rebuilt, data[:, lost]))
        dev_ok = bool(torch.equal(par_dev.cpu(), h_par))

        # stripe 0 on the host: bit-exact vs the reference, and the CPU legs
        host = [data[0, j].cpu().numpy() for j in range(n)]
        gpu_p = [h_par[0, i].numpy() for i in range(k)]
        cpu = {"cores": threads, "cpu_model": cpu_model(), "sample": f"stripe 0 ({n} x {ln} B)"}
        exact = None
        if ref is not None:
            rp = [np.zeros(ln, np.uint8) for _ in range(k)]
            t1 = ref.encode_timed(O.RS, n, k, host, rp, 1)
            exact = all(np.array_equal(a, b) for a, b in zip(rp, gpu_p))
            tall = min(ref.encode_timed(O.RS, n, k, host, rp, threads) for _ in range(2))
            cs, t_ck = ref.checkpoint_chunk_timed(O.RS, n, k, (layers, heads, dim), m, 0, 0, m, host, rp)
            sl = list(host) + list(rp)
            for j in lost:
                sl[j] = None
            outs = [np.zeros(ln, np.uint8) for _ in range(e)]
            r1 = ref.reconstruct_timed(O.RS, n, k, sl, lost, outs, 1)
            rall = min(ref.reconstruct_timed(O.RS, n, k, sl, lost, outs, threads) for _ in range(2))
            t_rc = ref.reconstruct_chunk_timed(O.RS, n, k, sl, outs)
            exact = exact and all(np.array_equal(outs[b], host[j]) for b, j in enumerate(lost))
            cpu.update({"kind": "reference",
                        "encode_1t_gbs": round(n * ln / t1 / 1e9, 3),
                        "encode_all_gbs": round(n * ln / tall / 1e9, 3),
                        "checkpoint_chunk_1t_ms": round(t_ck * 1e3, 2),
                        "reconstruct_1t_ms": round(r1 * 1e3, 2), "reconstruct_all_ms": round(rall * 1e3, 2),
                        "reconstruct_chunk_1t_ms": round(t_rc * 1e3, 2),
                        "per_config_ms_1t": {"encode": round(t1 * S * 1e3, 1),
                                             "checkpoint_chunk": round(t_ck * S * 1e3, 1),
                                             "reconstruct_chunk": round(t_rc * S * 1e3, 1)},
                        "note": "per_config = per-chunk time x stripes (the reference runs chunks serially)"})
        fp = None
        if c["fp"]:
            got = tuple(f"{port.fnv1a64(p):016x}" for p in gpu_p)
            fp = {"want": list(c["fp"]), "got": list(got), "ok": got == c["fp"]}

        data_b, par_b = S * n * ln, S * k * ln
        ts_off = max((n + k) * ln * S / (hbm * 1e9), par_b / (link["d2h"] * 1e9))
        ts_k1 = (n + k) * ln * S / (hbm * 1e9)
        ts_rec = max((n + e) * ln * S / (hbm * 1e9), e * ln * S / (link["h2d"] * 1e9))
        line = {"config": name, "workload": c["what"], "scheme": f"RS({n},{k})", "n_gpus": 1,
                "stripes": S, "slice_bytes": ln, "data_bytes": data_b, "parity_bytes": par_b,
                "encode_offload": {"gbs": round(data_b / t_off / 1e9, 2), "ms": round(t_off * 1e3, 3),
                                   "roofline_ms": round(ts_off * 1e3, 3), "frac": round(ts_off / t_off, 4),
                                   "bound": "host link (D2H)" if par_b / link["d2h"] > (n + k) * ln * S / hbm
                                   else "hbm"},
                "k1": {"gbs_hbm": round((n + k) * ln * S / t_k1 / 1e9, 1), "ms": round(t_k1 * 1e3, 3),
                       "frac": round(ts_k1 / t_k1, 4)},
                "recovery": {"lost": lost, "ms": round(t_rec * 1e3, 3), "bytes_rebuilt": S * e * ln,
                             "h2d_bytes": S * e * ln, "roofline_ms": round(ts_rec * 1e3, 3),
                             "frac": round(ts_rec / t_rec, 4), "decoder_specialised": dec.specialised},
                "peaks": {"hbm_gbs": hbm, "hbm_source": hbm_src, "d2h_gbs": link["d2h"], "h2d_gbs": link["h2d"]},
                "cpu_reference": cpu,
                "bit_exact": {"parity_vs_reference_stripe0": exact, "device_parity_eq_offloaded": dev_ok,
                              "rebuilt_eq_original_all_stripes": rec_ok, "fingerprints": fp},
                "timing": f"CUDA events on the compute stream, {reps} back-to-back calls"}
        print(json.dumps(line), flush=True)
        del data, h_par, par_dev, rebuilt
        torch.cuda.empty_cache()
    pipe.close()
