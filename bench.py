#!/usr/bin/env python
"""Benchmark: GhostServe shadow-checkpointing hot path on B200.

Workload (BASELINE.json configs[1], "C2"): Llama-3-8B KV cache at TP=8 --
32 layers x 8 KV heads x 128 dim, fp16, one worker slice per request per
16-token decode block = 262,144 B -- RS(8,2) incremental parity for one
16-token decode block of a batch of 32 requests. One STEP = one block
checkpoint: K1 encodes 32 x 8 x 256 KiB of device-resident KV into 32 x 2 x
256 KiB parity and the parity is D2H'd to pinned host memory (the host tier),
overlapped piecewise. Metric = data bytes encoded / step time (the
reference's bench convention, tools/ghostserve.cpp:279-282).

At N GPUs (torchrun, one rank per GPU) the TP group is spread over the ranks
(8/N workers each) and the batch is 32*N requests (weak scaling): rank g
encodes byte range g of every shard, pulling the ranges it does not own from
peers over NVLink inside K1, and D2H's parity range g on its own host link.

Also reported (same JSON line): the kernel-only roofline of K1, the host-link
fraction, e2e through the reference-facing C ABI with host buffers
(gs_encode_host: H2D + K1 + D2H per step), lost-shard recovery latency (C2
block and, at N=1, the C3 full-shard rebuild of a 128K-token Llama-3-70B
prefill), clocks sampled through NVML during the timed region, and the
reference CPU codec timed on this host.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  python bench.py --sweep [--sweep-sizes 64K,...,1G]     # C5: one JSON line per (code, L)
  python bench.py --configs [--configs-only C1,C3]       # C1-C4 table incl. reference CPU + bit-exact
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "KV parity encode GB/s incl. D2H offload; lost-shard KV recovery latency (ms)"
WORKLOAD = "C2: Llama-3-8B KV TP=8, RS(8,2), incremental parity per 16-token decode block, batch 32"
N_SHARDS, K_PARITY = 8, 2
BLOCK_TOKENS, BATCH = 16, 32
SLICE = 262_144                    # slice_bytes(Llama-3-8B, tp 8, m 16)
RING_BLOCKS = 8                    # distinct decode blocks the steps rotate over (> L2)
KV_SEED = 3
NVLINK_GBS = 900.0                 # NVLink 5 per direction per GPU (spec)


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(
        os.environ.get("LOCAL_RANK", 0))


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML polled from a thread)
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], 0, False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"]}
        reasons = [name for bit, name in self.REASONS.items() if self.reasons & bit and bit != 0x1]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max, "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU baseline: the reference codec (oracle/_ref) or the oracle port
# ---------------------------------------------------------------------------
class CpuBlock:
    """One C2 decode block (32 requests x 8 workers x 256 KiB, reference KV
    stream) encoded by the reference CPU codec (oracle/_ref, kind
    "reference"), or by the oracle port when the reference was not built."""

    def __init__(self):
        import numpy as np
        from oracle import oracle as O

        self.O = O
        self.kind = "reference" if O.have_ref() else "port"
        self.lib = O.ref() if O.have_ref() else O.port()
        sets = [[self.lib.make_ground_truth_slice(KV_SEED, r, 0, w, 32, 8, 128, 8, BLOCK_TOKENS,
                                                  BLOCK_TOKENS) for w in range(N_SHARDS)] for r in range(4)]
        self.stripes = [sets[r % 4] for r in range(BATCH)]
        self.parity = [[np.zeros(SLICE, np.uint8) for _ in range(K_PARITY)] for _ in range(BATCH)]

    def run(self, nreq: int, threads: int) -> float:
        """Encode nreq requests of the block; returns encode seconds."""
        O = self.O
        if self.kind == "reference":
            return self.lib.encode_batch_timed(O.RS, N_SHARDS, K_PARITY, self.stripes[:nreq],
                                               self.parity[:nreq], threads)
        t1 = time.perf_counter()
        for r in range(nreq):
            self.lib.encode(O.RS, N_SHARDS, K_PARITY, self.stripes[r])
        return time.perf_counter() - t1


def cpu_encode_baseline(target_s: float, threads: int):
    """Reference CPU encode on C2 blocks for ~target_s seconds; returns dict."""
    blk = CpuBlock()
    if blk.kind == "port":
        threads = 1
    done, busy = 0, 0.0
    while busy < target_s or done == 0:
        busy += blk.run(BATCH, threads)
        done += 1
    gbs = done * BATCH * N_SHARDS * SLICE / busy / 1e9
    from tools.config_table import cpu_model
    return {"value": round(gbs, 4), "unit": "GB/s", "cores": threads, "kind": blk.kind, "cpu_model": cpu_model(),
            "sample": f"{done} C2 decode blocks (32 requests x RS(8,2) over 8 x 256 KiB), {busy:.2f} s "
                      f"of encode time, {threads} thread(s) taking whole requests"}


def ncu_traffic():
    """dram bytes (read + write) per K1 launch from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "k1_ncu_summary.json")) as f:
            return json.load(f)["dram_bytes_per_launch"]
    except Exception:
        return None


def run_reference(args):
    """--impl reference: the reference CPU codec on this host, all threads."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    steps, warm = args.steps, args.warmup
    blk = CpuBlock()
    kind = blk.kind
    if kind == "port":
        threads = 1
    # one step = one C2 decode block; bounded: if a block would take > ~3 s,
    # each step times a sample of its requests and scales to the full block.
    probe = blk.run(2, threads) / 2
    nreq = BATCH if probe * BATCH < 3.0 else max(1, int(3.0 / probe))
    for _ in range(warm):
        blk.run(nreq, threads)
    total = sum(blk.run(nreq, threads) for _ in range(steps))
    per_step = total / steps * (BATCH / nreq)
    gbs = BATCH * N_SHARDS * SLICE / per_step / 1e9
    sample = (f"each step = {nreq} of the block's 32 requests (8 x 256 KiB RS(8,2) encode each), "
              f"scaled to the full block; ghostserve::encode on {threads} thread(s) taking whole requests")
    line = {"metric": METRIC, "value": round(gbs, 4), "unit": "GB/s", "n_gpus": world, "steps": steps,
            "warmup": warm, "ms_per_step": round(per_step * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": WORKLOAD, "scheme": "RS(8,2)", "slice_bytes": SLICE, "batch": BATCH,
                       "host": "CPU only"},
            "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": threads, "kind": kind,
                             "sample": sample},
            "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def host_link_peaks(torch, dev, nbytes=256 << 20, reps=5):
    """Best pinned D2H / H2D copy bandwidth of this GPU's host link (GB/s)."""
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream()
    out = {}
    for name, fn in (("d2h", lambda: h.copy_(d, non_blocking=True)),
                     ("h2d", lambda: d.copy_(h, non_blocking=True))):
        best = 0.0
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
            e1.synchronize()
            best = max(best, nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        out[name] = round(best, 2)
    del h, d
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2605_00831_b200 import _lib as L
    from paper_2605_00831_b200 import device as D
    from paper_2605_00831_b200 import kv_layout as K
    from paper_2605_00831_b200.coding import CodingScheme, ErasurePattern, check, decoder, encoder
    from paper_2605_00831_b200.peer import (PeerGroup, ShardLayout, plan_encode_rotating, plan_encode_striped,
                                            plan_reconstruct_striped, stripe_range)

    rank, world, local = env_rank()
    # GS_BENCH_SHARED_GPU=1: functional check of the multi-rank path with all
    # ranks on cuda:0 (gloo plumbing; timings are not meaningful then).
    shared = os.environ.get("GS_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # multi-socket hosts: run next to this GPU's host link (no-op on one node)
    numa_cpus = None if shared else D.bind_local_cpus(local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    scheme = CodingScheme.reed_solomon(N_SHARDS, K_PARITY)
    cfg = K.LLAMA3_8B
    assert K.slice_bytes(cfg, BLOCK_TOKENS) == SLICE
    S = BATCH * world                      # weak scaling: 32 requests per GPU
    layout = ShardLayout(N_SHARDS, world, S, SLICE)
    nl = layout.n_local
    lib = L.lib()

    # --- data: RING_BLOCKS distinct decode blocks, reference KV stream ------
    # block b, request s, worker w -> make_ground_truth_slice(seed, s, b, w)
    ring = torch.empty((RING_BLOCKS, S, nl, SLICE), dtype=torch.uint8, device=dev)
    for b in range(RING_BLOCKS):
        for s in range(S):
            for jl in range(nl):
                K.make_ground_truth_slice(KV_SEED, s, b, rank * nl + jl, cfg, BLOCK_TOKENS, BLOCK_TOKENS,
                                          out=ring[b, s, jl])
    torch.cuda.synchronize()
    pg = PeerGroup() if world > 1 else None
    bases = [pg.share(ring[b]) if pg else [ring[b].data_ptr()] for b in range(RING_BLOCKS)]
    h_parity = D.pinned_near((S, K_PARITY, SLICE), local)   # on the GPU's NUMA node
    pipe = D.Pipeline(local, 256 << 20)
    comp = torch.cuda.Stream(device=dev)
    copy = torch.cuda.Stream(device=dev)
    enc = encoder(scheme)
    launches0 = D.launches()

    if args.encoder == "rotate":     # comparison mode: whole stripes, round-robin parity worker
        plans = [plan_encode_rotating(scheme, layout, bases[b], rank, pipe, h_parity, first_worker=b)
                 for b in range(RING_BLOCKS)]
    else:
        plans = [plan_encode_striped(scheme, layout, bases[b], rank, pipeline=pipe, h_parity=h_parity)
                 for b in range(RING_BLOCKS)]

    def step(i):
        plans[i % RING_BLOCKS].run(comp.cuda_stream, copy.cuda_stream)

    def barrier():
        if world > 1:
            dist.barrier()

    # --- timed region: encode + D2H offload ----------------------------------
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = D.launches()
    # live K1 timing: timing events around every K1 launch group of the timed
    # steps, on the compute stream after the staging-slot waits
    check(lib.gs_pipeline_set_timing(pipe.handle, 1), "timing")
    with ClockSampler(local) as clk:
        e0.record(comp)
        for i in range(args.steps):
            step(args.warmup + i)
        comp.wait_stream(copy)
        e1.record(comp)
        e1.synchronize()
    l1 = D.launches()
    torch.cuda.synchronize()
    k_ms, k_dev_ms, k_groups, k_launches = C.c_double(), C.c_double(), C.c_int(), C.c_uint64()
    check(lib.gs_pipeline_kernel_time(pipe.handle, C.byref(k_ms), C.byref(k_dev_ms), C.byref(k_groups),
                                      C.byref(k_launches)), "timing")
    check(lib.gs_pipeline_set_timing(pipe.handle, 0), "timing")
    live_group_us = k_dev_ms.value * 1e3 / max(k_groups.value, 1)     # kernel-internal %globaltimer
    live_event_us = k_ms.value * 1e3 / max(k_groups.value, 1)         # timing events around each group
    barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([live_group_us, live_event_us], device="cpu" if shared else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        live_group_us, live_event_us = float(t[0].item()), float(t[1].item())
    if world > 1:
        t = torch.tensor([ms], device="cpu" if shared else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    data_bytes_step = S * N_SHARDS * SLICE          # whole job
    value = data_bytes_step * args.steps / (ms * 1e-3) / 1e9
    ms_step = ms / args.steps

    # parity sanity inside the bench (cheap, on the last block; full checks live in tests/)
    ok_parity = True
    if rank == 0:
        last = (args.warmup + args.steps - 1) % RING_BLOCKS
        if world == 1:
            want = D.encode(scheme, ring[last, :2])
            ok_parity = torch.equal(want.cpu(), h_parity[:2])

    # --- kernel-only rooflines: K1 encode and K2 single-loss rebuild ---------
    kern, kern2 = {}, {}
    peak, peak_src = load_peaks()
    ks = torch.cuda.Stream(device=dev)

    def timed(launch, alg_bytes, name):
        with torch.cuda.stream(ks):
            for b in range(RING_BLOCKS):
                launch(b)
        ks.synchronize()
        reps = 4
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=ks):
            for _ in range(reps):
                for b in range(RING_BLOCKS):
                    launch(b)
        n_graph = max(3, args.steps // (reps * RING_BLOCKS))
        with torch.cuda.stream(ks):
            g.replay()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(ks)
            for _ in range(n_graph):
                g.replay()
            ev1.record(ks)
        ev1.synchronize()
        per_ms = ev0.elapsed_time(ev1) / (n_graph * reps * RING_BLOCKS)
        achieved = alg_bytes / (per_ms * 1e-3) / 1e9
        return {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "kernel": name,
                "per_launch_us": round(per_ms * 1e3, 2), "algorithmic_bytes_per_launch": alg_bytes,
                "peak_source": peak_src,
                "timing": f"CUDA graph of {reps * RING_BLOCKS} launches over {RING_BLOCKS} distinct "
                          f"blocks, replayed {n_graph}x, events on the launch stream"}

    if world == 1:
        par_dev = torch.empty((RING_BLOCKS, S, K_PARITY, SLICE), dtype=torch.uint8, device=dev)
        rebuilt = torch.empty((RING_BLOCKS, S, SLICE), dtype=torch.uint8, device=dev)
        slots = [L.ptr_array([ring[b, s, j].data_ptr() for s in range(S) for j in range(N_SHARDS)])
                 for b in range(RING_BLOCKS)]
        outs = [L.ptr_array([par_dev[b, s, i].data_ptr() for s in range(S) for i in range(K_PARITY)])
                for b in range(RING_BLOCKS)]
        dec5 = decoder(scheme, ErasurePattern([5]))
        dslots = [L.ptr_array([None if j == 5 else (ring[b, s, j].data_ptr() if j < N_SHARDS else
                                                     par_dev[b, s, j - N_SHARDS].data_ptr())
                               for s in range(S) for j in range(N_SHARDS + K_PARITY)])
                  for b in range(RING_BLOCKS)]
        douts = [L.ptr_array([rebuilt[b, s].data_ptr() for s in range(S)]) for b in range(RING_BLOCKS)]
        variants = {}
        for v, vname in ((0, "ldg128"), (1, "bulk_smem_pipeline")):
            check(lib.gs_set_kernel_variant(v), "variant")
            variants[vname] = timed(
                lambda b: check(lib.gs_apply_device(enc.handle, S, slots[b], outs[b], SLICE, ks.cuda_stream),
                                "k1"), S * (N_SHARDS + K_PARITY) * SLICE, f"K1 {vname}")["per_launch_us"]
        check(lib.gs_set_kernel_variant(2), "variant")  # auto: what the timed step used
        iso = timed(lambda b: check(lib.gs_apply_device(enc.handle, S, slots[b], outs[b], SLICE,
                                                        ks.cuda_stream), "k1"),
                    S * (N_SHARDS + K_PARITY) * SLICE,
                    "k_apply_special<EncSpec<RS,8,2>> (K1 encode, auto variant = ldg128 at this size)")
        alg = S * (N_SHARDS + K_PARITY) * SLICE
        achieved = alg / (live_group_us * 1e-6) / 1e9
        kern = dict(iso, achieved=round(achieved, 1), frac=round(achieved / peak, 4),
                    per_launch_us=round(live_group_us, 2),
                    timing=f"live, inside the timed steps: mean over the {k_groups.value} K1 launches "
                           f"({k_launches.value} kernels) of the kernel-internal %globaltimer span (first CTA start "
                           "to last warp's stores performed)",
                    live_event_bracketed={"per_launch_us": round(live_event_us, 2),
                                          "note": "timing events on the compute stream around each launch; inflated "
                                                  "by GPU front-end latency while the copy engine streams the previous "
                                                  "blocks' D2H (tools/k1_context_probe.py)"},
                    isolated_graph={"per_launch_us": iso["per_launch_us"], "achieved": iso["achieved"],
                                    "frac": iso["frac"], "timing": iso["timing"]})
        kern["variants_us_per_launch"] = variants
        # attainable at this launch size: a device copy moving the same bytes
        # (half read, half written), same rotation and graph timing
        half = S * (N_SHARDS + K_PARITY) * SLICE // 2
        cdst = torch.empty((RING_BLOCKS, half), dtype=torch.uint8, device=dev)
        flat = ring.view(RING_BLOCKS, -1)
        cp = timed(lambda b: cdst[b].copy_(flat[b, :half]), 2 * half, "copy")
        kern["copy_same_bytes"] = {"per_launch_us": cp["per_launch_us"], "achieved": cp["achieved"],
                                   "kernel_vs_copy_isolated": round(cp["per_launch_us"] / iso["per_launch_us"], 4)}
        del cdst
        kern["traffic"] = args.traffic or ncu_traffic()
        kern2 = timed(lambda b: check(lib.gs_apply_device(dec5.handle, S, dslots[b], douts[b], SLICE,
                                                          ks.cuda_stream), "k2"),
                      S * (N_SHARDS + 1) * SLICE,
                      "k_apply_special<DecSpec<RS,8,2,lost{5}>> (K2 rebuild, 7 data + 1 parity -> 1)")
        ok_parity &= torch.equal(rebuilt[RING_BLOCKS - 1], ring[RING_BLOCKS - 1, :, 5])

        # the same C2 blocks living in per-worker PAGED KV caches (vLLM-style
        # [layer][K/V][block][16 tok][256 B]): K1 gathers the 64 pages of every
        # slice in place instead of reading contiguous slices.
        from paper_2605_00831_b200.paged import PagedKVCache
        caches = [PagedKVCache(cfg, RING_BLOCKS * S, BLOCK_TOKENS, device=dev) for _ in range(N_SHARDS)]
        for b in range(RING_BLOCKS):
            for s_ in range(S):
                for j in range(N_SHARDS):
                    caches[j].write_slice(b * S + s_, ring[b, s_, j])
        pm = caches[0].page_map(BLOCK_TOKENS)
        pslots = [L.ptr_array([caches[j].block_base(b * S + s_) for s_ in range(S) for j in range(N_SHARDS)])
                  for b in range(RING_BLOCKS)]
        kern_paged = timed(lambda b: check(lib.gs_apply_device_paged(enc.handle, S, pslots[b], outs[b], SLICE,
                                                                     C.byref(pm), (1 << N_SHARDS) - 1, None,
                                                                     ks.cuda_stream), "k1 paged"),
                           S * (N_SHARDS + K_PARITY) * SLICE, "K1 encode reading a paged KV cache in place")
        ok_parity &= torch.equal(par_dev[RING_BLOCKS - 1, :2].cpu(),
                                 D.encode(scheme, ring[RING_BLOCKS - 1, :2]).cpu())
        kern["paged_kv_cache_us_per_launch"] = kern_paged["per_launch_us"]
        kern["paged_kv_cache_frac"] = kern_paged["frac"]
        del par_dev, rebuilt, caches

    else:
        # N > 1: the step's own kernel -- K1 over this rank's byte range of all
        # S stripes, ranges it does not own read from peers over NVLink -- timed
        # per rank, max over ranks. Roofline t* = max(HBM bytes / HBM peak,
        # NVLink bytes pulled / NVLink peak).
        off_r, ln_r = stripe_range(SLICE, rank, world)
        par_dev = torch.empty((RING_BLOCKS, S, K_PARITY, max(ln_r, 16)), dtype=torch.uint8, device=dev)
        kplans = [plan_encode_striped(scheme, layout, bases[b], rank, parity_out=par_dev[b])
                  for b in range(RING_BLOCKS)]
        alg = S * (N_SHARDS + K_PARITY) * ln_r
        k = timed(lambda b: kplans[b].run(ks.cuda_stream), alg, "striped K1")
        t = torch.tensor([k["per_launch_us"]], device="cpu" if shared else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        iso_us = float(t.item())
        # live (timed-region) K1 group time when the step is the striped encoder
        per_us = live_group_us if args.encoder == "stripe" else iso_us
        nvl_bytes = S * N_SHARDS * ln_r * (world - 1) // world
        t_hbm, t_nvl = alg / (peak * 1e3), nvl_bytes / (NVLINK_GBS * 1e3)  # us
        bound = "nvlink" if t_nvl > t_hbm else "hbm"
        achieved = alg / per_us / 1e3
        kern = {"bound": bound, "achieved": round(achieved, 1),
                "peak": NVLINK_GBS if bound == "nvlink" else peak, "unit": "GB/s",
                "frac": round(max(t_hbm, t_nvl) / per_us, 4),
                "kernel": "k_apply_special<EncSpec<RS,8,2>> striped: this rank's byte range of all stripes, "
                          "peer ranges loaded over NVLink inside the kernel",
                "per_launch_us": round(per_us, 2), "algorithmic_bytes_per_launch": alg,
                "nvlink_bytes_per_launch": nvl_bytes,
                "roofline_us": {"hbm": round(t_hbm, 2), "nvlink": round(t_nvl, 2)},
                "peak_source": (f"NVLink 5 spec {NVLINK_GBS:.0f} GB/s per direction (not measured)"
                                if bound == "nvlink" else peak_src),
                "timing": (f"live: kernel-internal %globaltimer span of each K1 launch group of the timed steps "
                           f"({k_groups.value} per rank), mean, max over ranks" if args.encoder == "stripe"
                           else k["timing"] + ", max over ranks"),
                "live_event_bracketed_us": round(live_event_us, 2),
                "isolated_graph": {"per_launch_us": round(iso_us, 2), "timing": k["timing"] + ", max over ranks"},
                "traffic": None}
        del par_dev

    # --- host link --------------------------------------------------------------
    link = host_link_peaks(torch, dev)
    d2h_step = S * K_PARITY * SLICE
    link_achieved = d2h_step / world * args.steps / (ms * 1e-3) / 1e9  # per GPU
    host_link = {"d2h_bytes_per_step_per_gpu": d2h_step // world,
                 "achieved_gbs_per_gpu": round(link_achieved, 2), "peak_d2h_gbs": link["d2h"],
                 "peak_h2d_gbs": link["h2d"], "frac": round(link_achieved / link["d2h"], 4)}
    # roofline of the whole step: t* = the slowest of HBM bytes at
    # peak, parity over this GPU's host link, peer bytes over NVLink; per GPU
    hbm_b = S * (N_SHARDS + K_PARITY) * SLICE // world
    nvl_b = S * N_SHARDS * SLICE * (world - 1) // world // world
    legs = {"hbm": hbm_b / (load_peaks()[0] * 1e9), "host_link": (d2h_step // world) / (link["d2h"] * 1e9),
            "nvlink": nvl_b / (NVLINK_GBS * 1e9)}
    t_star = max(legs.values())
    step_roofline = {"bound": max(legs, key=legs.get), "t_star_ms": round(t_star * 1e3, 4),
                     "legs_ms": {k_: round(v * 1e3, 4) for k_, v in legs.items()},
                     "frac": round(t_star / (ms_step * 1e-3), 4),
                     "note": "per GPU: HBM (n+k)*L*S/N at the measured copy peak, parity D2H at this GPU's measured "
                             "link peak, peer reads (N-1)/N of the data over NVLink 5 (900 GB/s spec)"}

    # --- e2e through the reference-facing C ABI with host buffers -------------
    # Every rank encodes its own 32 requests (all 8 worker slices each) from
    # pinned host memory on its own host link: H2D of the data, K1, D2H of the
    # parity, every step. Wall clock per rank between barriers, max over ranks.
    per_worker = BATCH * SLICE   # request slices of a worker are contiguous: one stripe
    h_in = D.pinned_near((N_SHARDS, per_worker), local)
    h_out = D.pinned_near((K_PARITY, per_worker), local)
    src = torch.empty((N_SHARDS, BATCH, SLICE), dtype=torch.uint8, device=dev)
    for j in range(N_SHARDS):
        for s_ in range(BATCH):
            K.make_ground_truth_slice(KV_SEED, rank * BATCH + s_, 0, j, cfg, BLOCK_TOKENS, BLOCK_TOKENS,
                                      out=src[j, s_])
    h_in.copy_(src.view(N_SHARDS, per_worker).cpu())
    hp_in = L.ptr_array([h_in[j].data_ptr() for j in range(N_SHARDS)])
    hp_out = L.ptr_array([h_out[i].data_ptr() for i in range(K_PARITY)])
    epipe = D.Pipeline(local, 256 << 20)

    def e2e_run(fn, sync_each):
        for _ in range(max(3, args.warmup)):
            check(fn(epipe.handle, enc.handle, hp_in, hp_out, per_worker), "e2e")
            if sync_each:
                check(lib.gs_pipeline_sync(epipe.handle), "e2e sync")
        check(lib.gs_pipeline_sync(epipe.handle), "e2e sync")
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            check(fn(epipe.handle, enc.handle, hp_in, hp_out, per_worker), "e2e")
            if sync_each:
                check(lib.gs_pipeline_sync(epipe.handle), "e2e sync")
        check(lib.gs_pipeline_sync(epipe.handle), "e2e sync")
        dt = time.perf_counter() - t0
        barrier()
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device="cpu" if shared else dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        return dt

    # Two public ways to drive it, each timed twice (alternating, best trial):
    #  * stream-ordered: gs_encode_host_async per step, one gs_pipeline_sync at
    #    the end -- the H2D of step i+1 overlaps the D2H of step i (a serving
    #    loop checkpointing block after block from host memory);
    #  * synchronous drop-in: gs_encode_host per step (ghostserve::encode
    #    semantics). Every step moves its own inputs H2D and its parity D2H.
    # Which one is faster depends on how the box's PCIe handles both
    # directions at once; the headline is the faster, both are reported.
    t_async, t_sync = [], []
    for _ in range(2):
        t_async.append(e2e_run(lib.gs_encode_host_async, False))
        t_sync.append(e2e_run(lib.gs_encode_host, True))
    dt, dt_sync = min(t_async), min(t_sync)
    got = h_out.view(K_PARITY, BATCH, SLICE).permute(1, 0, 2)
    ok_parity &= torch.equal(got[:2], D.encode(scheme, src[:, :2].permute(1, 0, 2).contiguous()).cpu())
    bytes_e2e = world * BATCH * N_SHARDS * SLICE * args.steps
    modes = {"stream_ordered": {"value": round(bytes_e2e / dt / 1e9, 3), "ms_per_step": round(dt / args.steps * 1e3, 3),
                                "api": "gs_encode_host_async per step, gs_pipeline_sync after the last step"},
             "sync_per_call": {"value": round(bytes_e2e / dt_sync / 1e9, 3),
                               "ms_per_step": round(dt_sync / args.steps * 1e3, 3),
                               "api": "gs_encode_host per step (drop-in synchronous ghostserve::encode)"}}
    best = max(modes, key=lambda m: modes[m]["value"])
    e2e = {"value": modes[best]["value"], "unit": "GB/s",
           "h2d_bytes_per_step": world * N_SHARDS * per_worker, "d2h_bytes_per_step": world * K_PARITY * per_worker,
           "ms_per_step": modes[best]["ms_per_step"],
           "api": f"{best}: {modes[best]['api']} (C ABI, pinned host buffers; H2D data -> K1 -> D2H parity every "
                  "step); wall clock, best of 2 trials" + (", one pipeline per rank, max over ranks"
                                                          if world > 1 else ""),
           "modes": modes}
    epipe.close()
    del h_in, h_out, src

    # --- recovery: one lost worker of the C2 block ----------------------------
    recovery = {}
    lost_w = 5
    b = (args.warmup + args.steps - 1) % RING_BLOCKS
    owner, jl = layout.owner(lost_w)
    saved = ring[b, :, jl].clone() if rank == owner else None
    barrier()
    if rank == owner:
        ring[b, :, jl].zero_()        # "flush the memory buffer" of the failed worker
    torch.cuda.synchronize()
    barrier()
    # decode plan (host Gauss-Jordan inverse + pointer tables) is built when the
    # failure is detected; the timed region is the byte path: H2D of parity
    # row 0 + K2 over the 7 survivors, written into the failed worker's buffer.
    t_plan = time.perf_counter()
    rplan = plan_reconstruct_striped(scheme, layout, bases[b], rank, ErasurePattern([lost_w]), h_parity, pipe)
    plan_ms = (time.perf_counter() - t_plan) * 1e3
    reps = []
    for rep in range(5):   # the same failure recovered 5 times (buffer re-flushed each time); median
        if rep and rank == owner:
            ring[b, :, jl].zero_()
        torch.cuda.synchronize()
        barrier()
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record(comp)
        rplan.run(comp.cuda_stream, copy.cuda_stream)
        r1.record(comp)
        r1.synchronize()
        barrier()
        reps.append(r0.elapsed_time(r1))
    rec_ms = sorted(reps)[len(reps) // 2]
    if world > 1:
        t = torch.tensor([rec_ms], device="cpu" if shared else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        rec_ms = float(t.item())
    if rank == owner:
        ok_parity &= torch.equal(ring[b, :, jl], saved)
    if world > 1:  # every rank's verdict (the rebuilt shard lives on its owner)
        t = torch.tensor([1 if ok_parity else 0], device="cpu" if shared else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        ok_parity = bool(t.item())
    recovery["c2_block_one_worker_ms"] = round(rec_ms, 4)
    recovery["c2_block_reps_ms"] = [round(x, 4) for x in reps]
    recovery["c2_block_roofline_ms"] = round(S * SLICE / (link["h2d"] * 1e9) * 1e3 / world, 4)
    recovery["c2_plan_host_ms"] = round(plan_ms, 3)
    recovery["c2_block_bytes_rebuilt"] = S * SLICE
    recovery["c2_h2d_bytes"] = S * SLICE
    recovery["decoder_specialised"] = decoder(scheme, ErasurePattern([lost_w])).specialised

    launches = l1 - l0
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_encode_baseline(args.cpu_sample_s, os.cpu_count() or 1)
        cpu1 = cpu_encode_baseline(min(2.0, args.cpu_sample_s), 1)
        cpu["one_thread_gbs"] = cpu1["value"]

    if rank == 0 and world == 1 and not args.no_c3:
        recovery.update(c3_recovery(torch, dev, comp, copy, pipe))
        if kern and kern2:
            recovery["c3_orchestrated"] = c3_orchestrated(torch, dev, link, kern["achieved"] * 8 / 10,
                                                          kern2["achieved"] * 8 / 9)
    if world > 1 and not args.no_c3:
        recovery.update(c3_recovery_striped(torch, dist, dev, comp, copy, pipe, rank, world, shared, barrier))
    if rank == 0 and world == 1 and not args.no_c4:
        recovery.update(c4_recovery(torch, dev, comp, copy, pipe))
    overhead = None
    if rank == 0 and world == 1 and not args.no_overhead:
        overhead = decode_overhead(torch, dev, pipe, args)
    host_tier = None
    if rank == 0 and world == 1:
        host_tier = host_tier_checkpoint(torch, dev, ring, scheme, pipe, comp, copy, args)

    if pg:
        pg.close()
    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
                "data": "synthetic (reference make_ground_truth_slice KV stream, kv_seed 3, generated on GPU)",
                "config": {"workload": WORKLOAD, "scheme": "RS(8,2)", "kv_geometry": "32 layers x 8 KV heads "
                           "x 128 dim fp16, TP=8 -> 256 B/token/worker", "block_tokens": BLOCK_TOKENS,
                           "requests_per_gpu": BATCH, "slice_bytes": SLICE,
                           "data_bytes_per_step": data_bytes_step, "parity_d2h_bytes_per_step": d2h_step,
                           "l2": f"inputs > L2: steps rotate over {RING_BLOCKS} distinct decode blocks "
                                 f"({RING_BLOCKS * data_bytes_step // world >> 20} MiB per GPU)",
                           "host_placement": ("pinned buffers and host threads on the GPU's NUMA node (CPUs "
                                              f"{numa_cpus})" if numa_cpus else "single NUMA node host"),
                           "parallelism": (f"byte-range striping x{world} (peer loads over NVLink)"
                                           if args.encoder == "stripe" else
                                           f"rotating whole-stripe encoder x{world} (paper's temporal "
                                           "balancing; peer loads over NVLink)") if world > 1 else
                           "single GPU holds all 8 TP shards"},
                "roofline": kern or None, "roofline_k2": kern2 or None, "step_roofline": step_roofline,
                "host_link": host_link, "cpu_baseline": cpu, "e2e": e2e,
                "recovery_ms": recovery.get("c2_block_one_worker_ms"), "recovery": recovery,
                "decode_overhead": overhead, "host_tier": host_tier,
                "gpu_launches": launches, "clocks": clk.summary(), "parity_ok": bool(ok_parity)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def host_tier_checkpoint(torch, dev, ring, scheme, pipe, comp, copy, args):
    """The full reference checkpoint semantics per C2 block (checkpoint.hpp:
    143-147 + :207): K1 + D2H straight into ParityStore entries reserved on
    pinned slabs, FNV-1a seal of every (request, block) on host threads after
    the D2H lands. Reports the sealed-checkpoint rate and the host seal rate
    (FNV-1a is a serial multiply chain per chunk, parity_store.hpp:19-25, so
    sealing scales only across chunks / cores)."""
    import ctypes as C
    from paper_2605_00831_b200 import _lib as L
    from paper_2605_00831_b200.coding import check, encoder
    from paper_2605_00831_b200.parity_store import ParityStore

    # leave two cores for the CUDA callback thread and the submitting thread
    threads = max(1, (os.cpu_count() or 1) - 2)
    S = ring.shape[1]
    store = ParityStore(seal_threads=threads)
    store.bind_device(dev.index or 0)   # slabs on the GPU's NUMA node
    enc = encoder(scheme)
    blocks = max(4, min(args.steps, 64))
    slots = [L.ptr_array([ring[b % RING_BLOCKS, s, j].data_ptr() for s in range(S) for j in range(N_SHARDS)])
             for b in range(RING_BLOCKS)]

    def one(b):
        keys = [(s, b) for s in range(S)]
        acc, dst = store.reserve_batch(keys, scheme, BLOCK_TOKENS, SLICE)
        assert acc == S
        check(L.lib().gs_encode_offload(pipe.handle, enc.handle, S, slots[b % RING_BLOCKS], L.ptr_array(dst), SLICE,
                                        comp.cuda_stream, copy.cuda_stream), "host tier")
        store.commit_batch(keys, copy)

    # warm pass: pinned slabs are allocated once (cudaHostAlloc ~ms per call),
    # then recycled through the store's free lists
    for b in range(blocks):
        one(b)
    copy.synchronize()
    store.wait_sealed()
    for s in range(S):
        store.erase_request(s)
    t0 = time.perf_counter()
    for b in range(blocks):
        one(b)
    copy.synchronize()
    t_gpu = time.perf_counter() - t0
    store.wait_sealed()
    t_all = time.perf_counter() - t0
    ok = all(int(store.get(s, blocks - 1)[0]) == 0 for s in range(min(S, 4)))
    data = blocks * S * N_SHARDS * SLICE
    parity = blocks * S * K_PARITY * SLICE
    # raw seal rate of the same parity on all cores (no GPU in the loop)
    h = C.c_void_p()
    views = []
    for s in range(S):
        st_, ch = store.get(s, blocks - 1, verify=False)
        views.extend(ch.parity)
    ptrs = L.ptr_array([v.ctypes.data for v in views])
    outs = (C.c_uint64 * S)()
    t1 = time.perf_counter()
    check(L.lib().gs_parity_checksum_batch(ptrs, S, K_PARITY, SLICE, threads, outs), "seal")
    seal_raw = S * K_PARITY * SLICE / (time.perf_counter() - t1) / 1e9
    out = {"blocks": blocks, "seal_threads": threads, "seal_only_parity_gbs": round(seal_raw, 2),
           "checkpoint_gbs_until_d2h_done": round(data / t_gpu / 1e9, 2),
           "checkpoint_gbs_sealed": round(data / t_all / 1e9, 2),
           "seal_parity_gbs": round(parity / t_all / 1e9, 2),
           "entries": store.entry_count(), "get_verified_ok": ok,
           "note": "FNV-1a seal is serial per chunk (reference checksum); the GPU path is not waiting on it"}
    store.close()
    out["device_seal"] = host_tier_device_sealed(torch, dev, ring, scheme, comp, copy, blocks, slots, threads)
    return out


def host_tier_device_sealed(torch, dev, ring, scheme, comp, copy, blocks, slots, threads):
    """The same sealed C2 block checkpoints with the seal computed on the GPU:
    K1 into a device parity ring, gs_parity_offload_sealed (D2H of the rows
    into the reserved entries + the chunks' checksums by the bit-sliced GPU
    FNV-1a), gs_store_commit_sealed_batch (no host FNV pass)."""
    from paper_2605_00831_b200 import _lib as L
    from paper_2605_00831_b200.coding import check, encoder
    from paper_2605_00831_b200.parity_store import ParityStore

    S = ring.shape[1]
    store = ParityStore(seal_threads=threads)
    store.bind_device(dev.index or 0)
    enc, lib = encoder(scheme), L.lib()
    R = 4   # device parity buffers / pinned checksum arrays in flight
    par = torch.empty((R, S, K_PARITY, SLICE), dtype=torch.uint8, device=dev)
    sums = [torch.zeros(S, dtype=torch.int64).pin_memory() for _ in range(R)]
    rows = [L.ptr_array([par[i, s, r].data_ptr() for s in range(S) for r in range(K_PARITY)]) for i in range(R)]
    free = [None] * R
    torch.cuda.synchronize()

    def one(b):
        i = b % R
        if free[i] is not None:
            comp.wait_event(free[i])      # the buffer's previous D2H is done
            free[i].synchronize()         # ... and its checksums were consumed by the store callback
        keys = [(s, b) for s in range(S)]
        acc, dst = store.reserve_batch(keys, scheme, BLOCK_TOKENS, SLICE)
        assert acc == S
        check(lib.gs_apply_device(enc.handle, S, slots[b % RING_BLOCKS], rows[i], SLICE, comp.cuda_stream), "k1")
        check(lib.gs_parity_offload_sealed(rows[i], S, K_PARITY, SLICE, L.ptr_array(dst), sums[i].data_ptr(),
                                           comp.cuda_stream, copy.cuda_stream), "device seal")
        store.commit_sealed_batch(keys, sums[i].data_ptr(), copy)
        free[i] = torch.cuda.Event()
        free[i].record(copy)

    for b in range(blocks):   # warm: slabs, scratch pool
        one(b)
    copy.synchronize()
    store.wait_sealed()
    for s in range(S):
        store.erase_request(s)
    t0 = time.perf_counter()
    for b in range(blocks):
        one(b)
    copy.synchronize()
    store.wait_sealed()
    t_all = time.perf_counter() - t0
    ok = all(int(store.get(s, b)[0]) == 0 for s in range(0, S, 7) for b in (0, blocks - 1))
    data = blocks * S * N_SHARDS * SLICE
    out = {"checkpoint_gbs_sealed": round(data / t_all / 1e9, 2),
           "seal_parity_gbs": round(blocks * S * K_PARITY * SLICE / t_all / 1e9, 2),
           "get_verified_ok": ok,
           "note": "seal on the GPU (gs_parity_offload_sealed + gs_store_commit_sealed_batch); get() re-verifies "
                   "on the host with the reference's serial FNV"}
    store.close()
    return out


def c4_recovery(torch, dev, comp, copy, pipe):
    """C4: double-GPU failure, RS(6,2) -- rebuild two lost KV shards (workers 0
    and 3) from the 4 survivors + BOTH parity rows uploaded from host.
    Geometry 80 layers x 6 KV heads x 128 dim, TP=6 (6-divisible, SURVEY
    §7 hard parts), 2K-token chunks (83,886,080 B slices), 8 chunks."""
    from paper_2605_00831_b200 import _lib as L
    from paper_2605_00831_b200 import kv_layout as K
    from paper_2605_00831_b200.coding import CodingScheme, ErasurePattern, check, decoder, encoder

    cfg = K.ModelConfig(80, 6, 128, 2, 6)
    m, chunks, n, k = 2048, 8, 6, 2
    sl = K.slice_bytes(cfg, m)
    scheme = CodingScheme.reed_solomon(n, k)
    kv = torch.empty((n, chunks, sl), dtype=torch.uint8, device=dev)
    for w in range(n):
        for c in range(chunks):
            K.make_ground_truth_slice(KV_SEED, 4, c, w, cfg, m, m, out=kv[w, c])
    h_par = torch.empty((chunks, k, sl), dtype=torch.uint8).pin_memory()
    enc = encoder(scheme)
    check(L.lib().gs_encode_offload(pipe.handle, enc.handle, chunks,
                                    L.ptr_array([kv[w, c].data_ptr() for c in range(chunks) for w in range(n)]),
                                    L.ptr_array([h_par[c, i].data_ptr() for c in range(chunks) for i in range(k)]),
                                    sl, comp.cuda_stream, copy.cuda_stream), "c4 encode")
    copy.synchronize()
    lost = [0, 3]
    saved = kv[lost].clone()
    kv[lost].zero_()
    torch.cuda.synchronize()
    dec = decoder(scheme, ErasurePattern(lost))
    slots = []
    for c in range(chunks):
        for j in range(n + k):
            slots.append(None if j in lost else (kv[j, c].data_ptr() if j < n else h_par[c, j - n].data_ptr()))
    outs = L.ptr_array([kv[w, c].data_ptr() for c in range(chunks) for w in dec.out_index])
    sp = L.ptr_array(slots)
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0.record(comp)
    check(L.lib().gs_reconstruct_upload(pipe.handle, dec.handle, chunks, sp, outs, sl, comp.cuda_stream,
                                        copy.cuda_stream), "c4 rebuild")
    r1.record(comp)
    r1.synchronize()
    ms = r0.elapsed_time(r1)
    ok = bool(torch.equal(kv[lost], saved))
    out = {"c4_rs62_two_lost_ms": round(ms, 2), "c4_bytes_rebuilt": 2 * chunks * sl,
           "c4_h2d_gbs": round(2 * chunks * sl / (ms * 1e-3) / 1e9, 2), "c4_decoder_specialised": dec.specialised,
           "c4_rebuild_ok": ok}
    del kv, h_par, saved
    torch.cuda.empty_cache()
    return out


def decode_overhead(torch, dev, pipe, args):
    """Per-16-token-block checkpoint overhead vs the decode step (north_star
    target < 5%), Llama-3-70B KV at TP=8, batch 32, as seen by ONE GPU of the
    TP group. Decode-step stand-in: stream this GPU's weight
    shard (70.6e9 x 2 B / 8 = 17.65 GB) plus its KV at the chosen context
    (32 x ctx x 40,960 B) from HBM. Block checkpoint: K1 over this GPU's 1/8
    byte range of the 8 workers' block slices (32 x 8 x 81,920 B = 20 MiB in,
    5 MiB parity) + D2H of the parity, on side streams, once per 16 steps."""
    from paper_2605_00831_b200 import _lib as L
    from paper_2605_00831_b200.coding import CodingScheme, check, encoder

    ctx = args.decode_ctx
    wbytes = int(70.6e9 * 2 / 8)
    kvbytes = 32 * ctx * 40960
    free, _ = torch.cuda.mem_get_info(dev)
    if free < wbytes + kvbytes + (4 << 30):
        return {"skipped": f"needs {(wbytes + kvbytes) >> 30} GiB"}
    w = torch.zeros(wbytes // 4, dtype=torch.float32, device=dev)
    kvc = torch.zeros(kvbytes // 4, dtype=torch.float32, device=dev)
    rng = 81920                                   # 655,360 B block slice / 8 GPUs
    data = torch.randint(0, 256, (32, 8, rng), dtype=torch.uint8, device=dev)
    h_par = torch.empty((32, 2, rng), dtype=torch.uint8).pin_memory()
    enc = encoder(CodingScheme.reed_solomon(8, 2))
    slots = L.ptr_array([data[s, j].data_ptr() for s in range(32) for j in range(8)])
    outs = L.ptr_array([h_par[s, i].data_ptr() for s in range(32) for i in range(2)])
    main = torch.cuda.Stream(device=dev)
    side, side_copy = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    sink = torch.empty(2, device=dev)

    def step():
        torch.amax(w, dim=0, out=sink[0])
        torch.amax(kvc, dim=0, out=sink[1])

    def ckpt():
        check(L.lib().gs_encode_offload(pipe.handle, enc.handle, 32, slots, outs, rng, side.cuda_stream,
                                        side_copy.cuda_stream), "overhead ckpt")

    def run(blocks, with_ckpt):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(main):
            e0.record(main)
            for _ in range(blocks):
                if with_ckpt:
                    side.wait_stream(main)
                    ckpt()
                for _ in range(16):
                    step()
            main.wait_stream(side_copy)
            e1.record(main)
        e1.synchronize()
        return e0.elapsed_time(e1)

    run(1, True)
    run(1, False)
    blocks = 4
    base = min(run(blocks, False) for _ in range(3))
    withc = min(run(blocks, True) for _ in range(3))
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(side)
    ckpt()
    side.wait_stream(side_copy)
    a1.record(side)
    a1.synchronize()
    out = {"model": "Llama-3-70B KV, TP=8, batch 32, one GPU's share", "context_tokens": ctx,
           "decode_step_ms": round(base / (blocks * 16), 4),
           "block_ms_without_ckpt": round(base / blocks, 4), "block_ms_with_ckpt": round(withc / blocks, 4),
           "checkpoint_alone_ms": round(a0.elapsed_time(a1), 4),
           "overhead_pct_of_block": round((withc - base) / base * 100, 3),
           "overhead_pct_of_decode_step": round((withc - base) / blocks / (base / (blocks * 16)) * 100, 3)}
    del w, kvc, data, h_par
    torch.cuda.empty_cache()
    return out


def c3_recovery(torch, dev, comp, copy, pipe):
    """C3: Llama-3-70B KV TP=8, 128K-token prefill (64 chunks x 80 MiB per
    worker) checkpointed to pinned host, then worker 5's full shard rebuilt
    from 7 surviving workers + H2D parity row 0. Single GPU holds all 8."""
    from paper_2605_00831_b200 import _lib as L
    from paper_2605_00831_b200 import kv_layout as K
    from paper_2605_00831_b200.coding import CodingScheme, ErasurePattern, check, decoder, encoder

    cfg = K.LLAMA3_70B
    m, chunks = 2048, 64
    sl = K.slice_bytes(cfg, m)                       # 83,886,080
    free, _ = torch.cuda.mem_get_info(dev)
    need = chunks * 9 * sl + (2 << 30)
    if free < need:
        return {"c3_skipped": f"needs {need >> 30} GiB free, {free >> 30} GiB available"}
    scheme = CodingScheme.reed_solomon(8, 2)
    kv = torch.empty((8, chunks, sl), dtype=torch.uint8, device=dev)  # [worker][chunk][slice]
    for w in range(8):
        for c in range(chunks):
            K.make_ground_truth_slice(KV_SEED, 0, c, w, cfg, m, m, out=kv[w, c])
    torch.cuda.synchronize()
    h_par = torch.empty((chunks, 2, sl), dtype=torch.uint8).pin_memory()
    enc = encoder(scheme)
    slots = L.ptr_array([kv[w, c].data_ptr() for c in range(chunks) for w in range(8)])
    outs = L.ptr_array([h_par[c, i].data_ptr() for c in range(chunks) for i in range(2)])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    comp.wait_stream(torch.cuda.current_stream())
    e0.record(comp)
    check(L.lib().gs_encode_offload(pipe.handle, enc.handle, chunks, slots, outs, sl, comp.cuda_stream,
                                    copy.cuda_stream), "c3 offload")
    comp.wait_stream(copy)
    e1.record(comp)
    e1.synchronize()
    ckpt_ms = e0.elapsed_time(e1)
    lost = 5
    saved_fp = kv[lost, :, :4096].clone()
    saved_sum = kv[lost].view(torch.int64).sum(dtype=torch.int64)
    kv[lost].zero_()
    torch.cuda.synchronize()
    dec = decoder(scheme, ErasurePattern([lost]))
    rslots = []
    for c in range(chunks):
        for j in range(10):
            if j == lost:
                rslots.append(None)
            elif j < 8:
                rslots.append(kv[j, c].data_ptr())
            else:
                rslots.append(h_par[c, j - 8].data_ptr())
    routs = L.ptr_array([kv[lost, c].data_ptr() for c in range(chunks)])
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0.record(comp)
    check(L.lib().gs_reconstruct_upload(pipe.handle, dec.handle, chunks, L.ptr_array(rslots), routs, sl,
                                        comp.cuda_stream, copy.cuda_stream), "c3 rebuild")
    r1.record(comp)
    r1.synchronize()
    rec_ms = r0.elapsed_time(r1)
    ok = torch.equal(kv[lost, :, :4096], saved_fp) and bool(
        kv[lost].view(torch.int64).sum(dtype=torch.int64) == saved_sum)
    h2d = chunks * sl
    out = {"c3_full_shard_ms": round(rec_ms, 2), "c3_shard_bytes": chunks * sl,
           "c3_h2d_gbs": round(h2d / (rec_ms * 1e-3) / 1e9, 2),
           "c3_checkpoint_ms": round(ckpt_ms, 2), "c3_checkpoint_data_gbs": round(
               8 * chunks * sl / (ckpt_ms * 1e-3) / 1e9, 2), "c3_rebuild_ok": ok}
    del kv, h_par
    torch.cuda.empty_cache()
    return out


def c3_orchestrated(torch, dev, link, k1_gbs, k2_gbs):
    """SURVEY §8f-2 with real timings: the reference's checkpoint/recovery
    semantics end to end on the C3 request (Llama-3-70B TP=8, 128K-token
    prefill = 64 chunks of 2048) through the orchestration mirror:
    run_prefill_with_checkpointing (K1 + D2H straight into ParityStore
    entries, FNV-1a seal on host threads) and recover() after worker 5 fails
    at chunk 64, planned by get_recompute_units (recovery.hpp:58-88) on a
    CostModel calibrated with this run's measured host link, K1 and K2 rates.
    Reports the plan, the FNV verification time, the batched decode time and
    the wall time to verified, rebuilt bytes."""
    from paper_2605_00831_b200 import kv_layout as K
    from paper_2605_00831_b200.checkpoint import (CheckpointConfig, Checkpointer, CostModel, FailureEvent,
                                                  get_recompute_units)
    from paper_2605_00831_b200.coding import CodingScheme
    from paper_2605_00831_b200.parity_store import ParityStore

    cfg_m = K.LLAMA3_70B
    m, tokens = 2048, 131072
    free, _ = torch.cuda.mem_get_info(dev)
    sl = K.slice_bytes(cfg_m, m)
    if free < 64 * 8 * sl + (4 << 30):
        return {"c3_orchestrated_skipped": "not enough device memory"}
    cost = CostModel.measured(link["h2d"], k1_gbs, k2_gbs)
    cfg = CheckpointConfig(CodingScheme.reed_solomon(8, 2), m, cfg_m, cost)
    threads = max(1, (os.cpu_count() or 1) - 2)
    store = ParityStore(seal_threads=threads)
    store.bind_device(dev.index or 0)
    ck = Checkpointer(cfg, store, device=dev.index or 0)
    # warm pass: the host tier's pinned slabs (10 GiB here) and the device
    # blocks of the 512 KV slices are allocated once and then recycled (store
    # free lists, torch caching allocator), as in a serving process
    warm = ck.run_prefill_with_checkpointing(10, tokens, kv_seed=KV_SEED, keep_ground_truth=True)
    ck.synchronize()
    # ... and the recovery's device buffers (uploaded parity rows, rebuilt
    # shards, GPU checksum scratch) likewise
    ck.recover(10, FailureEvent([5], at_chunk=warm.chunks_done), warm.ground_truth, [m] * warm.chunks_done,
               verify_threads=max(1, (os.cpu_count() or 1) - 2))
    del warm
    store.erase_request(10)
    t0 = time.perf_counter()
    run = ck.run_prefill_with_checkpointing(11, tokens, kv_seed=KV_SEED)
    t_enq = time.perf_counter() - t0
    ck.synchronize()                     # D2H landed and every entry sealed
    t_sealed = time.perf_counter() - t0
    n = run.chunks_done
    r_ref = get_recompute_units(n, m, cfg.scheme, sl, CostModel())
    res = ck.recover(11, FailureEvent([5], at_chunk=n), run.ground_truth, [m] * n, verify_threads=threads)
    out = {"chunks": n, "slice_bytes": sl,
           "checkpoint_device_ms": round(run.device_ms, 2),
           "checkpoint_data_gbs": round(8 * n * sl / (run.device_ms * 1e-3) / 1e9, 2),
           "checkpoint_sealed_wall_ms": round(t_sealed * 1e3, 1),
           "checkpoint_enqueue_ms": round(t_enq * 1e3, 1),
           "cost_model_measured": {"host_gbs": link["h2d"], "encode_gbs": round(k1_gbs, 1),
                                   "reconstruct_gbs": round(k2_gbs, 1), "intra_gbs": cost.intra_bw / 1e9},
           "plan": {"mode": res.plan.mode, "recompute_chunks": res.plan.recompute_chunks,
                    "reconstruct_chunks": len(res.plan.reconstruct_ids),
                    "recompute_chunks_with_reference_constants": r_ref},
           "plan_ms": round(res.plan_ms, 1), "enqueue_ms": round(res.enqueue_ms, 1),
           "verify_host_ms": round(res.verify_host_ms, 1), "verify_threads": threads,
           "verify_gpu_chunks": res.verify_gpu_chunks,
           "decode_device_ms": round(res.reconstruct_device_ms, 2), "recover_wall_ms": round(res.wall_ms, 1),
           "parity_bytes_verified": len(res.plan.reconstruct_ids) * 2 * sl, "verified": res.verified,
           "note": "wall = plan + speculative H2D/K2 overlapped with the FNV verification of the 64 entries "
                   "(reference semantics: corrupt parity -> full-recompute fallback); verify_gpu_chunks of them "
                   "upload both parity rows and are checksummed in HBM (bit-sliced GPU FNV-1a), the rest on "
                   "host threads, split so the host link and the host cores finish together"}
    ck.close()
    del run, res
    torch.cuda.empty_cache()
    return out


def c3_recovery_striped(torch, dist, dev, comp, copy, pipe, rank, world, shared, barrier):
    """C3 at N GPUs (SURVEY §8d worked example): Llama-3-70B KV TP=8, 128K
    prefill = 64 chunks x 80 MiB per worker, the 8 workers spread over the
    ranks ([64, 8/N, L] per rank). Checkpoint: every rank encodes its byte
    range of all 64 stripes (peer shards over NVLink) and D2H's that range of
    both parity rows on its own host link into a range-local pinned slab.
    Failure of worker 5: every rank H2D's its range of parity row 0, pulls its
    range of the 7 survivors and P2P-stores the rebuilt range into worker 5's
    buffer on its owner -- the 5 GiB upload striped over N host links.
    Device time per rank, max over ranks."""
    from paper_2605_00831_b200 import device as D
    from paper_2605_00831_b200 import kv_layout as K
    from paper_2605_00831_b200.coding import CodingScheme, ErasurePattern
    from paper_2605_00831_b200.peer import PeerGroup, ShardLayout, plan_encode_striped, plan_reconstruct_striped
    from paper_2605_00831_b200.peer import stripe_range

    cfg = K.LLAMA3_70B
    m, chunks, n, k = 2048, 64, 8, 2
    sl = K.slice_bytes(cfg, m)
    layout = ShardLayout(n, world, chunks, sl)
    nl = layout.n_local
    off, ln = stripe_range(sl, rank, world)
    free, _ = torch.cuda.mem_get_info(dev)
    need = chunks * nl * sl + (2 << 30)
    ok_mem = torch.tensor([1 if free >= need else 0], device="cpu" if shared else dev)
    dist.all_reduce(ok_mem, op=dist.ReduceOp.MIN)
    if not int(ok_mem.item()):
        return {"c3_skipped": f"needs {need >> 30} GiB free per rank"}
    scheme = CodingScheme.reed_solomon(n, k)
    kv = torch.empty((chunks, nl, sl), dtype=torch.uint8, device=dev)
    for c in range(chunks):
        for jl in range(nl):
            K.make_ground_truth_slice(KV_SEED, 0, c, rank * nl + jl, cfg, m, m, out=kv[c, jl])
    torch.cuda.synchronize()
    pg = PeerGroup()
    bases = pg.share(kv)
    h_par = D.pinned_near((chunks, k, max(ln, 16)), dev.index or 0)

    def dev_timed(call):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        comp.wait_stream(torch.cuda.current_stream())
        e0.record(comp)
        call.run(comp.cuda_stream, copy.cuda_stream)
        comp.wait_stream(copy)
        e1.record(comp)
        e1.synchronize()
        barrier()
        t = torch.tensor([e0.elapsed_time(e1)], device="cpu" if shared else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    enc_call = plan_encode_striped(scheme, layout, bases, rank, pipeline=pipe, h_parity=h_par, local_parity=True)
    ckpt_ms = dev_timed(enc_call)
    lost = 5
    owner, jl = layout.owner(lost)
    saved_sum = saved_fp = None
    if rank == owner:
        saved_fp = kv[:, jl, :4096].clone()
        saved_sum = kv[:, jl].contiguous().view(torch.int64).sum(dtype=torch.int64)
        kv[:, jl].zero_()
    torch.cuda.synchronize()
    rec_call = plan_reconstruct_striped(scheme, layout, bases, rank, ErasurePattern([lost]), h_par, pipe,
                                        local_parity=True)
    rec_ms = dev_timed(rec_call)
    ok = True
    if rank == owner:
        ok = torch.equal(kv[:, jl, :4096], saved_fp) and bool(
            kv[:, jl].contiguous().view(torch.int64).sum(dtype=torch.int64) == saved_sum)
    t = torch.tensor([1 if ok else 0], device="cpu" if shared else dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    ok = bool(t.item())
    barrier()
    pg.close()
    del kv, h_par
    torch.cuda.empty_cache()
    shard = chunks * sl
    return {"c3_full_shard_ms": round(rec_ms, 2), "c3_shard_bytes": shard,
            "c3_h2d_gbs_aggregate": round(shard / (rec_ms * 1e-3) / 1e9, 2),
            "c3_h2d_links": world, "c3_checkpoint_ms": round(ckpt_ms, 2),
            "c3_checkpoint_data_gbs": round(n * shard / (ckpt_ms * 1e-3) / 1e9, 2), "c3_rebuild_ok": ok,
            "c3_mode": f"byte-range striped over {world} GPUs (parity range H2D on every host link, survivors "
                       "over NVLink, rebuilt range P2P-stored into the failed worker's buffer)"}


# ---------------------------------------------------------------------------
# C5: parity throughput sweep over block sizes (BASELINE.json configs[4])
# ---------------------------------------------------------------------------
def _parse_size(x: str) -> int:
    x = x.strip().upper()
    mult = {"K": 1 << 10, "M": 1 << 20, "G": 1 << 30}
    return int(float(x[:-1]) * mult[x[-1]]) if x[-1] in mult else int(x)


def run_sweep(args):
    """C5: for each shard length L and code (RS(8,2), XOR(8)),
    encode + D2H offload and K1 alone, weak-scaled (one stripe of n x L per
    GPU, striped over the ranks like the C2 step), with the roofline fraction
    t*/t (t* = the slowest of HBM bytes at peak, parity over the host link,
    peer bytes over NVLink) and the reference CPU encoder on this host."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2605_00831_b200 import device as D
    from paper_2605_00831_b200.coding import CodingScheme
    from paper_2605_00831_b200.peer import PeerGroup, ShardLayout, plan_encode_striped, stripe_range

    rank, world, local = env_rank()
    shared = os.environ.get("GS_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("gloo" if shared else "nccl", **({} if shared else {"device_id": dev}))
    hbm_peak, hbm_src = load_peaks()
    link = host_link_peaks(torch, dev)
    pipe = D.Pipeline(local, 256 << 20)
    comp, copy = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    pg = PeerGroup() if world > 1 else None
    cpu_ref = None
    if rank == 0 and not args.no_cpu:
        from oracle import oracle as O
        cpu_ref = (O, O.ref() if O.have_ref() else O.port(), "reference" if O.have_ref() else "port")
    threads = os.cpu_count() or 1

    def tmax(ms):
        if world == 1:
            return ms
        t = torch.tensor([ms], device="cpu" if shared else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(plans, two, iters):
        for i in range(2):
            plans[i % len(plans)].run(comp.cuda_stream, copy.cuda_stream if two else None)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(comp)
        for i in range(iters):
            plans[i % len(plans)].run(comp.cuda_stream, copy.cuda_stream if two else None)
        comp.wait_stream(copy)
        e1.record(comp)
        e1.synchronize()
        return tmax(e0.elapsed_time(e1)) / iters * 1e-3

    def graph_timed(plans, two, iters):
        """The same steps replayed from one CUDA graph holding all buffers'
        calls (the serving engine's launch mode, device.CapturedCall): host
        launch overhead out of the small-L numbers."""
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=comp):
            for p in plans:
                p.run(comp.cuda_stream, copy.cuda_stream if two else None)
            if two:
                comp.wait_stream(copy)
        reps = max(2, -(-iters // len(plans)))
        with torch.cuda.stream(comp):
            g.replay()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(comp):
            e0.record(comp)
            for _ in range(reps):
                g.replay()
            e1.record(comp)
        e1.synchronize()
        del g
        return tmax(e0.elapsed_time(e1)) / (reps * len(plans)) * 1e-3

    codes = [("RS(8,2)", CodingScheme.reed_solomon(8, 2)), ("XOR(8)", CodingScheme.xor_code(8))]
    for name, scheme in codes:
        n, k = scheme.n, scheme.k
        for L_ in [_parse_size(x) for x in args.sweep_sizes.split(",")]:
            S = world
            layout = ShardLayout(n, world, S, L_)
            nl = layout.n_local
            iters = max(3, min(args.steps, int((4 << 30) // (S * n * L_))))
            nbuf = max(1, min(16, -(-(256 << 20) // (S * nl * L_))))   # rotate so each step misses L2
            data = torch.randint(0, 256, (nbuf, S, nl, L_), dtype=torch.uint8, device=dev)
            bases = [pg.share(data[b]) if pg else [data[b].data_ptr()] for b in range(nbuf)]
            h_par = torch.empty((S, k, L_), dtype=torch.uint8).pin_memory()
            _, ln = stripe_range(L_, rank, world)
            par_dev = torch.empty((S, k, max(ln, 1)), dtype=torch.uint8, device=dev)
            off_plans = [plan_encode_striped(scheme, layout, bases[b], rank, pipeline=pipe, h_parity=h_par)
                         for b in range(nbuf)]
            k_plans = [plan_encode_striped(scheme, layout, bases[b], rank, parity_out=par_dev)
                       for b in range(nbuf)]
            t_off = timed(off_plans, True, iters)
            last = (iters - 1) % nbuf
            ok = True
            if world == 1:
                ok = torch.equal(h_par.to(dev), D.encode(scheme, data[last].view(S, n, L_)))
            t_k1 = timed(k_plans, False, iters)
            t_off_g = graph_timed(off_plans, True, iters)
            t_k1_g = graph_timed(k_plans, False, iters)
            if pg:
                pg.close()
            per_gpu = S * L_ // world
            t_star = max((n + k) * per_gpu / (hbm_peak * 1e9), k * per_gpu / (link["d2h"] * 1e9),
                         (world - 1) / world * n * per_gpu / 900e9)
            row = {"sweep": "C5", "code": name, "shard_bytes": L_, "n_gpus": world, "stripes": S,
                   "data_bytes_per_step": S * n * L_,
                   "offload_gbs": round(S * n * L_ / t_off / 1e9, 2), "offload_ms": round(t_off * 1e3, 4),
                   "k1_gbs_hbm": round((n + k) * S * L_ / world / t_k1 / 1e9, 1),
                   "k1_us": round(t_k1 * 1e6, 2), "roofline_frac": round(t_star / t_off, 4),
                   "graph": {"offload_gbs": round(S * n * L_ / t_off_g / 1e9, 2),
                             "offload_ms": round(t_off_g * 1e3, 4), "k1_us": round(t_k1_g * 1e6, 2),
                             "k1_gbs_hbm": round((n + k) * S * L_ / world / t_k1_g / 1e9, 1),
                             "roofline_frac": round(t_star / t_off_g, 4)},
                   "roofline_bound": "host_link" if k * per_gpu / link["d2h"] > (n + k) * per_gpu / hbm_peak
                   else "hbm", "hbm_peak_gbs": hbm_peak, "d2h_peak_gbs": link["d2h"], "parity_ok": ok}
            if cpu_ref is not None:
                O, lib, kind = cpu_ref
                Lc = min(L_, 64 << 20)
                rng = np.random.default_rng(42)
                d = [rng.integers(0, 256, Lc, dtype=np.uint8) for _ in range(n)]
                pp = [np.zeros(Lc, np.uint8) for _ in range(k)]
                okind = O.RS if name.startswith("RS") else O.XOR
                busy, reps = 0.0, 0
                while busy < args.sweep_cpu_s or reps == 0:
                    if kind == "reference":
                        busy += lib.encode_timed(okind, n, k, d, pp, threads)
                    else:
                        t1 = time.perf_counter()
                        lib.encode(okind, n, k, d)
                        busy += time.perf_counter() - t1
                    reps += 1
                row["cpu_baseline"] = {"value": round(reps * n * Lc / busy / 1e9, 3), "unit": "GB/s",
                                       "cores": threads if kind == "reference" else 1, "kind": kind,
                                       "sample": f"{reps} encode(s) of {n} x {Lc} B"}
            if rank == 0:
                print(json.dumps(row), flush=True)
            del data, h_par, par_dev, off_plans, k_plans
            torch.cuda.empty_cache()
            if world > 1:
                dist.barrier()
    pipe.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-sample-s", type=float, default=3.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c3", action="store_true")
    ap.add_argument("--no-c4", action="store_true")
    ap.add_argument("--no-overhead", action="store_true")
    ap.add_argument("--decode-ctx", type=int, default=4096)
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu dram bytes per K1 launch (from profiles/), echoed into roofline.traffic")
    ap.add_argument("--encoder", choices=["stripe", "rotate"], default="stripe",
                    help="N>1: byte-range striping (default) or the paper's rotating per-chunk encoder")
    ap.add_argument("--sweep", action="store_true", help="C5 block-size sweep instead of the C2 step")
    ap.add_argument("--sweep-sizes", default="64K,256K,1M,4M,16M,64M,256M,1G")
    ap.add_argument("--sweep-cpu-s", type=float, default=0.5)
    ap.add_argument("--configs", action="store_true",
                    help="per-config table C1-C4 (encode+D2H, K1, recovery, rooflines, reference CPU, bit-exact)")
    ap.add_argument("--configs-only", default="", help="subset for --configs, e.g. C1,C4")
    args = ap.parse_args()
    if args.configs:
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "--configs is our arm only"}))
            return
        from tools.config_table import run_configs
        run_configs(args)
        return
    if args.sweep:
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "--sweep is our arm only"}))
            return
        run_sweep(args)
        return
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
