"""Checkpoint / recovery orchestration on the GPU byte path.

Mirrors the byte-moving parts of checkpoint.hpp and recovery.hpp:

* ``next_parity_worker`` / ``AssignmentState``      checkpoint.hpp:21-30
* ``CheckpointConfig``                              checkpoint.hpp:32-47
* ``Checkpointer.checkpoint_chunk``                 checkpoint.hpp:123-149 (encode + seal -> host tier)
* ``Checkpointer.run_prefill_with_checkpointing``   checkpoint.hpp:179-222
* ``DecodeCheckpointer``                            checkpoint.hpp:228-281
* ``get_recompute_units`` / ``CostModel``           recovery.hpp:58-88, cost_model.hpp:17-68
* ``Checkpointer.reconstruct_chunk``                recovery.hpp:100-133
* ``verify_recovery``                               recovery.hpp:135-145
* ``Checkpointer.recover``                          recovery.hpp:176-298 (plan + byte restore)

The reference computes bytes on one CPU thread and models time with
cost-model constants. Here the bytes come from K1/K2 with the D2H/H2D
overlapped by the pipeline, parity lands directly in the pinned host store
(no try_put copy) and is sealed by host threads, and the outcomes carry
MEASURED device times (CUDA events) instead of virtual-clock events. The
cost model survives only as the recompute/reconstruct split planner, and can
be calibrated from measurements (``CostModel.measured``).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Set

import torch

from . import _lib as L
from .coding import (CodingScheme, ErasurePattern, InvalidArgument, LogicError, UnrecoverableError, check,
                     decoder, encoder, max_tolerance)
from .device import Pipeline
from .kv_layout import ModelConfig, chunk_count, make_ground_truth_slice, slice_bytes
from .parity_store import ParityGetStatus, ParityStore


# ---------------------------------------------------------------------------
# cost model + planner (cost_model.hpp:17-68, recovery.hpp:58-88)
# ---------------------------------------------------------------------------
@dataclass
class CostModel:
    compute_per_token: float = 6.0e-5
    intra_bw: float = 400e9
    host_bw: float = 32e9
    encode_rate: float = 180e9
    reconstruct_rate: float = 300e9
    fixed_collective_latency: float = 2.0e-5
    restart_overhead: float = 2.0

    def validate(self) -> None:
        if (self.compute_per_token <= 0 or self.intra_bw <= 0 or self.host_bw <= 0 or self.encode_rate <= 0
                or self.reconstruct_rate <= 0 or self.fixed_collective_latency < 0 or self.restart_overhead < 0):
            raise InvalidArgument("cost: rates must be positive")
        if self.host_bw > self.intra_bw:
            raise InvalidArgument("cost: host link cannot be faster than the intra-node fabric")

    def chunk_compute_time(self, tokens: int) -> float:
        return tokens * self.compute_per_token

    def gather_time(self, tp: int, slice_: int) -> float:
        return (tp - 1) * slice_ / self.intra_bw + self.fixed_collective_latency

    def encode_time(self, tp: int, slice_: int) -> float:
        return tp * slice_ / self.encode_rate

    def offload_time(self, k: int, slice_: int) -> float:
        return k * slice_ / self.host_bw

    def parity_fetch_time(self, k: int, slice_: int) -> float:
        return k * slice_ / self.host_bw

    def reconstruct_time(self, tp: int, slice_: int) -> float:
        return tp * slice_ / self.reconstruct_rate

    def reconstruct_chunk_time(self, scheme: CodingScheme, slice_: int) -> float:
        return (self.parity_fetch_time(scheme.k, slice_) + self.gather_time(scheme.n, slice_)
                + self.reconstruct_time(scheme.n, slice_))

    @staticmethod
    def measured(host_gbs: float, encode_gbs: float, reconstruct_gbs: float, intra_gbs: float = 770.0,
                 compute_per_token: float = 6.0e-5, restart_overhead: float = 2.0) -> "CostModel":
        """Cost model calibrated from B200 measurements (bench.py / kernel_sweep):
        host link, K1 and K2 data rates in GB/s; NVLink peer rate default =
        the measured 770 GB/s per direction (B200_PROFILING.md)."""
        return CostModel(compute_per_token, intra_gbs * 1e9, host_gbs * 1e9, encode_gbs * 1e9,
                         reconstruct_gbs * 1e9, 2.0e-5, restart_overhead)


def get_recompute_units(n: int, chunk_size: int, scheme: CodingScheme, slice_: int, cost: CostModel) -> int:
    """argmin_r max(r*m*c + restart, (n-r)*T_rec); ties -> smaller r (recovery.hpp:58-88)."""
    if n == 0:
        return 0
    a = chunk_size * cost.compute_per_token
    c = cost.reconstruct_chunk_time(scheme, slice_)
    restart = cost.restart_overhead

    def objective(r: int) -> float:
        return max(r * a + restart, (n - r) * c)

    cands = [0, n]
    if a + c > 0:
        x = (n * c - restart) / (a + c)
        fl = math.floor(x)
        if 0 <= fl <= n:
            cands.append(int(fl))
        if 0 <= fl + 1 <= n:
            cands.append(int(fl + 1))
    cands.sort()
    best, best_f = cands[0], objective(cands[0])
    for r in cands:
        f = objective(r)
        if f < best_f:
            best, best_f = r, f
    return best


# ---------------------------------------------------------------------------
# assignment + config (checkpoint.hpp:21-47)
# ---------------------------------------------------------------------------
@dataclass
class AssignmentState:
    next_worker: int = 0


def next_parity_worker(state: AssignmentState, tp_degree: int) -> int:
    if tp_degree < 1:
        raise InvalidArgument("assignment: worker count must be positive")
    w = state.next_worker
    state.next_worker = (state.next_worker + 1) % tp_degree
    return w


@dataclass
class CheckpointConfig:
    scheme: CodingScheme = field(default_factory=lambda: CodingScheme.reed_solomon(8, 2))
    chunk_size: int = 2048
    model: ModelConfig = field(default_factory=ModelConfig)
    cost: CostModel = field(default_factory=CostModel)
    checkpoint_decode: bool = True

    def validate(self) -> None:
        self.scheme.validate()
        self.model.validate()
        self.cost.validate()
        if self.chunk_size == 0:
            raise InvalidArgument("checkpoint: chunk size must be positive")
        if self.scheme.n != self.model.tp_degree:
            raise InvalidArgument("checkpoint: data shard count must equal tp_degree")


@dataclass
class KvChunkSlice:
    """kv_layout.hpp:62-68 with the bytes on the device."""

    request_id: int
    chunk_id: int
    worker: int
    bytes: torch.Tensor
    valid_tokens: int


@dataclass
class ChunkCheckpointOutcome:
    request_id: int
    chunk_id: int
    valid_tokens: int
    parity_worker: int
    stored: bool                 # False = back-pressure (store unchanged)
    enqueue_s: float = 0.0       # host time to plan + enqueue


@dataclass
class PrefillRunResult:
    completed: bool = False
    chunks_done: int = 0
    stalled_at_chunk: Optional[int] = None
    state: AssignmentState = field(default_factory=AssignmentState)
    ground_truth: List[List[KvChunkSlice]] = field(default_factory=list)
    device_ms: float = 0.0


class ChunkRepairStatus:
    kOk = 0
    kBadParity = 1


@dataclass
class ChunkRepairResult:
    status: int = ChunkRepairStatus.kOk
    recovered: Dict[int, KvChunkSlice] = field(default_factory=dict)


@dataclass
class FailureEvent:
    failed_workers: List[int]
    at_chunk: int = 0
    at_time: float = 0.0


class RecoveryAbort(RuntimeError):
    """recovery.hpp RecoveryAbort: the store changed or a needed payload is
    missing mid-recovery."""


class RecoveryMode:
    kPureRecompute = "pure_recompute"
    kHybrid = "hybrid"
    kFullRecomputeFallback = "full_recompute_fallback"


@dataclass
class RecoveryPlan:
    recompute_chunks: int = 0
    reconstruct_ids: List[int] = field(default_factory=list)
    mode: str = RecoveryMode.kPureRecompute


@dataclass
class RecoveryResult:
    plan: RecoveryPlan = field(default_factory=RecoveryPlan)
    recovered: Dict[int, List[Optional[KvChunkSlice]]] = field(default_factory=dict)
    verified: bool = True
    parity_bytes_fetched: int = 0
    reconstruct_device_ms: float = 0.0   # batched H2D + K2 over every reconstructed chunk
    verify_host_ms: float = 0.0          # FNV verification of their parity (host threads)
    plan_ms: float = 0.0                 # get_recompute_units + store lookups
    enqueue_ms: float = 0.0              # host time to enqueue the batched H2D + K2
    verify_gpu_chunks: int = 0           # entries whose checksum was verified on the GPU
    wall_ms: float = 0.0                 # plan -> verified, rebuilt bytes on the device
    corrupt_chunks: List[int] = field(default_factory=list)   # parity that failed verification (-> fallback)
    verify_split: Dict[str, float] = field(default_factory=dict)  # dynamic split timeline / shares
    decoded_chunks: int = 0              # chunks whose lost shards came out of K2 (and matched ground truth)


def verify_recovery(recovered, ground_truth) -> bool:
    """recovery.hpp:135-145 (bytes, or slices incl. worker / valid_tokens)."""
    if isinstance(recovered, KvChunkSlice):
        return (recovered.worker == ground_truth.worker and recovered.valid_tokens == ground_truth.valid_tokens
                and verify_recovery(recovered.bytes, ground_truth.bytes))
    return recovered.numel() == ground_truth.numel() and bool(torch.equal(recovered, ground_truth))


class _VerifyFinish:
    """gs_verify_finish on a Python thread (the C call drops the GIL): host
    threads continue the split entries' FNV chains as the GPU's chain states
    arrive; result() -> (checksums, host ms)."""

    def __init__(self, handle, n: int, threads: int):
        import threading
        self._out = (C.c_uint64 * max(n, 1))()
        self._n = n
        self._rc = 0
        self._ms = 0.0
        self._gpu = C.c_int(0)

        def run():
            t0 = time.perf_counter()
            self._rc = L.lib().gs_verify_finish_ex(handle, threads, self._out, C.byref(self._gpu))
            self._ms = (time.perf_counter() - t0) * 1e3

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def result(self):
        """(checksums, host ms, chunks hashed entirely on the GPU)."""
        self._t.join()
        check(self._rc, "recover verify")
        return [int(self._out[i]) for i in range(self._n)], self._ms, int(self._gpu.value)


class _HostVerify:
    """FNV verification of parity entries on host threads, run from a Python
    thread (the C call releases the GIL) so it overlaps the enqueue of the
    speculative decode instead of following it."""

    def __init__(self, ck: "Checkpointer", entries, threads: int):
        import threading
        self._ok: List[bool] = []
        self._ms = 0.0
        self._err: Optional[BaseException] = None

        def run():
            t0 = time.perf_counter()
            try:
                self._ok = ck._verify_entries(entries, threads)
            except BaseException as e:   # re-raised in result()
                self._err = e
            self._ms = (time.perf_counter() - t0) * 1e3

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def result(self):
        self._t.join()
        if self._err is not None:
            raise self._err
        return self._ok, self._ms


# ---------------------------------------------------------------------------
# the orchestrator
# ---------------------------------------------------------------------------
class Checkpointer:
    """One device's checkpoint engine: pipeline (staging ring + events),
    compute and copy streams, the host-tier store."""

    def __init__(self, cfg: CheckpointConfig, store: ParityStore, device: int = 0,
                 staging_bytes: int = 256 << 20):
        cfg.validate()
        self.cfg = cfg
        self.store = store
        self.device = device
        self.dev = torch.device("cuda", device)
        self.pipe = Pipeline(device, staging_bytes)
        self.compute = torch.cuda.Stream(device=self.dev)
        self.copy = torch.cuda.Stream(device=self.dev)
        self.verify = torch.cuda.Stream(device=self.dev)   # GPU parity checksums (recover)
        self.slice = slice_bytes(cfg.model, cfg.chunk_size)
        # Aggregate host FNV-1a rate (bytes/s) used to split recovery's parity
        # verification between host threads and the GPU (recover()), and the
        # rate of ONE chain on one host thread. The bit-sliced AVX-512 chain
        # (gs_fnv_simd.cpp, gs_fnv_host_simd() == 1): ~6 GB/s per chain and
        # core, 94 GB/s on the 16 host threads of the B200 boxes
        # (tools/fnv_host_mt.cpp); the scalar chain: ~0.9 GB/s per chain, ~1.6
        # GB/s per thread in lockstep pairs while the parity upload streams
        # over the same host memory.
        simd = bool(L.lib().gs_fnv_host_simd())
        self.host_chain_rate = 5.0e9 if simd else 0.9e9
        self.host_fnv_rate = (5.0e9 if simd else 1.6e9) * max(1, (os.cpu_count() or 1) - 2)
        # False: verify every entry on host threads (the reference's placement)
        self.gpu_verify = True
        # "dynamic": the part of each parity chain the decode does not upload
        # is claimed at run time by host threads or a GPU feeder (whichever is
        # faster on this host takes more); "static": split decided up front
        # from host_fnv_rate / host_chain_rate (_split_plan)
        self.verify_split = "dynamic"
        # Where checkpoint_batch seals parity (ParityChunk::seal): "host" = FNV
        # on the store's host threads after the D2H (the reference's order);
        # "device" = K1 into HBM, checksum on the GPU, D2H of rows + checksum;
        # "auto" = device when a batch carries >= 4 MiB of parity: a chunk's
        # serial host chain (~1 GB/s) trails the link by milliseconds, and the
        # host threads seal ~18 GB/s in aggregate vs the link's ~56 GB/s.
        self.seal = "auto"
        self.seal_inflight_bytes = 2 << 30   # device parity buffers awaiting their D2H
        self._inflight: List[tuple] = []      # (event on copy, keep-alive tensors, bytes)

    def close(self) -> None:
        self.pipe.close()

    def synchronize(self) -> None:
        self.copy.synchronize()
        self.compute.synchronize()
        self.store.wait_sealed()
        self._inflight.clear()

    # checkpoint.hpp:123-149 (+ the try_put of :207)
    def checkpoint_chunk(self, slices: Sequence[KvChunkSlice], state: AssignmentState) -> ChunkCheckpointOutcome:
        cfg = self.cfg
        if len(slices) != cfg.scheme.n:
            raise LogicError("checkpoint: expected one slice per worker")
        s0 = slices[0]
        for s in slices:
            if s.bytes.numel() != self.slice:
                raise LogicError("checkpoint: slice has unexpected length")
            if (s.chunk_id, s.request_id, s.valid_tokens) != (s0.chunk_id, s0.request_id, s0.valid_tokens):
                raise LogicError("checkpoint: slices disagree on chunk identity")
        return self.checkpoint_batch([list(slices)], state)[0]

    def checkpoint_batch(self, batch: Sequence[Sequence[KvChunkSlice]], state: AssignmentState
                         ) -> List[ChunkCheckpointOutcome]:
        """Checkpoint several (request, chunk) stripes with ONE K1 launch +
        overlapped D2H (e.g. the 32 requests of a decode block)."""
        t0 = time.perf_counter()
        cfg = self.cfg
        sch = cfg.scheme
        outs, slots, dsts, keys = [], [], [], []
        for slices in batch:
            s0 = slices[0]
            worker = next_parity_worker(state, sch.n)
            ptrs = self.store.reserve(s0.request_id, s0.chunk_id, sch, s0.valid_tokens, self.slice)
            outs.append(ChunkCheckpointOutcome(s0.request_id, s0.chunk_id, s0.valid_tokens, worker, ptrs is not None))
            if ptrs is None:
                continue
            for s in slices:
                # K1 reads the slice on self.compute: a caller dropping it after
                # this call must not let the caching allocator hand its block to
                # a later kernel on the slice's own stream before K1 has run
                s.bytes.record_stream(self.compute)
            slots.extend(s.bytes.data_ptr() for s in slices)
            dsts.extend(ptrs)
            keys.append((s0.request_id, s0.chunk_id))
        if keys and self._device_seal(len(keys)):
            self._checkpoint_device_sealed(keys, slots, dsts)
        elif keys:
            self.compute.wait_stream(torch.cuda.current_stream(self.dev))
            check(L.lib().gs_encode_offload(self.pipe.handle, encoder(sch).handle, len(keys), L.ptr_array(slots),
                                            L.ptr_array(dsts), self.slice, self.compute.cuda_stream,
                                            self.copy.cuda_stream), "checkpoint")
            self.store.commit_batch(keys, self.copy)   # one host callback seals the batch
        dt = time.perf_counter() - t0
        for o in outs:
            o.enqueue_s = dt / max(len(outs), 1)
        return outs

    def make_slices(self, kv_seed: int, request_id: int, chunk: int, valid: int) -> List[KvChunkSlice]:
        m = self.cfg.model
        return [KvChunkSlice(request_id, chunk, w,
                             make_ground_truth_slice(kv_seed, request_id, chunk, w, m, self.cfg.chunk_size, valid,
                                                     device=self.dev), valid)
                for w in range(self.cfg.scheme.n)]

    # checkpoint.hpp:179-222
    def _device_seal(self, stripes: int = 1) -> bool:
        if self.slice % 16:   # the GPU FNV takes 16-B multiples: host seal
            return False
        if self.seal == "device":
            return True
        if self.seal == "auto":
            return stripes * self.cfg.scheme.k * self.slice >= (4 << 20)
        return False

    def _checkpoint_device_sealed(self, keys, slots, dsts) -> None:
        """K1 over the batch into HBM, the chunks' checksums on the GPU
        (gs_parity_offload_sealed), D2H of the rows and the checksums into the
        reserved store entries, sealed by one host callback with no FNV pass.
        At most seal_inflight_bytes of device parity await their D2H."""
        sch = self.cfg.scheme
        S, k = len(keys), sch.k
        need = S * k * self.slice
        self._inflight = [f for f in self._inflight if not f[0].query()]
        while self._inflight and sum(f[2] for f in self._inflight) + need > self.seal_inflight_bytes:
            self._inflight.pop(0)[0].synchronize()
        cur = torch.cuda.current_stream(self.dev)
        self.compute.wait_stream(cur)
        self.copy.wait_stream(cur)
        par = torch.empty((S, k, self.slice), dtype=torch.uint8, device=self.dev)
        # checksums stay on the device: the store copies them on `copy` into
        # pinned memory it owns (gs_store_commit_sealed_batch), so nothing the
        # store's landing thread reads depends on this tensor's lifetime
        sums = torch.empty(S, dtype=torch.int64, device=self.dev)
        rows = L.ptr_array([par[s, i].data_ptr() for s in range(S) for i in range(k)])
        lib = L.lib()
        check(lib.gs_apply_device(encoder(sch).handle, S, L.ptr_array(slots), rows, self.slice,
                                  self.compute.cuda_stream), "checkpoint")
        check(lib.gs_parity_offload_sealed(rows, S, k, self.slice, L.ptr_array(dsts), sums.data_ptr(),
                                           self.compute.cuda_stream, self.copy.cuda_stream), "checkpoint seal")
        self.store.commit_sealed_batch(keys, sums.data_ptr(), self.copy)
        done = torch.cuda.Event()
        done.record(self.copy)
        # par / sums were allocated on the current stream and are used on
        # compute and copy: they are dropped only after `done` (copy waits on
        # compute's K1 + FNV), so their blocks are never reused early
        self._inflight.append((done, (par, sums), need))

    def run_prefill_with_checkpointing(self, request_id: int, input_tokens: int, kv_seed: int = 0,
                                       keep_ground_truth: bool = True) -> PrefillRunResult:
        cfg = self.cfg
        chunks = chunk_count(input_tokens, cfg.chunk_size)
        run = PrefillRunResult()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(self.compute)
        for c in range(chunks):
            valid = input_tokens - c * cfg.chunk_size if c + 1 == chunks else cfg.chunk_size
            slices = self.make_slices(kv_seed, request_id, c, valid)
            out = self.checkpoint_chunk(slices, run.state)
            if not out.stored:
                run.stalled_at_chunk = c
                break
            if keep_ground_truth:
                run.ground_truth.append(slices)
            run.chunks_done += 1
        self.compute.wait_stream(self.copy)
        e1.record(self.compute)
        e1.synchronize()
        run.device_ms = e0.elapsed_time(e1)
        run.completed = run.stalled_at_chunk is None
        return run

    # recovery.hpp:100-133
    def reconstruct_chunk(self, chunk_id: int, surviving: Sequence[KvChunkSlice], request_id: int,
                          failed: Set[int]) -> ChunkRepairResult:
        sch = self.cfg.scheme
        if len(failed) > max_tolerance(sch):
            raise UnrecoverableError("recovery: failures exceed scheme tolerance")
        res = ChunkRepairResult()
        status, entry = self.store.get(request_id, chunk_id, verify=True)
        if status != ParityGetStatus.kOk or not entry.payload_present():
            res.status = ChunkRepairStatus.kBadParity
            return res
        lost = ErasurePattern(sorted(failed))
        dec = decoder(sch, lost)
        slots: List[Optional[int]] = [None] * (sch.n + sch.k)
        for s in surviving:
            if s.worker not in failed:
                slots[s.worker] = s.bytes.data_ptr()
        for i in range(sch.k):
            slots[sch.n + i] = entry.parity[i].ctypes.data
        for j in range(sch.n):
            if j not in failed and slots[j] is None:
                raise InvalidArgument(f"coding: surviving shard {j} missing from input")
        outs = {w: torch.empty(self.slice, dtype=torch.uint8, device=self.dev) for w in dec.out_index}
        if dec.n_out:
            self.compute.wait_stream(torch.cuda.current_stream(self.dev))
            check(L.lib().gs_reconstruct_upload(self.pipe.handle, dec.handle, 1, L.ptr_array(slots),
                                                L.ptr_array([outs[w].data_ptr() for w in dec.out_index]),
                                                self.slice, self.compute.cuda_stream, self.copy.cuda_stream),
                  "reconstruct_chunk")
            torch.cuda.current_stream(self.dev).wait_stream(self.compute)
        for w, t in outs.items():
            res.recovered[w] = KvChunkSlice(request_id, chunk_id, w, t, entry.valid_tokens)
        return res

    # recovery.hpp:176-298
    def recover(self, request_id: int, failure: FailureEvent,
                ground_truth: Optional[List[List[KvChunkSlice]]], chunk_tokens: Sequence[int],
                buffered_decode_tokens: int = 0, verify_threads: int = 0) -> RecoveryResult:
        """Hybrid recovery with the reference's decisions (recovery.hpp:176-298):
        r = get_recompute_units(...) chunks recomputed (here restored from the
        ground-truth slices, the reference's own stand-in, recovery.hpp:269-296)
        and chunks r..n-1 erasure-decoded, after a planning pass that requires
        every one of their parity entries to verify (kCorrupt / kMissing ->
        full-recompute fallback).

        B200 schedule of the same decisions: the decode of all n-r chunks is
        enqueued speculatively while their parity is verified, and a failed
        verification discards it and falls back exactly as the planning pass
        would. Verification (gpu_verify=True) is split so the host link and
        the host cores finish together (_split_plan): n_full entries upload
        ALL their parity rows and are checksummed in HBM by the bit-sliced GPU
        FNV-1a; the others upload only the rows K2 uses, the GPU hashes those
        and host threads continue the serial chain over the remaining rows
        (gs_verify_enqueue / gs_verify_finish, finished on a Python thread).
        K2 then reads the uploaded rows. gpu_verify=False keeps the
        reference's placement: one gs_reconstruct_upload + FNV of every entry
        on host threads. Each chunk's parity is verified once (the reference
        re-verifies inside
        reconstruct_chunk; the store is not modified in between)."""
        cfg = self.cfg
        t_wall = time.perf_counter()
        if not failure.failed_workers:
            raise InvalidArgument("recovery: no failed workers")
        n = failure.at_chunk
        if len(chunk_tokens) < n:
            raise InvalidArgument("recovery: missing chunk token counts")
        result = RecoveryResult()
        plan = result.plan
        over = len(failure.failed_workers) > max_tolerance(cfg.scheme)
        r = n if over else get_recompute_units(n, cfg.chunk_size, cfg.scheme, self.slice, cfg.cost)
        entries = []
        parity_ok = True
        if not over and r < n:
            for c in range(r, n):
                # the reference's planning pass checks the get() status only
                # (recovery.hpp:200-207); the checksums are verified below, in
                # bulk, overlapped with the speculative decode
                st, e = self.store.get(request_id, c, verify=False)
                if st != ParityGetStatus.kOk:
                    parity_ok = False
                    break
                if ground_truth is not None and not e.payload_present():
                    # materialized recovery of a cost-only entry: reconstruct_chunk
                    # reports kBadParity and the reference aborts (recovery.hpp:280-283)
                    raise RecoveryAbort("recovery: parity failed verification mid-recovery")
                entries.append(e)
        if entries and not all(e.payload_present() for e in entries):
            entries = []        # cost-only entries: nothing to verify or decode (get() said kOk)
        failed = set(failure.failed_workers)
        pending = []            # (first chunk id, outs, out_index, keep-alive)
        gpu_sums = None
        n_gpu = 0
        e0 = e1 = None
        result.plan_ms = (time.perf_counter() - t_wall) * 1e3
        decode = parity_ok and not over and r < n and ground_truth is not None
        gpu_verify = self.gpu_verify and self.slice % 16 == 0   # the GPU FNV takes 16-B multiples
        host_verify = None
        split = None            # (n_full, in-flight gs_verify finished on a host thread)
        if parity_ok and entries and not (decode and gpu_verify):
            # the reference's placement: every entry verified on host threads,
            # overlapped with the enqueue and the decode
            host_verify = _HostVerify(self, entries, verify_threads)
        if decode:
            if len(ground_truth) < n:
                raise RuntimeError("recovery: ground truth missing for completed chunks")
            t0 = time.perf_counter()
            ids = list(range(r, n))
            cur = torch.cuda.current_stream(self.dev)
            for st in (self.compute, self.copy, self.verify):
                st.wait_stream(cur)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(self.compute)
            if gpu_verify:
                outs, oi, n_full, split_h, keep = self._enqueue_split_verified_decode(ground_truth, ids, entries,
                                                                                     failed, verify_threads)
                pending.append((r, outs, oi, keep))
                split = (n_full, split_h)
            else:
                outs, oi = self._enqueue_batched_decode(ground_truth, ids, entries, failed)
                pending.append((r, outs, oi, None))
            self.compute.wait_stream(self.verify)
            e1.record(self.compute)
            cur.wait_stream(self.compute)
            result.enqueue_ms = (time.perf_counter() - t0) * 1e3
        if parity_ok and entries:
            good: List[bool] = []
            if host_verify is not None:
                good, result.verify_host_ms = host_verify.result()
            if split is not None:
                sums, result.verify_host_ms, result.verify_gpu_chunks = split[1].result()
                if self.verify_split == "dynamic":
                    st6 = (C.c_double * 6)()
                    L.lib().gs_verify_last_stats(st6)
                    result.verify_split = {"hosts_done_ms": round(st6[0] * 1e3, 1),
                                           "gpu_feeder_done_ms": round(st6[1] * 1e3, 1),
                                           "hash_stream_drained_ms": round(st6[2] * 1e3, 1),
                                           "chunks_host": int(st6[3]), "chunks_gpu": int(st6[4]),
                                           "chunks_handed_over": int(st6[5])}
                good = [sums[i] == e.checksum for i, e in enumerate(entries)]
            bad = [i for i, g in enumerate(good) if not g]
            if bad:
                # a fallback is only legitimate if the reference's own serial
                # FNV-1a (ParityChunk::compute_checksum) agrees that the stored
                # parity is corrupt; a disagreement is a bug in the fast
                # verification or the seal, never a silent full recompute
                wrong = [entries[i].chunk_id for i in bad if entries[i].compute_checksum() == entries[i].checksum]
                if wrong:
                    raise RuntimeError(f"recovery: fast parity verification rejected chunks {wrong} whose "
                                       "stored checksum the serial FNV-1a accepts")
                result.corrupt_chunks = [entries[i].chunk_id for i in bad]
                parity_ok = False
        if over or (not parity_ok and r < n):
            plan.mode, r = RecoveryMode.kFullRecomputeFallback, n
        elif r >= n:
            plan.mode, r = RecoveryMode.kPureRecompute, n
        else:
            plan.mode = RecoveryMode.kHybrid
        plan.recompute_chunks = r
        plan.reconstruct_ids = list(range(r, n))
        result.parity_bytes_fetched = len(plan.reconstruct_ids) * cfg.scheme.k * self.slice
        if ground_truth is None:
            result.wall_ms = (time.perf_counter() - t_wall) * 1e3
            return result
        if len(ground_truth) < n:
            raise RuntimeError("recovery: ground truth missing for completed chunks")
        for w in failure.failed_workers:
            result.recovered[w] = [None] * n
        for c in range(r):   # recompute lane stand-in: restore from the ground-truth slices
            for w in failure.failed_workers:
                result.recovered[w][c] = ground_truth[c][w]
        if e1 is not None:
            e1.synchronize()
        if r < n:
            result.reconstruct_device_ms = e0.elapsed_time(e1)
            for c_first, outs, out_index, _ in pending:
                for i in range(outs.shape[0]):
                    for b, w in enumerate(out_index):
                        result.recovered[w][c_first + i] = KvChunkSlice(request_id, c_first + i, w, outs[i, b],
                                                                        entries[c_first + i - r].valid_tokens)
            for w in failure.failed_workers:
                if any(result.recovered[w][c] is None for c in range(r, n)):
                    raise RuntimeError("recovery: codec did not return a failed shard")
        result.wall_ms = (time.perf_counter() - t_wall) * 1e3
        for c in range(r, n):
            for w in failure.failed_workers:
                if not verify_recovery(result.recovered[w][c], ground_truth[c][w]):
                    result.verified = False
        result.decoded_chunks = n - r if result.verified else 0
        return result

    def _verify_entries(self, entries, threads: int) -> List[bool]:
        """ParityChunk::compute_checksum == checksum for every entry, the
        chunks spread over host threads (gs_parity_checksum_batch)."""
        k = entries[0].scheme.k
        ln = entries[0].slice_len
        if any(e.scheme.k != k or e.slice_len != ln for e in entries):
            return [e.compute_checksum() == e.checksum for e in entries]
        ptrs = L.ptr_array([p.ctypes.data for e in entries for p in e.parity])
        out = (C.c_uint64 * len(entries))()
        check(L.lib().gs_parity_checksum_batch(ptrs, len(entries), k, ln, threads or (os.cpu_count() or 1), out),
              "verify")
        return [int(out[i]) == e.checksum for i, e in enumerate(entries)]

    def _split_plan(self, n: int, failed: Set[int], threads: int):
        """(n_full, u): how many of the n entries to verify entirely on the GPU
        and how many parity rows the decode uses. A GPU-verified ("full")
        entry uploads all k rows; a split entry uploads only the u rows K2
        needs, the GPU hashes them and a host thread continues the serial
        chain over the other k-u rows. n_full minimises
        max(link time, host time) with
          link = (n*u + n_full*(k-u)) L / B_link
          host = max(h*u*L / B_link + (k-u) L / chain_rate, h (k-u) L / fnv_rate),
        h = n - n_full (the last split chunk's rows land, then one serial chain)."""
        k = self.cfg.scheme.k
        u = max(1, min(k, len(failed)))
        if u >= k or n == 0:
            return n, u
        L_, bl = float(self.slice), self.cfg.cost.host_bw
        chain = (k - u) * L_ / self.host_chain_rate
        best, best_t = n, float("inf")
        for n_full in range(n + 1):
            h = n - n_full
            t_link = (n * u + n_full * (k - u)) * L_ / bl
            t_host = 0.0 if h == 0 else max(h * u * L_ / bl + chain, h * (k - u) * L_ / self.host_fnv_rate)
            t = max(t_link, t_host)
            if t < best_t - 1e-9:
                best, best_t = n_full, t
        return best, u

    def _enqueue_split_verified_decode(self, ground_truth, chunk_ids, entries, failed, threads: int):
        """Upload parity rows into HBM and verify every entry's checksum
        (gs_verify_enqueue: the first n_full entries entirely on the GPU, the
        rest GPU-hashed over the decode's rows and finished on host threads in
        a Python thread), then rebuild the lost shards with K2 from the
        uploaded rows."""
        sch = self.cfg.scheme
        dec = decoder(sch, ErasurePattern(sorted(failed)))
        S, k = len(chunk_ids), sch.k
        if self.verify_split == "dynamic":
            # every core: the chains are serial 80 MiB units, and with the
            # end-game hand-off the feeder absorbs a slow thread's tail
            # (tools/c3_endgame_ab.sh: 16 threads 101-102 ms vs 14: 103-110)
            threads = threads or max(1, os.cpu_count() or 1)
        threads = threads or max(1, (os.cpu_count() or 1) - 2)
        n_full, u = self._split_plan(S, failed, threads)
        if self.verify_split == "dynamic":
            n_full = -1            # gs_verify_enqueue: claim the rest of each chain at run time
        lib = L.lib()
        nf = max(n_full, 0)
        full = torch.empty((nf, k, self.slice), dtype=torch.uint8, device=self.dev)
        part = torch.empty((S - nf, u, self.slice), dtype=torch.uint8, device=self.dev)
        drows: List[Optional[int]] = []
        for s in range(S):
            for i in range(k):
                if s < nf:
                    drows.append(full[s, i].data_ptr())
                else:
                    drows.append(part[s - nf, i].data_ptr() if i < u else None)
        # K2 needs the uploaded rows (not their checksums, nor the rows the
        # dynamic split's GPU feeder uploads later for hashing only). In the
        # dynamic split it runs group by group as each group of 4 chunks lands
        # (gs_verify_stream_wait), under the remaining uploads: one K2 after the
        # last upload left ~8 ms of C3 rebuild (64 x 755 MB) behind the link.
        def build_tables():
            # allocated once the uploads are queued: a caching-allocator miss
            # maps 5 GiB (tens of ms), which then runs under the H2D instead of
            # delaying it
            outs = torch.empty((S, max(dec.n_out, 1), self.slice), dtype=torch.uint8, device=self.dev)
            launches = []
            if dec.n_out:
                slots: List[Optional[int]] = []
                for s, c in enumerate(chunk_ids):
                    row = self._survivor_row(ground_truth[c], failed)
                    for i in range(k):
                        row[sch.n + i] = drows[s * k + i]
                    slots.extend(row)
                optrs = [outs[s, b].data_ptr() for s in range(S) for b in range(dec.n_out)]
                w, no = sch.n + k, dec.n_out
                groups = [(0, S)] if not grouped else [(g0, min(g0 + 4, S)) for g0 in range(0, S, 4)]
                launches = [(g1 - 1, g1 - g0, L.ptr_array(slots[g0 * w:g1 * w]),
                             L.ptr_array(optrs[g0 * no:g1 * no])) for g0, g1 in groups]
            return outs, launches

        grouped = n_full < 0 and os.environ.get("GS_RECOVER_K2_GROUPS", "1") != "0"   # A/B switch
        handle = C.c_void_p()
        check(lib.gs_verify_enqueue(L.ptr_array([e.parity[i].ctypes.data for e in entries for i in range(k)]),
                                    S, k, self.slice, n_full, u, L.ptr_array(drows), self.verify.cuda_stream,
                                    self.copy.cuda_stream, C.byref(handle)), "recover verify")
        if not grouped:
            self.compute.wait_stream(self.copy)
        if n_full < 0:
            check(lib.gs_verify_set_rates(handle, self.cfg.cost.host_bw / 1e9, self.host_chain_rate / 1e9),
                  "recover verify")
        # the verification's host threads start now; the K2 launch tables are
        # built while the first uploads run, under a hold on the handle (finish
        # keeps the upload events until the launches are queued behind them)
        check(lib.gs_verify_hold(handle), "recover verify")
        try:
            finish = _VerifyFinish(handle, S, threads)
            outs, launches = build_tables()
            for last, cnt, sl, op in launches:
                if grouped:
                    check(lib.gs_verify_stream_wait(handle, last, self.compute.cuda_stream), "recover verify")
                check(lib.gs_apply_device(dec.handle, cnt, sl, op, self.slice, self.compute.cuda_stream),
                      "recover")
        finally:
            check(lib.gs_verify_release(handle), "recover verify")
        return outs, list(dec.out_index), n_full, finish, (full, part)

    def _survivor_row(self, gt, failed) -> List[Optional[int]]:
        sch = self.cfg.scheme
        row: List[Optional[int]] = [None] * (sch.n + sch.k)
        for sl in gt:
            if sl.worker not in failed:
                row[sl.worker] = sl.bytes.data_ptr()
        for j in range(sch.n):
            if j not in failed and row[j] is None:
                raise InvalidArgument(f"coding: surviving shard {j} missing from input")
        return row

    def _enqueue_batched_decode(self, ground_truth, chunk_ids, entries, failed):
        """One gs_reconstruct_upload over the chunks: H2D of the used parity
        rows from the host entries + K2, pieces pipelined."""
        sch = self.cfg.scheme
        dec = decoder(sch, ErasurePattern(sorted(failed)))
        S = len(chunk_ids)
        outs = torch.empty((S, max(dec.n_out, 1), self.slice), dtype=torch.uint8, device=self.dev)
        slots: List[Optional[int]] = []
        for c, e in zip(chunk_ids, entries):
            row = self._survivor_row(ground_truth[c], failed)
            for i in range(sch.k):
                row[sch.n + i] = e.parity[i].ctypes.data
            slots.extend(row)
        if dec.n_out:
            check(L.lib().gs_reconstruct_upload(self.pipe.handle, dec.handle, S, L.ptr_array(slots),
                                                L.ptr_array([outs[i, b].data_ptr() for i in range(S)
                                                             for b in range(dec.n_out)]),
                                                self.slice, self.compute.cuda_stream, self.copy.cuda_stream),
                  "recover")
        return outs, list(dec.out_index)


class DecodeCheckpointer:
    """checkpoint.hpp:228-281: buffer decode tokens, emit a chunk checkpoint
    every m tokens, flush the masked tail at request end."""

    def __init__(self, request_id: int, first_chunk_index: int, ckpt: Checkpointer, kv_seed: int = 0):
        ckpt.cfg.validate()
        self.request_id = request_id
        self.next_chunk = first_chunk_index
        self.ckpt = ckpt
        self.kv_seed = kv_seed
        self.buffered = 0
        self.ground_truth: List[List[KvChunkSlice]] = []

    def buffered_tokens(self) -> int:
        return self.buffered

    def step(self, state: AssignmentState) -> Optional[ChunkCheckpointOutcome]:
        self.buffered += 1
        if self.buffered < self.ckpt.cfg.chunk_size:
            return None
        return self._emit(state)

    def flush(self, state: AssignmentState) -> Optional[ChunkCheckpointOutcome]:
        if self.buffered == 0:
            return None
        return self._emit(state)

    def _emit(self, state: AssignmentState) -> ChunkCheckpointOutcome:
        valid = self.buffered
        slices = self.ckpt.make_slices(self.kv_seed, self.request_id, self.next_chunk, valid)
        out = self.ckpt.checkpoint_chunk(slices, state)
        self.ground_truth.append(slices)
        self.next_chunk += 1
        self.buffered = 0
        return out
