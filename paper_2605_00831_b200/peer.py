"""Multi-GPU striping over NVLink: one process per GPU, peers' KV shards read
in place through IPC-mapped pointers.

The paper gathers every worker's slice to one rotating encoder GPU with NCCL
(checkpoint.hpp:21-30) and offloads the whole chunk's
parity over that GPU's single PCIe link. Here every rank g encodes the byte
range g of ALL shards -- reading the ranges it does not own straight out of
the owners' HBM over NVLink inside K1 -- and D2H's parity range g on its own
host link. No reduction is involved (NCCL has no GF(2^8) op); the only
exchange on the data path is the peer loads, fused into the kernel. Recovery
mirrors it: rank g uploads parity range g, pulls range g of the survivors and
stores range g of the rebuilt shard directly into the replacement GPU's KV
buffer. The entries' checksums (one FNV-1a chain over a chunk's whole parity)
are relayed through the ranks' ranges as 8-byte chain states: through a board
in host memory the ranks of a node share (RelayBoard; host threads, and the
GPUs for rows in HBM), or in lockstep rounds of small all-gathers over any
process group (chain_striped).

Layout: with W ranks and n TP workers (W | n), rank r holds workers
[r*n/W, (r+1)*n/W) as a tensor [S, n/W, L] (S stripes = requests x chunks).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Callable, Dict, List, Optional, Sequence, Tuple

from . import _lib as L
from .coding import CodeKind, CodingScheme, ErasurePattern, InvalidArgument, check, decoder, encoder
from .device import row_ptrs


def stripe_range(total: int, rank: int, world: int) -> Tuple[int, int]:
    """4 KiB-aligned contiguous split of [0, total) (gs_stripe_range)."""
    off, ln = C.c_uint64(), C.c_uint64()
    check(L.lib().gs_stripe_range(total, rank, world, C.byref(off), C.byref(ln)), "stripe_range")
    return off.value, ln.value


@dataclass(frozen=True)
class ShardLayout:
    n: int          # TP workers = data shards
    world: int      # ranks (GPUs)
    stripes: int    # S
    length: int     # L bytes per shard per stripe

    def __post_init__(self):
        if self.world < 1 or self.n % self.world:
            raise InvalidArgument(f"layout: {self.world} ranks must divide {self.n} workers")

    @property
    def n_local(self) -> int:
        return self.n // self.world

    def owner(self, worker: int) -> Tuple[int, int]:
        return worker // self.n_local, worker % self.n_local

    def shard_offset(self, stripe: int, worker: int) -> int:
        """Byte offset of (stripe, worker) inside its owner's [S, n_local, L] tensor."""
        _, jl = self.owner(worker)
        return (stripe * self.n_local + jl) * self.length


def striped_slots(layout: ShardLayout, bases: Sequence[int], rank: int,
                  lost: Sequence[int] = ()) -> Tuple[int, int, List[List[Optional[int]]]]:
    """Rank `rank`'s byte range and per-stripe data-shard pointers into the
    owners' memory (`bases[r]` = rank r's tensor base as mapped locally).
    Lost workers get None."""
    off, ln = stripe_range(layout.length, rank, layout.world)
    slots = []
    for s in range(layout.stripes):
        row = []
        for j in range(layout.n):
            if j in lost:
                row.append(None)
            else:
                r, _ = layout.owner(j)
                row.append(bases[r] + layout.shard_offset(s, j) + off)
        slots.append(row)
    return off, ln, slots


class PeerGroup:
    """IPC-maps every rank's buffer into every other rank (same node)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = torch.cuda.current_device()
        self._opened: List[int] = []

    def share(self, tensor) -> List[int]:
        """All ranks' base pointers of `tensor` (collective)."""
        handle = (C.c_uint8 * L.IPC_HANDLE_BYTES)()
        off = C.c_uint64()
        check(L.lib().gs_ipc_handle(tensor.data_ptr(), handle, C.byref(off)), "ipc_handle")
        objs: List = [None] * self.world
        self.dist.all_gather_object(objs, (bytes(handle), off.value), group=self.group)
        ptrs = []
        for r, (h, o) in enumerate(objs):
            if r == self.rank:
                ptrs.append(tensor.data_ptr())
                continue
            base = C.c_void_p()
            hb = (C.c_uint8 * L.IPC_HANDLE_BYTES).from_buffer_copy(h)
            check(L.lib().gs_ipc_open(hb, self.device, C.byref(base)), "ipc_open")
            self._opened.append(base.value)
            ptrs.append(base.value + o)
        return ptrs

    def close(self) -> None:
        for p in self._opened:
            L.lib().gs_ipc_close(p)
        self._opened.clear()


class StripedCall:
    """A prepared striped encode / rebuild: pointer tables built once, so the
    timed path is a single C-ABI call (re-runnable, e.g. every decode step
    that reuses the same KV block buffers)."""

    def __init__(self, fn, args, offset: int, length: int, two_streams: bool = True):
        self.fn, self.args, self.offset, self.length = fn, args, offset, length
        self.two_streams = two_streams

    def run(self, stream: int, copy_stream: Optional[int] = None) -> None:
        if self.length == 0 or self.fn is None:
            return
        if not self.two_streams:
            check(self.fn(*self.args, stream), "striped")
            return
        check(self.fn(*self.args, stream, copy_stream if copy_stream is not None else stream), "striped")


def _host_rows(h_parity, off: int, local: bool) -> List[int]:
    """Row pointers p such that p + off is where byte `off` of each (stripe,
    parity row) lands: a full-width [S, k, L] host slab, or (local=True) a
    range-local [S, k, len_r] slab holding only this rank's byte range."""
    rows = row_ptrs(h_parity)
    return [r - off for r in rows] if local else rows


def require_position_independent(scheme: CodingScheme, layout: ShardLayout) -> None:
    """Byte-range striping needs a code whose parity byte b depends only on
    byte b of the shards (XOR, RS: coding.hpp:143-172, 269-275). RDP places
    cells at t*(p-1)+r and its P/Q tail at the END of the shard
    (coding.hpp:225-307), so a rank encoding its own range as a shard starting
    at 0 would produce a different code -- striped RDP is refused; the
    rotating encoder (whole stripes per rank) handles it."""
    if scheme.kind == CodeKind.RDP and layout.world > 1:
        raise InvalidArgument("striping: RDP parity depends on byte position; byte-range striping over "
                              f"{layout.world} ranks would not reproduce it (use plan_encode_rotating)")


def plan_encode_striped(scheme: CodingScheme, layout: ShardLayout, bases: Sequence[int], rank: int,
                        parity_out=None, pipeline=None, h_parity=None, local_parity: bool = False) -> StripedCall:
    """K1 over this rank's byte range of all stripes (see encode_striped).
    local_parity: h_parity is [S, k, len_r] (this rank's range only)."""
    require_position_independent(scheme, layout)
    enc = encoder(scheme)
    off, ln, slots = striped_slots(layout, bases, rank)
    if ln == 0:
        return StripedCall(None, (), off, 0)
    flat = L.ptr_array([p for row in slots for p in row])
    lib = L.lib()
    if pipeline is None:
        outs = L.ptr_array(row_ptrs(parity_out))
        return StripedCall(lib.gs_apply_device, (enc.handle, layout.stripes, flat, outs, ln), off, ln,
                           two_streams=False)
    outs = L.ptr_array([p + off for p in _host_rows(h_parity, off, local_parity)])
    return StripedCall(lib.gs_encode_offload, (pipeline.handle, enc.handle, layout.stripes, flat, outs, ln),
                       off, ln)


def rotating_stripes(layout: ShardLayout, rank: int, first_worker: int = 0) -> List[int]:
    """The paper's temporal balancing: stripe s is encoded
    whole by the GPU owning parity worker (first_worker + s) mod n, the
    reference's round-robin next_parity_worker (checkpoint.hpp:21-30)."""
    return [s for s in range(layout.stripes)
            if layout.owner((first_worker + s) % layout.n)[0] == rank]


def plan_encode_rotating(scheme: CodingScheme, layout: ShardLayout, bases: Sequence[int], rank: int,
                         pipeline, h_parity, first_worker: int = 0) -> StripedCall:
    """Comparison mode for the striped encoder: this rank
    gathers ALL n shards of its rotating stripes over NVLink (peer loads
    inside K1) and D2H's their whole parity through its own host link, so
    each stripe's parity crosses one link instead of W."""
    mine = rotating_stripes(layout, rank, first_worker)
    if not mine or layout.length == 0:
        return StripedCall(None, (), 0, 0)
    enc = encoder(scheme)
    slots = []
    for s in mine:
        for j in range(layout.n):
            r, _ = layout.owner(j)
            slots.append(bases[r] + layout.shard_offset(s, j))
    hp = row_ptrs(h_parity)
    k = scheme.k
    outs = [hp[s * k + i] for s in mine for i in range(k)]
    return StripedCall(L.lib().gs_encode_offload, (pipeline.handle, enc.handle, len(mine), L.ptr_array(slots),
                                                   L.ptr_array(outs), layout.length), 0, layout.length)


def encode_striped(scheme: CodingScheme, layout: ShardLayout, bases: Sequence[int], rank: int,
                   parity_out, stream: int, pipeline=None, h_parity=None, copy_stream=None) -> Tuple[int, int]:
    """K1 over this rank's byte range of all stripes.

    Without a pipeline: parity range -> `parity_out` device [S, k, len_r].
    With a pipeline: parity range -> pinned host `h_parity` [S, k, L] at the
    range's offset (encode + D2H overlapped on this rank's host link)."""
    call = plan_encode_striped(scheme, layout, bases, rank, parity_out, pipeline, h_parity)
    call.run(stream, copy_stream)
    return call.offset, call.length


def plan_reconstruct_striped(scheme: CodingScheme, layout: ShardLayout, bases: Sequence[int], rank: int,
                             lost: ErasurePattern, h_parity, pipeline, local_parity: bool = False) -> StripedCall:
    """K2 over this rank's byte range (see reconstruct_striped).
    local_parity: h_parity is [S, k, len_r] (this rank's range only)."""
    require_position_independent(scheme, layout)
    dec = decoder(scheme, lost)
    off, ln, slots = striped_slots(layout, bases, rank, lost.lost)
    if ln == 0 or dec.n_out == 0:
        return StripedCall(None, (), off, 0)
    n, k = scheme.n, scheme.k
    hp = _host_rows(h_parity, off, local_parity)
    full = []
    for s in range(layout.stripes):
        full.extend(slots[s])
        for i in range(k):
            full.append(None if lost.contains(n + i) else hp[s * k + i] + off)
    outs = []
    for s in range(layout.stripes):
        for w in dec.out_index:
            r, _ = layout.owner(w)
            outs.append(bases[r] + layout.shard_offset(s, w) + off)
    return StripedCall(L.lib().gs_reconstruct_upload,
                       (pipeline.handle, dec.handle, layout.stripes, L.ptr_array(full), L.ptr_array(outs), ln),
                       off, ln)


FNV_OFFSET = 0xcbf29ce484222325  # ParityChunk checksum seed (parity_store.hpp:19-53)


def dist_exchange(group=None) -> Callable:
    """Token exchange for chain_striped over torch.distributed (a CPU-tensor
    backend: gloo). Returns ex(local [m] uint64) -> [world, m] uint64."""
    import numpy as np
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)

    def ex(local):
        t = torch.from_numpy(np.ascontiguousarray(local).view(np.int64).copy())
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t, group=group)
        return np.stack([p.numpy() for p in parts]).view(np.uint64)

    return ex


def chain_striped(rows: Sequence[int], length: int, n_chunks: int, k: int, rank: int, world: int,
                  exchange: Callable, threads: int = 0, h0: int = FNV_OFFSET) -> List[int]:
    """ParityChunk checksums of chunks whose parity is byte-range striped over
    the ranks: the reference seals a chunk with ONE FNV-1a chain over its k
    rows in order (ParityChunk::compute_checksum, parity_store.hpp:19-53;
    verified on get, :92-101, before recover decodes, recovery.hpp:269-296),
    so at N>1 the chain runs through the ranks' ranges: (row 0, rank 0),
    (row 0, rank 1), ..., (row k-1, rank W-1). Every rank runs this with
    `rows[c*k + i]` = the host address of ITS range of parity row i of chunk c
    (`length` bytes, 0 for an empty range) and gets every chunk's checksum.

    Wavefront relay: chunk c enters the ring `c mod W` rounds late, so in
    round t chunk c is at chain position p = t - (c mod W) on rank p mod W --
    every rank continues n_chunks/W chains per round (host threads,
    gs_fnv1a64_continue_batch) and one all-gather of the 8-byte states hands
    them to the next rank. k*W + W - 1 rounds; a rank's host work is its own
    bytes only. The states passed on are plain FNV states: no hypotheses."""
    import numpy as np

    if n_chunks <= 0:
        return []
    npos = k * world
    state = np.full(n_chunks, h0 & 0xFFFFFFFFFFFFFFFF, dtype=np.uint64)
    if threads <= 0:
        threads = max(1, (os.cpu_count() or 1) // world)
    lib = L.lib()
    for t in range(npos + world - 1):
        mine, owner = [], np.full(n_chunks, -1, dtype=np.int64)
        for c in range(n_chunks):
            p = t - (c % world)
            if 0 <= p < npos:
                owner[c] = p % world
                if p % world == rank:
                    mine.append((c, p // world))
        if mine:
            m = len(mine)
            bufs = L.ptr_array([rows[c * k + i] if length else None for c, i in mine])
            lens = (C.c_uint64 * m)(*([length] * m))
            hin = (C.c_uint64 * m)(*[int(state[c]) for c, _ in mine])
            hout = (C.c_uint64 * m)()
            check(lib.gs_fnv1a64_continue_batch(bufs, lens, hin, hout, m, threads), "chain_striped")
            for q, (c, _) in enumerate(mine):
                state[c] = hout[q]
        if world > 1:
            got = exchange(state)
            act = owner >= 0
            state[act] = got[owner[act], np.nonzero(act)[0]]
    return [int(x) for x in state]


def verify_striped(rows: Sequence[int], length: int, n_chunks: int, k: int, rank: int, world: int,
                   exchange, expected: Sequence[int], threads: int = 0) -> List[bool]:
    """ParityStore::get's check at N>1: chunk c's striped parity is intact iff
    its relayed checksum equals the sealed one (every rank gets the same
    verdicts). `exchange`: a round exchange (dist_exchange) or a RelayBoard."""
    if isinstance(exchange, RelayBoard):
        got = exchange.chain(rows, length, n_chunks, k, threads=threads)
    else:
        got = chain_striped(rows, length, n_chunks, k, rank, world, exchange, threads)
    return [g == (e & 0xFFFFFFFFFFFFFFFF) for g, e in zip(got, expected)]


class RelayBoard:
    """chain_striped without rounds for the ranks of one node: the chain states
    go through a board in host memory the ranks' processes share (a /dev/shm
    file mapped by every rank, unlinked once all have it), and each rank's
    threads continue its segments as soon as their predecessors' states
    appear (gs_fnv_relay). Collective: construct, chain() and close() on
    every rank of `group` in the same order."""

    def __init__(self, max_chunks: int, k: int, group=None, timeout_s: float = 120.0):
        import mmap
        import tempfile
        import uuid

        import torch.distributed as dist

        self.dist, self.group, self.timeout_s = dist, group, timeout_s
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.slots = max_chunks * k
        size = int(L.lib().gs_relay_board_bytes(max_chunks, k, self.world))
        if size == 0:
            raise InvalidArgument("RelayBoard: bad shape")
        shm = "/dev/shm" if os.path.isdir("/dev/shm") else tempfile.gettempdir()
        name = [os.path.join(shm, f"gs-relay-{os.getpid()}-{uuid.uuid4().hex[:12]}") if self.rank == 0 else None]
        dist.broadcast_object_list(name, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                   group=group)
        self.path = name[0]
        if self.rank == 0:
            fd = os.open(self.path, os.O_CREAT | os.O_EXCL | os.O_RDWR, 0o600)
            os.ftruncate(fd, size)  # zero-filled: every tag starts at epoch 0
            os.close(fd)
        dist.barrier(group=group)
        fd = os.open(self.path, os.O_RDWR)
        try:
            self._mm = mmap.mmap(fd, size)
        finally:
            os.close(fd)
        self._view = (C.c_char * size).from_buffer(self._mm)
        self.addr = C.addressof(self._view)
        dist.barrier(group=group)
        if self.rank == 0:
            os.unlink(self.path)
        self.epoch = 0

    def chain(self, rows: Sequence[int], length: int, n_chunks: int, k: int, threads: int = 0,
              h0: int = FNV_OFFSET) -> List[int]:
        """chain_striped's result (every chunk's checksum, on every rank)."""
        if n_chunks * k > self.slots:
            raise InvalidArgument(f"RelayBoard: {n_chunks} x {k} segments exceed the board's {self.slots}")
        if n_chunks <= 0:
            return []
        if threads <= 0:
            threads = max(1, (os.cpu_count() or 1) // self.world)
        self.epoch += 1
        sums = (C.c_uint64 * n_chunks)()
        bufs = L.ptr_array(list(rows) if length else [])
        st = L.lib().gs_fnv_relay(self.addr, self.epoch, self.rank, self.world, bufs, length, n_chunks, k,
                                  h0 & 0xFFFFFFFFFFFFFFFF, threads, self.timeout_s, sums)
        # the next call re-tags the slots: nobody may still be reading this epoch
        self.dist.barrier(group=self.group)
        check(st, "fnv_relay")
        return list(sums)

    def chain_device(self, d_rows: Sequence[int], k_dev: int, h_rows: Sequence[int], length: int, n_chunks: int,
                     k: int, stream: int, ready: Optional[Sequence] = None, threads: int = 0, batch: int = 8,
                     h0: int = FNV_OFFSET) -> List[int]:
        """chain() with rows 0..k_dev-1 of every chunk hashed on this rank's
        GPU (gs_fnv_relay_device): d_rows[c*k_dev + i] = device address of this
        rank's range of row i of chunk c, h_rows[c*k + i] = host address (rows
        >= k_dev are read), ready[c] = a torch.cuda.Event recorded once chunk
        c's device rows are complete (None: already complete). Runs on the
        calling thread's current device."""
        if n_chunks * k > self.slots:
            raise InvalidArgument(f"RelayBoard: {n_chunks} x {k} segments exceed the board's {self.slots}")
        if n_chunks <= 0:
            return []
        if threads <= 0:
            threads = max(1, (os.cpu_count() or 1) // self.world)
        self.epoch += 1
        sums = (C.c_uint64 * n_chunks)()
        dev = L.ptr_array(list(d_rows) if length and k_dev else [])
        host = L.ptr_array(list(h_rows) if length and k_dev < k else [])
        evs = L.ptr_array([e.cuda_event if e is not None else None for e in ready]) if ready is not None else None
        st = L.lib().gs_fnv_relay_device(self.addr, self.epoch, self.rank, self.world, dev, k_dev, evs, host, length,
                                         n_chunks, k, h0 & 0xFFFFFFFFFFFFFFFF, threads, batch, stream,
                                         self.timeout_s, sums)
        self.dist.barrier(group=self.group)
        check(st, "fnv_relay_device")
        return list(sums)

    def close(self) -> None:
        if getattr(self, "_mm", None) is not None:
            del self._view
            self._mm.close()
            self._mm = None


def plan_reconstruct_striped_device(scheme: CodingScheme, layout: ShardLayout, bases: Sequence[int], rank: int,
                                    lost: ErasurePattern, d_parity: Sequence[Sequence[Optional[int]]],
                                    stripes: Sequence[int]) -> StripedCall:
    """K2 over this rank's byte range of `stripes` with the parity already in
    this GPU's HBM (uploaded by the caller, e.g. to checksum it there too):
    d_parity[s][i] = device address of this rank's range of parity row i of
    stripe s, None for a row not uploaded (the decoder reads only the first e
    surviving rows, coding.hpp:540-544). Survivors over NVLink, rebuilt range
    stored into the owners' buffers; one gs_apply_device launch."""
    require_position_independent(scheme, layout)
    dec = decoder(scheme, lost)
    off, ln, slots = striped_slots(layout, bases, rank, lost.lost)
    if ln == 0 or dec.n_out == 0 or not stripes:
        return StripedCall(None, (), off, 0)
    n, k = scheme.n, scheme.k
    full, outs = [], []
    for s in stripes:
        full.extend(slots[s])
        for i in range(k):
            full.append(None if lost.contains(n + i) else d_parity[s][i])
        for w in dec.out_index:
            r, _ = layout.owner(w)
            outs.append(bases[r] + layout.shard_offset(s, w) + off)
    return StripedCall(L.lib().gs_apply_device, (dec.handle, len(stripes), L.ptr_array(full), L.ptr_array(outs), ln),
                       off, ln, two_streams=False)


def reconstruct_striped(scheme: CodingScheme, layout: ShardLayout, bases: Sequence[int], rank: int,
                        lost: ErasurePattern, h_parity, pipeline, stream: int,
                        copy_stream: Optional[int] = None) -> Tuple[int, int]:
    """K2 over this rank's byte range: parity range H2D'd from this rank's
    pinned host slab, survivors pulled from peers, rebuilt bytes stored
    straight into the lost workers' buffers (on their owners' GPUs)."""
    call = plan_reconstruct_striped(scheme, layout, bases, rank, lost, h_parity, pipeline)
    call.run(stream, copy_stream)
    return call.offset, call.length
