"""Multi-GPU striping, world_size 2.

CPU (gloo): the host-side partition and pointer arithmetic of
paper_2605_00831_b200.peer -- rank r's byte range of every shard, resolved
through the owners' base addresses -- reassembles exactly the full parity /
rebuilt shard (checked with the CPU oracle).

GPU (gloo for the handle exchange, one B200 shared by both processes): the
real path -- IPC-mapped peer buffers read inside K1, parity ranges D2H'd to
each rank's pinned slab, K2 storing rebuilt bytes straight into the owner's
buffer through its IPC mapping.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
from fuzzutil import fuzz_trials
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from tests.golden.vectors import splitmix_bytes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N, K, S, LEN = 8, 2, 3, 3 * 4096 + 80


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _shards(stripe):
    return [splitmix_bytes(1000 * stripe + j, LEN) for j in range(N)]


def _cpu_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    from paper_2605_00831_b200.peer import ShardLayout, striped_slots
    try:
        _init(rank, world, port)
        lay = ShardLayout(N, world, S, LEN)
        mine = np.stack([np.stack(_shards(s)[rank * lay.n_local:(rank + 1) * lay.n_local]) for s in range(S)])
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)          # stands in for the IPC mapping
        bases = [g.ctypes.data for g in gathered]
        off, ln, slots = striped_slots(lay, bases, rank)
        port_lib = O.port()
        parts = []
        for s in range(S):
            data = [np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint8)), (ln,)).copy() for p in slots[s]]
            parts.append(port_lib.encode(O.RS, N, K, data) if ln else [np.zeros(0, np.uint8)] * K)
        out = [None] * world
        dist.all_gather_object(out, (off, ln, parts))
        if rank == 0:
            for s in range(S):
                full = O.port().encode(O.RS, N, K, _shards(s))
                got = [np.zeros(LEN, np.uint8) for _ in range(K)]
                covered = 0
                for (o, l_, pr) in out:
                    for i in range(K):
                        got[i][o:o + l_] = pr[s][i]
                    covered += l_
                assert covered == LEN
                for i in range(K):
                    assert np.array_equal(got[i], full[i])
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


def _run(target, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=target, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res


def test_striped_partition_reassembles_parity_cpu():
    _run(_cpu_worker)


def _relay_worker(rank, world, port, q, length=5 * 4096 + 123, chunks=7, k=2):
    """chain_striped: every rank holds only its byte range of each parity row;
    the relayed checksums equal ParityChunk::compute_checksum of the whole
    rows (oracle), on every rank; a flipped byte fails exactly its chunk."""
    import sys
    sys.path.insert(0, ROOT)
    try:
        from paper_2605_00831_b200.peer import (RelayBoard, chain_striped, dist_exchange, stripe_range,
                                                verify_striped)
        _init(rank, world, port)
        rows = [splitmix_bytes(7000 + r, length) for r in range(chunks * k)]
        want = [O.port().parity_checksum(rows[c * k:(c + 1) * k]) for c in range(chunks)]
        off, ln = stripe_range(length, rank, world)
        local = [np.ascontiguousarray(r[off:off + ln]) for r in rows]
        ptrs = [a.ctypes.data if ln else 0 for a in local]
        ex = dist_exchange()
        board = RelayBoard(chunks + 3, k)
        got = chain_striped(ptrs, ln, chunks, k, rank, world, ex, threads=2)
        assert got == want, (rank, got, want)
        for threads in (1, 3):  # the shared-memory relay, repeated on one board (epochs)
            assert board.chain(ptrs, ln, chunks, k, threads=threads) == want, (rank, threads)
        assert board.chain(ptrs[:2 * k], ln, 2, k) == want[:2]
        ok = verify_striped(ptrs, ln, chunks, k, rank, world, ex, want, threads=3)
        assert all(ok)
        # corrupt one byte of chunk 4, row 1, in the LAST rank's range: every rank must
        # see chunk 4 (and only chunk 4) fail
        if rank == world - 1 and ln:
            local[4 * k + 1][ln // 2] ^= 0x5A
        dist.barrier()
        last = stripe_range(length, world - 1, world)[1]
        expect = [c != 4 or last == 0 for c in range(chunks)]
        ok = verify_striped(ptrs, ln, chunks, k, rank, world, ex, want, threads=1)
        assert ok == expect, (rank, ok)
        assert verify_striped(ptrs, ln, chunks, k, rank, world, board, want, threads=2) == expect
        board.close()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


def test_striped_checksum_relay_cpu():
    _run(_relay_worker)


def test_striped_checksum_relay_three_ranks_ragged_cpu():
    # 3 ranks over 5 pages + 123 bytes: 4 KiB-aligned ranges of unequal length
    _run(_relay_worker, world=3)


def test_striped_checksum_relay_single_rank():
    import sys
    sys.path.insert(0, ROOT)
    from paper_2605_00831_b200.peer import chain_striped
    rows = [splitmix_bytes(90 + r, 3000 + r) for r in range(6)]
    # one rank: the chain is plain ParityChunk::compute_checksum (equal row lengths)
    rows = [r[:3000] for r in rows]
    ptrs = [r.ctypes.data for r in rows]
    got = chain_striped(ptrs, 3000, 3, 2, 0, 1, exchange=None, threads=2)
    assert got == [O.port().parity_checksum(rows[2 * c:2 * c + 2]) for c in range(3)]
    assert chain_striped([], 0, 0, 2, 0, 1, exchange=None) == []


def _relay_fuzz_worker(rank, world, port, q):
    """Random shapes for both relay forms: k = 1..3 rows, 1..9 chunks, lengths
    from a few bytes (most ranks' ranges empty) to several pages plus a ragged
    tail, every chain checked against the oracle's ParityChunk checksum."""
    import random
    import sys
    sys.path.insert(0, ROOT)
    try:
        from paper_2605_00831_b200.peer import RelayBoard, chain_striped, dist_exchange, stripe_range
        _init(rank, world, port)
        ex = dist_exchange()
        board = RelayBoard(9, 3)
        rng = random.Random(1234)   # same draws on every rank
        for trial in range(fuzz_trials(12)):
            k = rng.randint(1, 3)
            chunks = rng.randint(1, 9)
            length = rng.choice([rng.randint(1, 64), rng.randint(1, 4096 * world), rng.randint(4096, 6 * 4096 + 999)])
            rows = [splitmix_bytes(10_000 * trial + r, length) for r in range(chunks * k)]
            want = [O.port().parity_checksum(rows[c * k:(c + 1) * k]) for c in range(chunks)]
            off, ln = stripe_range(length, rank, world)
            local = [np.ascontiguousarray(r[off:off + ln]) for r in rows]
            ptrs = [a.ctypes.data if ln else 0 for a in local]
            got_r = chain_striped(ptrs, ln, chunks, k, rank, world, ex, threads=rng.randint(1, 3))
            got_b = board.chain(ptrs, ln, chunks, k, threads=rng.randint(1, 3))
            assert got_r == want and got_b == want, (rank, trial, k, chunks, length)
        board.close()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


def test_striped_checksum_relay_fuzz_cpu():
    _run(_relay_fuzz_worker, world=3)


def test_relay_board_times_out_without_the_peer():
    """A rank whose predecessor never delivers fails (GS_RUNTIME_ERROR) after the
    timeout instead of spinning forever; rank 0 of a 2-rank relay alone can
    only do its own row-0 segments."""
    import sys
    sys.path.insert(0, ROOT)
    from paper_2605_00831_b200 import _lib as L
    lib = L.lib()
    nbytes = lib.gs_relay_board_bytes(3, 2, 2)
    assert nbytes == 3 * 2 * 2 * 16 and lib.gs_relay_board_bytes(3, 0, 2) == 0
    board = (C.c_uint8 * nbytes)()
    rows = [splitmix_bytes(r, 4096) for r in range(6)]
    ptrs = L.ptr_array([r.ctypes.data for r in rows])
    sums = (C.c_uint64 * 3)()
    st = lib.gs_fnv_relay(board, 1, 1, 2, ptrs, 4096, 3, 2, 0xcbf29ce484222325, 2, 0.2, sums)
    assert st == L.GS_RUNTIME_ERROR and b"timed out" in lib.gs_last_error()
    assert lib.gs_fnv_relay(board, 0, 0, 2, ptrs, 4096, 3, 2, 1, 1, 0.2, sums) == L.GS_INVALID_ARGUMENT
    assert lib.gs_fnv_relay(board, 2, 2, 2, ptrs, 4096, 3, 2, 1, 1, 0.2, sums) == L.GS_INVALID_ARGUMENT


def _enable_peers(rank, world):
    """Distinct devices: peer access both ways (gs_peer_enable), on top of the
    lazy peer access the IPC mapping requests (cudaIpcMemLazyEnablePeerAccess)."""
    from paper_2605_00831_b200 import _lib as L
    for r in range(world):
        if r != rank:
            assert L.lib().gs_peer_enable(rank, r) == 0, L.last_error()


def _gpu_worker(rank, world, port, q, distinct=False):
    import sys
    sys.path.insert(0, ROOT)
    try:
        dev = rank if distinct else 0
        torch.cuda.set_device(dev)
        if distinct:
            _enable_peers(rank, world)
        from paper_2605_00831_b200 import device as D
        from paper_2605_00831_b200.coding import CodingScheme, ErasurePattern
        from paper_2605_00831_b200.peer import (PeerGroup, ShardLayout, encode_striped,
                                                reconstruct_striped)
        _init(rank, world, port)
        scheme = CodingScheme.reed_solomon(N, K)
        lay = ShardLayout(N, world, S, LEN)
        nl = lay.n_local
        mine = torch.stack([torch.from_numpy(np.stack(_shards(s)[rank * nl:(rank + 1) * nl])) for s in range(S)]).cuda()
        pg = PeerGroup()
        bases = pg.share(mine)
        h_par = torch.zeros((S, K, LEN), dtype=torch.uint8).pin_memory()
        pipe = D.Pipeline(dev, 1 << 20)
        comp, copy = torch.cuda.Stream(), torch.cuda.Stream()
        torch.cuda.synchronize()
        dist.barrier()
        off, ln = encode_striped(scheme, lay, bases, rank, None, comp.cuda_stream, pipeline=pipe,
                                 h_parity=h_par, copy_stream=copy.cuda_stream)
        copy.synchronize()
        torch.cuda.synchronize()
        parts = [None] * world
        dist.all_gather_object(parts, (off, ln, h_par[:, :, off:off + ln].clone().numpy()))
        full = np.zeros((S, K, LEN), np.uint8)
        for (o, l_, arr) in parts:
            full[:, :, o:o + l_] = arr
        for s in range(S):
            want = O.port().encode(O.RS, N, K, _shards(s))
            for i in range(K):
                assert np.array_equal(full[s, i], want[i]), (rank, s, i)
        # the entries' seal at N>1: checksums relayed through the ranks' ranges of
        # the pinned slabs equal ParityChunk::compute_checksum of the whole parity
        from paper_2605_00831_b200.peer import chain_striped, dist_exchange
        sums = chain_striped([p + off for p in D.row_ptrs(h_par)], ln, S, K, rank, world, dist_exchange())
        assert sums == [O.port().parity_checksum(list(full[s])) for s in range(S)], rank
        # every rank holds the full parity in its host slab now (stands in for
        # the shared host tier); lose worker 5 (owned by the last rank), zero
        # its buffer, rebuild striped: each rank writes its byte range of the
        # shard straight into the owner's memory through the IPC mapping.
        h_par.copy_(torch.from_numpy(full))
        lost = 5
        owner, jl = lay.owner(lost)
        if rank == owner:
            mine[:, jl].zero_()
        torch.cuda.synchronize()
        dist.barrier()
        reconstruct_striped(scheme, lay, bases, rank, ErasurePattern([lost]), h_par, pipe, comp.cuda_stream,
                            copy.cuda_stream)
        comp.synchronize()
        torch.cuda.synchronize()
        dist.barrier()
        if rank == owner:
            got = mine[:, jl].cpu().numpy()
            for s in range(S):
                assert np.array_equal(got[s], _shards(s)[lost]), s
        dist.barrier()
        pg.close()
        pipe.close()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.gpu
def test_ipc_striped_encode_and_rebuild_two_processes_one_gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device")
    _run(_gpu_worker)


def _gpu_worker_local(rank, world, port, q, distinct=False):
    """The C3 flow at N ranks: each rank keeps ONLY its byte range of the
    parity in a range-local pinned slab ([S, K, len_r]), and rebuilds from it."""
    import sys
    sys.path.insert(0, ROOT)
    try:
        dev = rank if distinct else 0
        torch.cuda.set_device(dev)
        if distinct:
            _enable_peers(rank, world)
        from paper_2605_00831_b200 import device as D
        from paper_2605_00831_b200.coding import CodingScheme, ErasurePattern
        from paper_2605_00831_b200.peer import (PeerGroup, ShardLayout, plan_encode_striped,
                                                plan_reconstruct_striped)
        _init(rank, world, port)
        scheme = CodingScheme.reed_solomon(N, K)
        lay = ShardLayout(N, world, S, LEN)
        nl = lay.n_local
        mine = torch.stack([torch.from_numpy(np.stack(_shards(s)[rank * nl:(rank + 1) * nl])) for s in range(S)]).cuda()
        pg = PeerGroup()
        bases = pg.share(mine)
        pipe = D.Pipeline(dev, 1 << 20)
        comp, copy = torch.cuda.Stream(), torch.cuda.Stream()
        from paper_2605_00831_b200.peer import stripe_range
        off, ln = stripe_range(LEN, rank, world)
        h_loc = torch.zeros((S, K, max(ln, 16)), dtype=torch.uint8).pin_memory()
        torch.cuda.synchronize()
        dist.barrier()
        enc = plan_encode_striped(scheme, lay, bases, rank, pipeline=pipe, h_parity=h_loc, local_parity=True)
        enc.run(comp.cuda_stream, copy.cuda_stream)
        copy.synchronize()
        torch.cuda.synchronize()
        for s in range(S):
            want = O.port().encode(O.RS, N, K, _shards(s))
            for i in range(K):
                assert np.array_equal(h_loc[s, i, :ln].numpy(), want[i][off:off + ln]), (rank, s, i)
        lost = 2
        owner, jl = lay.owner(lost)
        dist.barrier()
        if rank == owner:
            mine[:, jl].zero_()
        torch.cuda.synchronize()
        dist.barrier()
        rec = plan_reconstruct_striped(scheme, lay, bases, rank, ErasurePattern([lost]), h_loc, pipe,
                                       local_parity=True)
        rec.run(comp.cuda_stream, copy.cuda_stream)
        comp.synchronize()
        torch.cuda.synchronize()
        dist.barrier()
        if rank == owner:
            got = mine[:, jl].cpu().numpy()
            for s in range(S):
                assert np.array_equal(got[s], _shards(s)[lost]), s
        dist.barrier()
        # Verified rebuild from parity uploaded to HBM: the entries' checksums
        # relayed through the ranks with row 0 hashed on the GPUs (seeded window
        # kernel) and row 1 on host threads, then K2 reading the device rows.
        from paper_2605_00831_b200.peer import RelayBoard, plan_reconstruct_striped_device
        want_sums = [O.port().parity_checksum(O.port().encode(O.RS, N, K, _shards(s))) for s in range(S)]
        board = RelayBoard(S, K)
        d_loc = h_loc.to(torch.device("cuda", dev), non_blocking=True)
        ready = torch.cuda.Event()
        ready.record()
        hrows = [h_loc[s, i].data_ptr() for s in range(S) for i in range(K)]
        for k_dev in (0, 1, 2):
            d_rows = [d_loc[s, i].data_ptr() for s in range(S) for i in range(k_dev)]
            got = board.chain_device(d_rows, k_dev, hrows, ln, S, K, comp.cuda_stream, ready=[ready] * S,
                                     threads=2, batch=2)
            assert got == want_sums, (rank, k_dev, got, want_sums)
        if rank == world - 1:   # one flipped device byte of chunk 1: chunk 1 (only) fails on every rank
            d_loc[1, 0, 5] ^= 1
        torch.cuda.synchronize()
        dist.barrier()
        got = board.chain_device([d_loc[s, 0].data_ptr() for s in range(S)], 1, hrows, ln, S, K, comp.cuda_stream)
        assert [g == w for g, w in zip(got, want_sums)] == [s != 1 for s in range(S)], (rank, got)
        if rank == world - 1:
            d_loc[1, 0, 5] ^= 1
        board.close()
        if rank == owner:
            mine[:, jl].zero_()
        torch.cuda.synchronize()
        dist.barrier()
        plan_reconstruct_striped_device(scheme, lay, bases, rank, ErasurePattern([lost]),
                                        [[d_loc[s, 0].data_ptr(), None] for s in range(S)],
                                        range(S)).run(comp.cuda_stream)
        comp.synchronize()
        torch.cuda.synchronize()
        dist.barrier()
        if rank == owner:
            got = mine[:, jl].cpu().numpy()
            for s in range(S):
                assert np.array_equal(got[s], _shards(s)[lost]), ("device-parity rebuild", s)
        dist.barrier()
        pg.close()
        pipe.close()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))


def _relay_device_fuzz_worker(rank, world, port, q):
    """chain_device over random shapes: k = 1..3 rows of which k_dev = 0..k in
    HBM (the rest on host threads), 1..9 chunks, 16-B-multiple lengths from
    one granule to several pages, batches of 1..4 chunks per GPU launch, with
    and without ready events -- every chain against the oracle."""
    import random
    import sys
    sys.path.insert(0, ROOT)
    try:
        torch.cuda.set_device(0)
        from paper_2605_00831_b200.peer import RelayBoard, stripe_range
        _init(rank, world, port)
        board = RelayBoard(9, 3)
        stream = torch.cuda.Stream()
        rng = random.Random(77)
        for trial in range(fuzz_trials(10)):
            k = rng.randint(1, 3)
            k_dev = rng.randint(0, k)
            chunks = rng.randint(1, 9)
            length = 16 * rng.choice([1, rng.randint(1, 256 * world), rng.randint(256, 2048)])
            rows = [splitmix_bytes(50_000 * trial + r, length) for r in range(chunks * k)]
            want = [O.port().parity_checksum(rows[c * k:(c + 1) * k]) for c in range(chunks)]
            off, ln = stripe_range(length, rank, world)
            host = torch.stack([torch.from_numpy(np.ascontiguousarray(r[off:off + ln])) for r in rows]) \
                if ln else torch.zeros((chunks * k, 16), dtype=torch.uint8)
            dev = host.cuda()
            ev = torch.cuda.Event()
            ev.record()
            d_rows = [dev[c * k + i].data_ptr() for c in range(chunks) for i in range(k_dev)]
            h_rows = [host[c * k + i].data_ptr() for c in range(chunks) for i in range(k)]
            ready = [ev] * chunks if rng.random() < 0.5 else None
            got = board.chain_device(d_rows, k_dev, h_rows, ln, chunks, k, stream.cuda_stream, ready=ready,
                                     threads=rng.randint(1, 3), batch=rng.randint(1, 4))
            assert got == want, (rank, trial, k, k_dev, chunks, length)
        board.close()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.gpu
def test_striped_checksum_relay_on_gpus_fuzz_two_processes_one_gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device")
    _run(_relay_device_fuzz_worker)


@pytest.mark.gpu
def test_ipc_striped_range_local_parity_two_processes_one_gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device")
    _run(_gpu_worker_local)


@pytest.mark.gpu
@pytest.mark.parametrize("worker", ["full", "range_local"])
def test_ipc_striped_two_distinct_devices(worker):
    """The same striped encode + rebuild with each rank on its OWN GPU: K1
    reads the peer's shards over NVLink through the IPC mapping, K2 stores
    the rebuilt range into the owner's HBM on the other device (peer access
    enabled both ways). Needs two visible GPUs (skipped on a 1-GPU box)."""
    import functools
    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device")
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 visible GPUs (this box has 1)")
    _run(functools.partial(_gpu_worker if worker == "full" else _gpu_worker_local, distinct=True))


def test_rotating_assignment_covers_every_stripe_once():
    """Rotating mode: every stripe is encoded by exactly one rank, the owner
    of the round-robin parity worker (checkpoint.hpp:21-30)."""
    from paper_2605_00831_b200.peer import ShardLayout, rotating_stripes
    for world in (1, 2, 4, 8):
        for first in (0, 3, 7):
            lay = ShardLayout(8, world, 37, 4096)
            got = sorted(s for r in range(world) for s in rotating_stripes(lay, r, first))
            assert got == list(range(37))
            for r in range(world):
                for s in rotating_stripes(lay, r, first):
                    assert lay.owner((first + s) % 8)[0] == r


def _gpu_rotating_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    try:
        torch.cuda.set_device(0)
        from paper_2605_00831_b200 import device as D
        from paper_2605_00831_b200.coding import CodingScheme
        from paper_2605_00831_b200.peer import PeerGroup, ShardLayout, plan_encode_rotating, rotating_stripes
        _init(rank, world, port)
        scheme = CodingScheme.reed_solomon(N, K)
        lay = ShardLayout(N, world, S, LEN)
        nl = lay.n_local
        mine = torch.stack([torch.from_numpy(np.stack(_shards(s)[rank * nl:(rank + 1) * nl])) for s in range(S)]).cuda()
        pg = PeerGroup()
        bases = pg.share(mine)
        h_par = torch.zeros((S, K, LEN), dtype=torch.uint8).pin_memory()
        pipe = D.Pipeline(0, 1 << 20)
        comp, copy = torch.cuda.Stream(), torch.cuda.Stream()
        torch.cuda.synchronize()
        dist.barrier()
        plan_encode_rotating(scheme, lay, bases, rank, pipe, h_par, first_worker=1).run(comp.cuda_stream,
                                                                                         copy.cuda_stream)
        copy.synchronize()
        torch.cuda.synchronize()
        for s in rotating_stripes(lay, rank, 1):
            want = O.port().encode(O.RS, N, K, _shards(s))
            for i in range(K):
                assert np.array_equal(h_par[s, i].numpy(), want[i]), (rank, s, i)
        dist.barrier()
        pg.close()
        pipe.close()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.gpu
def test_ipc_rotating_encode_two_processes_one_gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device")
    _run(_gpu_rotating_worker)


def test_striped_partition_fuzz_single_process():
    """Random TP widths, world sizes (dividing n), stripe counts and lengths:
    every rank's byte range of every shard, resolved through the owners' base
    addresses (all ranks simulated in one process), reassembles exactly the
    full parity (no GPU: the pointer arithmetic of peer.striped_slots)."""
    import random
    import sys
    sys.path.insert(0, ROOT)
    from paper_2605_00831_b200.peer import ShardLayout, striped_slots
    rng = random.Random(808)
    port_lib = O.port()
    for trial in range(fuzz_trials(25)):
        n = rng.choice([2, 4, 6, 8, 12, 16])
        world = rng.choice([w for w in (1, 2, 3, 4, 6, 8) if n % w == 0])
        k = rng.randint(1, min(4, n))
        S = rng.randint(1, 4)
        L = rng.choice([1, 17, 4095, 4096, 4097, 3 * 4096 + 80, 65536 + 3])
        lay = ShardLayout(n, world, S, L)
        shards = [[splitmix_bytes(50_000 + 1000 * trial + 31 * s + j, L) for j in range(n)] for s in range(S)]
        mem = [np.stack([np.stack(shards[s][r * lay.n_local:(r + 1) * lay.n_local]) for s in range(S)])
               for r in range(world)]
        bases = [m.ctypes.data for m in mem]
        got = [[np.zeros(L, np.uint8) for _ in range(k)] for _ in range(S)]
        covered = 0
        for rank in range(world):
            off, ln, slots = striped_slots(lay, bases, rank)
            covered += ln
            if not ln:
                continue
            for s in range(S):
                data = [np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint8)), (ln,)).copy() for p in slots[s]]
                part = port_lib.encode(O.RS, n, k, data)
                for i in range(k):
                    got[s][i][off:off + ln] = part[i]
        assert covered == L, (trial, n, world, L)
        for s in range(S):
            want = port_lib.encode(O.RS, n, k, shards[s])
            for i in range(k):
                assert np.array_equal(got[s][i], want[i]), (trial, n, world, k, S, L, s, i)


def test_striped_planners_refuse_position_dependent_rdp():
    """RDP parity depends on byte position (coding.hpp:225-307): a rank
    encoding its byte range as a shard of its own would produce a different
    code, so the striped planners refuse RDP at world > 1 (the oracle shows
    the difference) and accept it at world 1 (one range = the whole shard)."""
    import sys
    sys.path.insert(0, ROOT)
    from paper_2605_00831_b200.coding import CodingScheme, ErasurePattern, InvalidArgument
    from paper_2605_00831_b200.peer import ShardLayout, plan_encode_striped, plan_reconstruct_striped
    from paper_2605_00831_b200.peer import require_position_independent
    port_lib = O.port()
    L = 10000
    shards = [splitmix_bytes(900 + j, L) for j in range(8)]
    whole = port_lib.encode(O.RDP, 8, 2, shards)
    half = port_lib.encode(O.RDP, 8, 2, [s[:4096] for s in shards])
    assert not np.array_equal(whole[1][:4096], half[1])   # range-local RDP is a different code
    rdp = CodingScheme.rdp(8)
    require_position_independent(rdp, ShardLayout(8, 1, 1, L))
    require_position_independent(CodingScheme.reed_solomon(8, 2), ShardLayout(8, 2, 1, L))
    with pytest.raises(InvalidArgument):
        plan_encode_striped(rdp, ShardLayout(8, 2, 1, L), [0, 0], 0, parity_out=None)
    with pytest.raises(InvalidArgument):
        plan_reconstruct_striped(rdp, ShardLayout(8, 2, 1, L), [0, 0], 0, ErasurePattern([1]), None, None)
