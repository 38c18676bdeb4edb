"""Checkpoint / recovery orchestration (checkpoint.hpp, recovery.hpp,
cost_model.hpp): planner + assignment logic on CPU; the byte path on GPU,
checked against the CPU oracle (checkpoint_test.cpp:151-292,
recovery_test.cpp:135-317)."""
import itertools
import random

import numpy as np
import pytest
from fuzzutil import fuzz_trials

from oracle import oracle as O
from paper_2605_00831_b200.checkpoint import (AssignmentState, CheckpointConfig, CostModel, FailureEvent,
                                              RecoveryMode, get_recompute_units, next_parity_worker)
from paper_2605_00831_b200.coding import CodingScheme, InvalidArgument
from paper_2605_00831_b200.kv_layout import ModelConfig


def sweep(n, m, scheme, slice_, cost):
    best, best_f = 0, float("inf")
    for r in range(n + 1):
        f = max(r * m * cost.compute_per_token + cost.restart_overhead, (n - r) * cost.reconstruct_chunk_time(scheme, slice_))
        if f < best_f:
            best, best_f = r, f
    return best


def test_recompute_units_match_sweep_oracle():
    # recovery_test.cpp:67-89 / acceptance.cpp C6(a)
    rng = random.Random(99)
    for _ in range(1000):
        cost = CostModel(compute_per_token=rng.uniform(1e-7, 1e-3), intra_bw=rng.uniform(50e9, 900e9))
        cost.host_bw = rng.uniform(0.5e9, cost.intra_bw)
        cost.encode_rate = rng.uniform(10e9, 500e9)
        cost.reconstruct_rate = rng.uniform(10e9, 500e9)
        cost.fixed_collective_latency = rng.uniform(0, 1e-4)
        cost.restart_overhead = rng.uniform(0, 5.0)
        n, m = rng.randrange(200), 1 + rng.randrange(4096)
        slice_ = 1 + rng.randrange(200 << 20)
        scheme = CodingScheme.reed_solomon(8, 1 + rng.randrange(4))
        assert get_recompute_units(n, m, scheme, slice_, cost) == sweep(n, m, scheme, slice_, cost)
    assert get_recompute_units(0, 2048, CodingScheme.reed_solomon(8, 2), 1 << 20, CostModel()) == 0
    free = CostModel(fixed_collective_latency=0)
    assert get_recompute_units(32, 2048, CodingScheme.reed_solomon(8, 2), 0, free) == 0


@pytest.mark.skipif(not O.have_ref(), reason="reference not compiled here (oracle/_ref)")
def test_recompute_units_match_the_reference_planner():
    """Same decisions as the reference's own get_recompute_units (recovery.hpp:
    58-88, compiled in place) on random cost models, incl. exact ties."""
    import ctypes as C
    fn = O.ref().fn("get_recompute_units")
    fn.argtypes = [C.c_uint32, C.c_uint32, C.c_int, C.c_int, C.c_int, C.c_uint64] + [C.c_double] * 7 + \
        [C.POINTER(C.c_uint32)]
    rng = random.Random(7)
    out = C.c_uint32()
    for i in range(2000):
        cost = CostModel(compute_per_token=rng.uniform(1e-7, 1e-3), intra_bw=rng.uniform(50e9, 900e9))
        cost.host_bw = rng.uniform(0.5e9, cost.intra_bw)
        cost.encode_rate = rng.uniform(10e9, 500e9)
        cost.reconstruct_rate = rng.uniform(10e9, 500e9)
        cost.fixed_collective_latency = rng.uniform(0, 1e-4) if i % 5 else 0.0
        cost.restart_overhead = rng.uniform(0, 5.0) if i % 7 else 0.0
        n, m = rng.randrange(300), 1 + rng.randrange(4096)
        slice_ = rng.randrange(200 << 20) if i % 11 else 0
        k = 1 + rng.randrange(4)
        scheme = CodingScheme.reed_solomon(8, k)
        assert fn(n, m, 2, 8, k, slice_, cost.compute_per_token, cost.intra_bw, cost.host_bw, cost.encode_rate,
                  cost.reconstruct_rate, cost.fixed_collective_latency, cost.restart_overhead, C.byref(out)) == 0
        assert get_recompute_units(n, m, scheme, slice_, cost) == out.value, (i, n, m, k, slice_)


def test_round_robin_fairness_and_config_validation():
    rng = random.Random(777)  # acceptance.cpp C7
    for _ in range(300):
        n, c = 1 + rng.randrange(32), 1 + rng.randrange(5000)
        st = AssignmentState()
        counts = [0] * n
        for _ in range(c):
            counts[next_parity_worker(st, n)] += 1
        assert max(counts) - min(counts) <= 1
    with pytest.raises(InvalidArgument):
        next_parity_worker(AssignmentState(), 0)
    with pytest.raises(InvalidArgument):
        CheckpointConfig(CodingScheme.reed_solomon(4, 2), 16, ModelConfig(2, 8, 8, 2, 8)).validate()
    with pytest.raises(InvalidArgument):
        CostModel(host_bw=500e9, intra_bw=400e9).validate()
    m = CostModel.measured(55.2, 5030.0, 5600.0)
    m.validate()
    assert m.host_bw == 55.2e9 and m.intra_bw == 770e9


# ---------------------------------------------------------------- GPU ------
def _ck(n, k, tp, chunk=16, capacity=None, layers=2, heads=8, dim=8, restart=1e-4):
    torch = pytest.importorskip("torch")
    from paper_2605_00831_b200.checkpoint import Checkpointer
    from paper_2605_00831_b200.parity_store import ParityStore
    cfg = CheckpointConfig(CodingScheme.reed_solomon(n, k), chunk, ModelConfig(layers, heads, dim, 2, tp))
    cfg.cost.restart_overhead = restart
    store = ParityStore() if capacity is None else ParityStore(capacity)
    return Checkpointer(cfg, store), store, torch


@pytest.mark.gpu
@pytest.mark.parametrize("seal", ["host", "device"])
def test_prefill_stored_parity_equals_encode_of_ground_truth(seal):
    """Stored parity == encode of the ground truth and the seal == the
    reference checksum (checkpoint_test.cpp:207-219), with the seal computed
    by the store's host threads or by the GPU (gs_parity_offload_sealed)."""
    ck, store, torch = _ck(4, 2, 4)
    ck.seal = seal
    ck.seal_inflight_bytes = 1   # device seal: every batch waits for the previous D2H (bound exercised)
    run = ck.run_prefill_with_checkpointing(11, 3 * 16 + 5, kv_seed=13)
    ck.synchronize()
    assert run.completed and run.chunks_done == 4
    port = O.port()
    for c in range(run.chunks_done):
        st, entry = store.get(11, c)
        assert int(st) == 0
        valid = 16 if c < 3 else 5
        assert entry.valid_tokens == valid
        host = [port.make_ground_truth_slice(13, 11, c, w, 2, 8, 8, 4, 16, valid) for w in range(4)]
        want = port.encode(O.RS, 4, 2, host)
        for i in range(2):
            assert np.array_equal(entry.parity[i], want[i]), (c, i)
        assert entry.checksum == port.parity_checksum(want)
    assert [s.worker for s in run.ground_truth[0]] == [0, 1, 2, 3]
    store.corrupt_entry(11, 1)   # a GPU-computed seal still catches host-tier corruption
    assert int(store.get(11, 1)[0]) != 0 and int(store.get(11, 2)[0]) == 0


@pytest.mark.gpu
def test_large_chunks_seal_on_device_and_recover():
    """auto seal policy: >= 16 MiB of parity per chunk is sealed on the GPU;
    the host re-verification (get) and a recovery from those entries agree."""
    ck, store, torch = _ck(8, 2, 8, chunk=2048, layers=32, heads=8, dim=128)   # 32 MiB slices
    assert ck._device_seal()
    run = ck.run_prefill_with_checkpointing(21, 4 * 2048, kv_seed=8)
    ck.synchronize()
    assert run.completed and run.chunks_done == 4
    for c in range(4):
        st, e = store.get(21, c, verify=True)
        assert int(st) == 0 and e.checksum == O.port().parity_checksum(e.parity)
    ck.cfg.cost.restart_overhead = 1e9
    res = ck.recover(21, FailureEvent([2], at_chunk=4), run.ground_truth, [2048] * 4)
    assert res.verified and len(res.plan.reconstruct_ids) == 4


@pytest.mark.gpu
def test_prefill_back_pressure_stops_at_the_offending_chunk():
    slice_ = 2 * 2 * 16 * (8 * 8 // 4) * 2
    ck, store, _ = _ck(4, 2, 4, capacity=2 * (2 * slice_ + 64) + 10)
    run = ck.run_prefill_with_checkpointing(1, 5 * 16, kv_seed=3)
    ck.synchronize()
    assert not run.completed and run.stalled_at_chunk == 2 and run.chunks_done == 2
    assert store.entry_count() == 2 and store.audit()


@pytest.mark.gpu
def test_decode_checkpointer_emits_every_m_tokens_and_flushes_tail():
    from paper_2605_00831_b200.checkpoint import DecodeCheckpointer
    ck, store, _ = _ck(8, 2, 8)
    dc = DecodeCheckpointer(5, 100, ck, kv_seed=21)
    st = AssignmentState()
    emitted = [o for o in (dc.step(st) for _ in range(40)) if o is not None]
    assert [o.chunk_id for o in emitted] == [100, 101] and dc.buffered_tokens() == 8
    tail = dc.flush(st)
    assert tail.chunk_id == 102 and tail.valid_tokens == 8 and dc.flush(st) is None
    ck.synchronize()
    port = O.port()
    for c, valid in ((100, 16), (101, 16), (102, 8)):
        entry = store.get(5, c)[1]
        host = [port.make_ground_truth_slice(21, 5, c, w, 2, 8, 8, 8, 16, valid) for w in range(8)]
        want = port.encode(O.RS, 8, 2, host)
        assert all(np.array_equal(entry.parity[i], want[i]) for i in range(2))


@pytest.mark.gpu
def test_every_double_failure_rs42_bit_exact():
    ck, store, _ = _ck(4, 2, 4)   # recovery_test.cpp:180-203
    run = ck.run_prefill_with_checkpointing(9, 4 * 16, kv_seed=17)
    ck.synchronize()
    for pair in itertools.combinations(range(4), 2):
        res = ck.recover(9, FailureEvent(list(pair), at_chunk=run.chunks_done), run.ground_truth,
                         [16] * run.chunks_done)
        assert res.verified
        for w in pair:
            for c in range(run.chunks_done):
                assert res.recovered[w][c] is not None


@pytest.mark.gpu
def test_long_request_single_failure_rs82_bit_exact():
    # recovery_test.cpp:299-317: 64K tokens, 32 chunks of 2048 through RS(8,2), worker 5 lost
    ck, store, _ = _ck(8, 2, 8, chunk=2048)
    run = ck.run_prefill_with_checkpointing(6, 65536, kv_seed=36)
    assert run.completed and run.chunks_done == 32
    ck.synchronize()
    ck.cfg.cost.restart_overhead = 1e9   # force pure reconstruction of all 32 chunks
    res = ck.recover(6, FailureEvent([5], at_chunk=32), run.ground_truth, [2048] * 32)
    assert res.plan.mode == RecoveryMode.kHybrid and res.plan.recompute_chunks == 0
    assert res.verified and len(res.plan.reconstruct_ids) == 32
    # dynamic verification split (default): every chunk's row 0 hashed on the
    # GPU, the rest of each chain claimed at run time by host threads or the
    # GPU feeder
    assert 0 <= res.verify_gpu_chunks <= 32 and ck.verify_split == "dynamic"
    for threads in (1, 2):   # few host threads: the GPU feeder takes most of the chains
        res = ck.recover(6, FailureEvent([5], at_chunk=32), run.ground_truth, [2048] * 32, verify_threads=threads)
        assert res.verified and res.decoded_chunks == 32 and res.verify_gpu_chunks > 0, threads
    # the same with the scalar host chain (hosts without the AVX-512 FNV): same plan, same bytes
    from paper_2605_00831_b200 import _lib as L
    hw = L.lib().gs_fnv_host_simd()
    try:
        L.lib().gs_fnv_host_set_simd(0)
        res = ck.recover(6, FailureEvent([5], at_chunk=32), run.ground_truth, [2048] * 32)
        assert res.verified and res.decoded_chunks == 32 and not res.corrupt_chunks
    finally:
        assert L.lib().gs_fnv_host_set_simd(1) == hw
    # static split (decided from the host-rate estimates): all in HBM / all split / host only
    ck.verify_split = "static"
    for gpu, rate, want in [(True, 1.0, 32), (True, 1e30, 0), (False, None, 0)]:
        ck.gpu_verify = gpu
        if rate:
            ck.host_fnv_rate = ck.host_chain_rate = rate
        res = ck.recover(6, FailureEvent([5], at_chunk=32), run.ground_truth, [2048] * 32)
        assert res.verified and res.verify_gpu_chunks == want and len(res.plan.reconstruct_ids) == 32


@pytest.mark.gpu
def test_bad_parity_and_over_tolerance_fallbacks():
    ck, store, _ = _ck(4, 2, 4)
    run = ck.run_prefill_with_checkpointing(3, 4 * 16, kv_seed=5)
    ck.synchronize()
    store.corrupt_entry(3, 2)
    rep = ck.reconstruct_chunk(2, run.ground_truth[2], 3, {1})
    assert rep.status == 1 and not rep.recovered
    res = ck.recover(3, FailureEvent([0, 1, 2], at_chunk=4), run.ground_truth, [16] * 4)
    assert res.plan.mode == RecoveryMode.kFullRecomputeFallback and res.plan.recompute_chunks == 4
    ck.cfg.cost.restart_overhead = 1e9
    res = ck.recover(3, FailureEvent([1], at_chunk=4), run.ground_truth, [16] * 4)
    assert res.plan.mode == RecoveryMode.kFullRecomputeFallback   # corrupt chunk 2 -> fallback
    # the corrupt entry caught by the dynamic split, by the GPU checksum (every
    # entry verified in HBM), by host threads continuing GPU states, and by the
    # host threads alone
    res = ck.recover(3, FailureEvent([1], at_chunk=4), run.ground_truth, [16] * 4)
    assert res.plan.mode == RecoveryMode.kFullRecomputeFallback and res.corrupt_chunks == [2]
    ck.verify_split = "static"
    for gpu, rate in [(True, 1.0), (True, 1e30), (False, None)]:
        ck.gpu_verify = gpu
        if rate:   # 1.0: host FNV "slow" -> every entry on the GPU; 1e30: host "fast" -> all split
            ck.host_fnv_rate = ck.host_chain_rate = rate
        res = ck.recover(3, FailureEvent([1], at_chunk=4), run.ground_truth, [16] * 4)
        assert res.plan.mode == RecoveryMode.kFullRecomputeFallback, (gpu, rate)
        assert res.verify_gpu_chunks == (4 if rate == 1.0 else 0)
        assert res.corrupt_chunks == [2] and res.decoded_chunks == 0


@pytest.mark.gpu
def test_serving_loop_example_runs_bit_exact():
    """examples/serving_loop.py end to end: prefill + decode checkpoints
    (incl. a masked tail), worker failure, planned recovery, bit-exact."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "examples", "serving_loop.py"), "--tokens", "256",
                          "--decode", "40", "--chunk", "16", "--lost", "3"], capture_output=True, text=True,
                         timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "bit-exact: True" in out.stdout and "masked tail of 8 tokens" in out.stdout, out.stdout


@pytest.mark.gpu
def test_orchestration_fuzz():
    """Random schemes (RS(tp, k)), geometries, chunk sizes, prompt and decode
    lengths and 1..k failed workers: prefill + decode checkpointing, then
    recover() -- every recovered slice bit-exact (recovery.hpp:135-145)."""
    import random
    from paper_2605_00831_b200.checkpoint import DecodeCheckpointer
    rng = random.Random(5150)
    for trial in range(fuzz_trials(10)):
        tp = rng.choice([2, 4, 6, 8])
        k = rng.randint(1, min(3, tp))
        chunk = rng.choice([4, 16, 32])
        ck, store, torch = _ck(tp, k, tp, chunk=chunk, layers=rng.choice([1, 2, 3]), heads=tp,
                               dim=rng.choice([8, 16]), restart=1e9)
        req = 100 + trial
        tokens = rng.randint(1, 5 * chunk)
        run = ck.run_prefill_with_checkpointing(req, tokens, kv_seed=trial)
        ground, counts = list(run.ground_truth), [min(chunk, tokens - c * chunk) for c in range(run.chunks_done)]
        if tokens % chunk == 0:
            dec = DecodeCheckpointer(req, run.chunks_done, ck, kv_seed=trial)
            steps = rng.randint(0, 3 * chunk)
            for _ in range(steps):
                dec.step(run.state)
            dec.flush(run.state)
            ground += dec.ground_truth
            counts += [s[0].valid_tokens for s in dec.ground_truth]
        ck.synchronize()
        failed = sorted(rng.sample(range(tp), rng.randint(1, k)))
        res = ck.recover(req, FailureEvent(failed, at_chunk=len(ground)), ground, counts)
        assert res.verified, (trial, tp, k, chunk, tokens, failed, res.plan.mode)
        assert res.plan.recompute_chunks == 0 and len(res.plan.reconstruct_ids) == len(ground)
        ck.close()


@pytest.mark.gpu
def test_odd_slice_sizes_fall_back_to_host_fnv():
    """Slices that are not 16-B multiples (24 B here) cannot use the GPU FNV:
    seal="device" and gpu_verify fall back to the host chain, bit-exact."""
    ck, store, torch = _ck(4, 2, 4, chunk=3, layers=1, heads=4, dim=2, restart=1e9)
    assert ck.slice == 24 and not ck._device_seal(64)
    ck.seal = "device"
    run = ck.run_prefill_with_checkpointing(5, 4 * 3, kv_seed=2)
    ck.synchronize()
    for c in range(run.chunks_done):
        st, e = store.get(5, c, verify=True)
        assert int(st) == 0 and e.checksum == O.port().parity_checksum(e.parity)
    res = ck.recover(5, FailureEvent([1], at_chunk=run.chunks_done), run.ground_truth, [3] * run.chunks_done)
    assert res.verified and res.verify_gpu_chunks == 0 and len(res.plan.reconstruct_ids) == run.chunks_done


@pytest.mark.gpu
def test_c3_full_geometry_sealed_on_device_and_recovered_hybrid():
    """The true C3 geometry (Llama-3-70B KV TP=8, 128K-token prefill = 64
    chunks x 8 workers x 83,886,080 B, RS(8,2)) with the default policies:
    seal="auto" (every chunk sealed on the GPU), seal_inflight_bytes 2 GiB
    (10 GiB of parity -> in-flight buffers are popped while their checksums
    are still being committed), gpu_verify=True. Every stored checksum equals
    the reference's compute_checksum of the stored bytes, chunks 0 and 63
    equal the oracle's encode, and the recovery of worker 5 at chunk 64 is
    hybrid with all 64 chunks decoded bit-exact (recovery.hpp:176-298,
    parity_store.hpp:46-53)."""
    import concurrent.futures as cf
    import torch
    from paper_2605_00831_b200.checkpoint import Checkpointer
    from paper_2605_00831_b200.kv_layout import LLAMA3_70B
    from paper_2605_00831_b200.parity_store import ParityStore
    cfg = CheckpointConfig(CodingScheme.reed_solomon(8, 2), 2048, LLAMA3_70B)
    store = ParityStore(seal_threads=8)
    ck = Checkpointer(cfg, store)
    assert ck.slice == 83886080 and ck.seal == "auto" and ck._device_seal() and ck.gpu_verify
    assert ck.seal_inflight_bytes < 64 * 2 * ck.slice
    run = ck.run_prefill_with_checkpointing(7, 131072, kv_seed=3)
    ck.synchronize()
    assert run.completed and run.chunks_done == 64
    port = O.port()
    entries = [store.get(7, c, verify=False)[1] for c in range(64)]
    with cf.ThreadPoolExecutor(16) as ex:   # the oracle's serial FNV releases the GIL
        sums = list(ex.map(lambda e: port.parity_checksum(e.parity), entries))
    bad = [c for c in range(64) if sums[c] != entries[c].checksum]
    assert not bad, f"stored checksums disagree with the reference FNV for chunks {bad}"
    for c in (0, 63):
        host = [run.ground_truth[c][w].bytes.cpu().numpy() for w in range(8)]
        want = port.encode(O.RS, 8, 2, host)
        assert all(np.array_equal(entries[c].parity[i], want[i]) for i in range(2)), c
    del entries
    res = ck.recover(7, FailureEvent([5], at_chunk=64), run.ground_truth, [2048] * 64)
    assert res.plan.mode == RecoveryMode.kHybrid, (res.plan.mode, res.corrupt_chunks)
    assert len(res.plan.reconstruct_ids) == 64 and res.decoded_chunks == 64 and res.verified
    assert res.reconstruct_device_ms > 0
    for c in range(64):
        assert torch.equal(res.recovered[5][c].bytes, run.ground_truth[c][5].bytes), c
    ck.close()
    store.close()
