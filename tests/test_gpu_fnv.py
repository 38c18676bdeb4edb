"""GPU FNV-1a (gs_fnv1a64_device, gs_fnv_gpu.cu) against the oracle's serial
FNV-1a (parity_store.hpp:19-25) and ParityChunk::compute_checksum
(parity_store.hpp:46-50): bit-exact on random chains, chain lengths around
the 16 KiB block and 64-byte thread boundaries, several buffers per chain,
arbitrary seeds h0, the golden "foobar"-style KAT extended to 16-B multiples,
and a full-size C3 chunk (2 x 80 MiB) against the reference checksum."""
import ctypes as C

import numpy as np
import pytest
from fuzzutil import fuzz_trials

from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2605_00831_b200 import _lib as L  # noqa: E402

OFFSET = 0xCBF29CE484222325


@pytest.fixture(scope="module", autouse=True)
def cuda0():
    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device")
    torch.cuda.set_device(0)
    yield


def device_fnv(bufs, n_chains, k, ln, h0=OFFSET):
    out = torch.full((max(n_chains, 1),), 7, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    rc = L.lib().gs_fnv1a64_device(L.ptr_array([b.data_ptr() for b in bufs]), n_chains, k, ln, h0,
                                   out.data_ptr(), st.cuda_stream)
    assert rc == 0, L.lib().gs_last_error()
    st.synchronize()
    return [int(v) & (2**64 - 1) for v in out.cpu().tolist()[:n_chains]]


@pytest.mark.parametrize("ln", [16, 48, 64, 1008, 16368, 16384, 16400, 32768 + 48, 3 * 16384 + 4096 + 16,
                                262144, 1 << 20])
@pytest.mark.parametrize("k", [1, 2, 3])
def test_chains_match_serial_fnv(ln, k):
    rng = np.random.default_rng(ln * 7 + k)
    n_chains = 3
    host = [rng.integers(0, 256, ln, dtype=np.uint8) for _ in range(n_chains * k)]
    dev = [torch.from_numpy(h).cuda() for h in host]
    got = device_fnv(dev, n_chains, k, ln)
    port = O.port()
    for c in range(n_chains):
        assert got[c] == port.parity_checksum(host[c * k:(c + 1) * k]), (ln, k, c)


def test_seeds_and_special_bytes():
    port = O.port()
    rng = np.random.default_rng(3)
    for h0 in [0, 1, 0xFF, 0x100, OFFSET, 2**64 - 1, int(rng.integers(0, 2**63)) * 2 + 1]:
        for fill in [None, 0, 0xFF, 0x80]:
            ln = 16384 * 2 + 32
            h = rng.integers(0, 256, ln, dtype=np.uint8) if fill is None else np.full(ln, fill, np.uint8)
            got = device_fnv([torch.from_numpy(h).cuda()], 1, 1, ln, h0)
            assert got[0] == port.fnv1a64(h, h0), (h0, fill)


def test_many_chains_and_jobs():
    """More chains than one job's pointer table (480 / k) and zero-length
    chains (hash = h0)."""
    port = O.port()
    rng = np.random.default_rng(11)
    k, ln, n_chains = 2, 4096, 300
    host = [rng.integers(0, 256, ln, dtype=np.uint8) for _ in range(n_chains * k)]
    flat = torch.from_numpy(np.concatenate(host)).cuda()
    dev = [flat[i * ln:(i + 1) * ln] for i in range(n_chains * k)]
    got = device_fnv(dev, n_chains, k, ln)
    for c in range(0, n_chains, 37):
        assert got[c] == port.parity_checksum(host[c * k:(c + 1) * k]), c
    assert got[-1] == port.parity_checksum(host[-k:])
    z = torch.zeros(16, dtype=torch.uint8, device="cuda")
    assert device_fnv([z, z], 2, 1, 0, 12345) == [12345, 12345]


def test_rejects_bad_arguments():
    lib = L.lib()
    x = torch.zeros(64, dtype=torch.uint8, device="cuda")
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    assert lib.gs_fnv1a64_device(L.ptr_array([x.data_ptr()]), 1, 1, 17, OFFSET, out.data_ptr(), None) == \
        L.GS_INVALID_ARGUMENT
    assert lib.gs_fnv1a64_device(L.ptr_array([x.data_ptr() + 1]), 1, 1, 16, OFFSET, out.data_ptr(), None) == \
        L.GS_INVALID_ARGUMENT
    assert lib.gs_fnv1a64_device(L.ptr_array([None]), 1, 1, 16, OFFSET, out.data_ptr(), None) == \
        L.GS_INVALID_ARGUMENT


def test_full_size_c3_chunk_checksum():
    """One C3 chunk's parity (RS(8,2), 2 x 83,886,080 B) sealed on the GPU
    equals the host seal (the reference's compute_checksum)."""
    ln = 83886080
    g = torch.Generator(device="cuda").manual_seed(5)
    par = torch.randint(0, 256, (2, ln), dtype=torch.uint8, device="cuda", generator=g)
    got = device_fnv([par[0], par[1]], 1, 2, ln)
    hp = par.cpu().numpy()
    want = L.lib().gs_parity_checksum(L.ptr_array([hp[0].ctypes.data, hp[1].ctypes.data]), 2, ln)
    assert got[0] == want


@pytest.mark.parametrize("n_full,u", [(0, 1), (2, 1), (5, 1), (1, 2), (0, 3)])
def test_split_verification_matches_reference_checksum(n_full, u):
    """gs_verify_enqueue / gs_verify_finish: entries verified entirely on the
    GPU, or GPU-hashed over rows < u and finished by host threads over the
    rest -- every checksum equals ParityChunk::compute_checksum; the uploaded
    rows equal the host rows."""
    port = O.port()
    rng = np.random.default_rng(100 + 10 * n_full + u)
    n, k, ln = 5, 3, 16384 * 3 + 48
    host = [torch.from_numpy(rng.integers(0, 256, ln, dtype=np.uint8)).pin_memory() for _ in range(n * k)]
    dev = torch.zeros((n, k, ln), dtype=torch.uint8, device="cuda")
    drows = [dev[c, i].data_ptr() if (c < n_full or i < u) else None for c in range(n) for i in range(k)]
    lib = L.lib()
    comp, copy = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()   # dev zeroed before the side streams write it
    h = C.c_void_p()
    assert lib.gs_verify_enqueue(L.ptr_array([t.data_ptr() for t in host]), n, k, ln, n_full, u,
                                 L.ptr_array(drows), comp.cuda_stream, copy.cuda_stream, C.byref(h)) == 0
    out = (C.c_uint64 * n)()
    assert lib.gs_verify_finish(h, 3, out) == 0, lib.gs_last_error()
    torch.cuda.synchronize()
    for c in range(n):
        rows = [host[c * k + i].numpy() for i in range(k)]
        assert out[c] == port.parity_checksum(rows), (c, n_full, u)
        for i in range(k):
            if c < n_full or i < u:
                assert torch.equal(dev[c, i].cpu(), host[c * k + i])


def test_upload_checksum_entry_point():
    """gs_parity_upload_checksum: rows land in HBM and every chunk's checksum
    equals the reference's."""
    port = O.port()
    rng = np.random.default_rng(77)
    n, k, ln = 6, 2, 16384 + 32
    host = [torch.from_numpy(rng.integers(0, 256, ln, dtype=np.uint8)).pin_memory() for _ in range(n * k)]
    dev = torch.zeros((n, k, ln), dtype=torch.uint8, device="cuda")
    sums = torch.zeros(n, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    assert L.lib().gs_parity_upload_checksum(L.ptr_array([t.data_ptr() for t in host]), n, k, ln,
                                             L.ptr_array([dev[c, i].data_ptr() for c in range(n) for i in range(k)]),
                                             sums.data_ptr(), st.cuda_stream, st.cuda_stream) == 0
    st.synchronize()
    got = [int(v) & (2**64 - 1) for v in sums.cpu().tolist()]
    for c in range(n):
        assert got[c] == port.parity_checksum([host[c * k + i].numpy() for i in range(k)])


def test_fnv_fuzz_random_chains():
    """Random chain counts, buffer counts, lengths (16-B multiples around the
    64-B thread and 16 KiB block grains) and seeds: bit-exact every time."""
    port = O.port()
    rng = np.random.default_rng(2026)
    for trial in range(fuzz_trials(30)):
        n_chains = int(rng.integers(1, 9))
        k = int(rng.integers(1, 5))
        ln = 16 * int(rng.choice([1, 3, 4, 63, 64, 65, 1023, 1024, 1025, int(rng.integers(1, 12000))]))
        h0 = int(rng.integers(0, 2**63)) * 2 + int(rng.integers(0, 2))
        host = [rng.integers(0, 256, ln, dtype=np.uint8) for _ in range(n_chains * k)]
        flat = torch.from_numpy(np.concatenate(host)).cuda()
        dev = [flat[i * ln:(i + 1) * ln] for i in range(n_chains * k)]
        got = device_fnv(dev, n_chains, k, ln, h0)
        for c in range(n_chains):
            h = h0
            for i in range(k):
                h = port.fnv1a64(host[c * k + i], h)
            assert got[c] == h, (trial, n_chains, k, ln, c)


def test_multi_job_chains_beyond_the_scratch_budget():
    """14 chains of 2 x 80 MiB: the low-byte scratch (2.2 GiB) exceeds the
    per-job budget (2 GiB), so the chains are hashed in two jobs -- every
    checksum still equals the host seal (the reference's compute_checksum)."""
    ln, n = 83886080, 14
    g = torch.Generator(device="cuda").manual_seed(9)
    par = torch.randint(0, 256, (n, 2, ln), dtype=torch.uint8, device="cuda", generator=g)
    got = device_fnv([par[c, i] for c in range(n) for i in range(2)], n, 2, ln)
    hp = par.cpu().numpy()
    out = (C.c_uint64 * n)()
    assert L.lib().gs_parity_checksum_batch(L.ptr_array([hp[c, i].ctypes.data for c in range(n) for i in range(2)]),
                                            n, 2, ln, 16, out) == 0
    assert got == [int(out[c]) for c in range(n)]


@pytest.mark.parametrize("where", ["device", "pinned"])
def test_sealed_commit_owns_its_checksums(where):
    """gs_store_commit_sealed_batch copies the checksums on the commit's stream
    into memory the store owns: overwriting the caller's buffer once the
    stream has passed the commit (device: a later kernel on the same stream;
    pinned: a host write after the stream drained) never changes what the
    entries are sealed with."""
    from paper_2605_00831_b200.coding import CodingScheme
    from paper_2605_00831_b200.parity_store import ParityStore
    store = ParityStore(seal_threads=2)
    sch = CodingScheme.reed_solomon(4, 2)
    st = torch.cuda.Stream()
    for rnd in range(50):
        keys = [(rnd, c) for c in range(3)]
        acc, _ = store.reserve_batch(keys, sch, 16, 4096)
        assert acc == 3
        vals = [rnd * 1000 + c + 1 for c in range(3)]
        if where == "device":
            buf = torch.tensor(vals, dtype=torch.int64, device="cuda")
            torch.cuda.synchronize()
            store.commit_sealed_batch(keys, buf.data_ptr(), st)
            with torch.cuda.stream(st):
                buf.fill_(-1)            # stream-ordered after the store's copy
        else:
            buf = torch.tensor(vals, dtype=torch.int64).pin_memory()
            store.commit_sealed_batch(keys, buf.data_ptr(), st)
            st.synchronize()
            buf.fill_(-1)                # the landing thread may not have run yet
        del buf
    store.wait_sealed()
    for rnd in range(50):
        for c in range(3):
            status, e = store.get(rnd, c, verify=False)
            assert int(status) == 0 and e.checksum == rnd * 1000 + c + 1, (rnd, c)
    store.close()


@pytest.mark.parametrize("u,threads,rates,ln", [(1, 1, None, 16384 * 5 + 32), (1, 4, None, 16384 * 5 + 32),
                                                (2, 3, None, 16384 * 5 + 32), (3, 2, None, 16384 * 5 + 32),
                                                (2, 4, (1000.0, 1000.0), (6 << 20) + 48),
                                                (1, 3, (30.0, 0.5), (6 << 20) + 48)])
def test_dynamic_split_verification(u, threads, rates, ln):
    """gs_verify_enqueue(n_full = -1): rows < u of every chunk uploaded and
    hashed on the GPU, the rest of each chain claimed at run time by host
    threads (from the front) or the GPU feeder (from the back, seeded GPU
    FNV), incl. host threads handing a chain over to the GPU mid-row when
    they fall behind it (rates: a link so fast that every host claim hands
    off after its first 4 MiB slice): every checksum equals
    ParityChunk::compute_checksum, the uploaded rows equal the host rows."""
    port = O.port()
    rng = np.random.default_rng(500 + 10 * u + threads)
    n, k = (13, 3) if rates is None else (6, 3)
    host = [torch.from_numpy(rng.integers(0, 256, ln, dtype=np.uint8)).pin_memory() for _ in range(n * k)]
    dev = torch.zeros((n, u, ln), dtype=torch.uint8, device="cuda")
    drows = [dev[c, i].data_ptr() if i < u else None for c in range(n) for i in range(k)]
    lib = L.lib()
    comp, copy = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    h = C.c_void_p()
    assert lib.gs_verify_enqueue(L.ptr_array([t.data_ptr() for t in host]), n, k, ln, -1, u,
                                 L.ptr_array(drows), comp.cuda_stream, copy.cuda_stream, C.byref(h)) == 0
    if rates is not None:
        assert lib.gs_verify_set_rates(h, *rates) == 0
    out = (C.c_uint64 * n)()
    gpu = C.c_int(-1)
    handoffs0 = lib.gs_verify_handoffs()
    # the hand-off safety net needs a host slower than the link: the scalar chain
    simd = lib.gs_fnv_host_set_simd(0 if rates == (1000.0, 1000.0) else 1)
    try:
        assert lib.gs_verify_finish_ex(h, threads, out, C.byref(gpu)) == 0, lib.gs_last_error()
    finally:
        lib.gs_fnv_host_set_simd(1)
    assert simd == 0 or rates != (1000.0, 1000.0)
    torch.cuda.synchronize()
    assert 0 <= gpu.value <= n and (u < k or gpu.value == n)
    if rates == (1000.0, 1000.0):
        assert lib.gs_verify_handoffs() > handoffs0
    for c in range(n):
        assert out[c] == port.parity_checksum([host[c * k + i].numpy() for i in range(k)]), (c, u, threads)
        for i in range(u):
            assert torch.equal(dev[c, i].cpu(), host[c * k + i])


def test_seeded_device_fnv_continues_chains():
    """gs_fnv1a64_device_seeded: hashing the second half of each chain from
    the device-resident state after the first half equals hashing the whole
    chain (the continuation the dynamic verification's GPU feeder uses)."""
    port = O.port()
    rng = np.random.default_rng(71)
    n, ln = 5, 16384 * 3 + 48
    host = [rng.integers(0, 256, ln, dtype=np.uint8) for _ in range(n * 4)]
    dev = [torch.from_numpy(x).cuda() for x in host]
    first = torch.zeros(n, dtype=torch.int64, device="cuda")
    both = torch.zeros(n, dtype=torch.int64, device="cuda")
    lib = L.lib()
    st = torch.cuda.current_stream()
    assert lib.gs_fnv1a64_device(L.ptr_array([dev[c * 4 + i].data_ptr() for c in range(n) for i in range(2)]), n, 2,
                                 ln, OFFSET, first.data_ptr(), st.cuda_stream) == 0
    assert lib.gs_fnv1a64_device_seeded(L.ptr_array([dev[c * 4 + 2 + i].data_ptr() for c in range(n)
                                                     for i in range(2)]), n, 2, ln, first.data_ptr(),
                                        both.data_ptr(), st.cuda_stream) == 0
    assert lib.gs_fnv1a64_device_seeded(L.ptr_array([dev[0].data_ptr()]), 1, 1, ln, first.data_ptr(),
                                        first.data_ptr(), st.cuda_stream) == L.GS_INVALID_ARGUMENT
    st.synchronize()
    got = [int(v) & (2**64 - 1) for v in both.cpu().tolist()]
    for c in range(n):
        assert got[c] == port.parity_checksum(host[c * 4:(c + 1) * 4]), c


def test_offload_sealed_orders_rows_and_checksums_on_the_copy_stream():
    """gs_parity_offload_sealed: once the COPY stream is synchronised (nothing
    else), the rows and the checksums are in host memory -- the checksums travel
    on the compute stream after the GPU FNV, and the copy stream waits for them
    before anything queued after the call (a store commit reads them there)."""
    S, k, ln = 6, 2, 3 * 65536 + 4096
    comp, copy = torch.cuda.Stream(), torch.cuda.Stream()
    rows = torch.randint(0, 256, (S, k, ln), dtype=torch.uint8, device="cuda")
    h_rows = torch.zeros((S, k, ln), dtype=torch.uint8).pin_memory()
    h_sums = torch.zeros(S, dtype=torch.int64).pin_memory()
    torch.cuda.synchronize()
    with torch.cuda.stream(comp):
        torch.cuda._sleep(2_000_000)   # keep the compute stream busy: the FNV lands late
    rc = L.lib().gs_parity_offload_sealed(L.ptr_array([rows[s, i].data_ptr() for s in range(S) for i in range(k)]),
                                          S, k, ln,
                                          L.ptr_array([h_rows[s, i].data_ptr() for s in range(S) for i in range(k)]),
                                          h_sums.data_ptr(), comp.cuda_stream, copy.cuda_stream)
    assert rc == 0, L.lib().gs_last_error()
    copy.synchronize()
    host = rows.cpu()
    assert torch.equal(h_rows, host)
    want = [O.port().parity_checksum([host[s, i].numpy() for i in range(k)]) for s in range(S)]
    assert [int(v) & (2**64 - 1) for v in h_sums.tolist()] == want
    torch.cuda.synchronize()
