"""C-ABI host-side checks (no GPU): the library loads, exports every symbol
include/gs_capi.h declares, and its host planning (field, Cauchy matrix,
decode-matrix inversion, validation, errors) matches the pinned oracle."""
import ctypes as C
import itertools
import os
import re

import numpy as np
import pytest
from fuzzutil import fuzz_trials

from oracle import oracle as O
from paper_2605_00831_b200 import _lib as L
from paper_2605_00831_b200 import coding as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "gs_capi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gs_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = L.lib()
    syms = declared_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in gs_capi.h but not exported"
        assert s in L.SIGNATURES, f"{s} has no ctypes signature"
    assert set(L.SIGNATURES) == set(syms)


def test_gf_field_matches_oracle(port, golden):
    lib = L.lib()
    for a in range(256):
        for b in range(0, 256, 3):
            assert lib.gs_gf_mul(a, b) == port.gf_mul(a, b)
    inv = bytes([0] + [G.gf256.inv(a) for a in range(1, 256)])
    assert inv.hex() == golden["gf"]["inv_hex"]
    with pytest.raises(G.DomainError):
        G.gf256.inv(0)
    with pytest.raises(G.DomainError):
        G.gf256.div(3, 0)
    assert G.gf256.div(0, 7) == 0
    assert G.gf256.mul(G.gf256.div(0x53, 0xCA), 0xCA) == 0x53


def test_encoding_matrices_match_reference(golden):
    for key, hx in golden["matrices"].items():
        kind, n, k = map(int, key.split("_"))
        m = G.build_encoding_matrix(G.CodingScheme(G.CodeKind(kind), n, k))
        assert m.coef.tobytes().hex() == hx, key
        assert (m.rows, m.cols) == (k, n)


def test_validation_statuses_match_reference(golden):
    for rec in golden["errors"]:
        if rec["op"] != "validate":
            continue
        assert L.lib().gs_scheme_validate(rec["kind"], rec["n"], rec["k"]) == rec["status"], rec
    with pytest.raises(G.InvalidArgument):
        G.CodingScheme.reed_solomon(4, 5).validate()
    with pytest.raises(G.InvalidArgument):
        G.build_encoding_matrix(G.CodingScheme.reed_solomon(300, 1))
    assert G.max_tolerance(G.CodingScheme.reed_solomon(8, 3)) == 3
    assert G.max_tolerance(G.CodingScheme.rdp(8)) == 2
    assert G.memory_overhead_ratio(G.CodingScheme.reed_solomon(8, 2)) == 0.25


@pytest.mark.parametrize("kind,n,k", [(O.XOR, 4, 1), (O.XOR, 8, 1), (O.RS, 4, 2), (O.RS, 6, 2),
                                      (O.RS, 8, 2), (O.RS, 8, 3), (O.RS, 10, 4), (O.RS, 4, 1)])
def test_decode_plans_match_oracle(port, kind, n, k):
    """Host decode planning == coding.hpp:535-566 (via the pinned oracle) for
    every erasure pattern within tolerance, for both kernel back ends."""
    scheme = G.CodingScheme(G.CodeKind(kind), n, k)
    tol = 1 if kind == O.XOR else k
    for e in range(1, tol + 1):
        for lost in itertools.combinations(range(n + k), e):
            cd, cp = port.decode_matrix(kind, n, k, list(lost))
            for generic in (False, True):
                c = G.codec_ex(scheme, G.ErasurePattern(lost), generic=generic)
                lost_data = [i for i in lost if i < n]
                assert c.out_index == lost_data
                got = c.coefficients()
                if not lost_data:
                    assert got.size == 0
                    continue
                want = np.concatenate([cd, cp], axis=1)
                assert np.array_equal(got, want), (lost, generic)
                if generic:
                    assert not c.specialised


def test_specialised_registry_covers_configs():
    for n, k in [(4, 2), (8, 2), (6, 2), (8, 3), (4, 1)]:
        assert G.encoder(G.CodingScheme.reed_solomon(n, k)).specialised
    assert G.encoder(G.CodingScheme.xor_code(8)).specialised
    for lost in ([0], [5], [3, 8], [0, 7], [8, 2]):
        assert G.decoder(G.CodingScheme.reed_solomon(8, 2), G.ErasurePattern(lost)).specialised, lost
    for pair in itertools.combinations(range(6), 2):
        assert G.decoder(G.CodingScheme.reed_solomon(6, 2), G.ErasurePattern(pair)).specialised
    # unusual shapes fall back to the generic GPU kernel, not to the CPU
    assert not G.encoder(G.CodingScheme.reed_solomon(9, 2)).specialised
    assert not G.decoder(G.CodingScheme.reed_solomon(8, 3), G.ErasurePattern([1])).specialised


def test_decoder_errors_match_reference(golden):
    for rec in golden["errors"]:
        if rec["op"] != "reconstruct" or rec["drop"] is not None:
            continue
        h = C.c_void_p()
        lost = rec["lost"]
        arr = (C.c_int * len(lost))(*lost)
        st = L.lib().gs_decoder_create(rec["kind"], rec["n"], rec["k"], arr, len(lost), C.byref(h))
        assert st == rec["status"], rec
        if st == 0:
            c = G.Codec(h.value)
            assert sorted(c.out_index) == rec["rebuilt"]


def test_rdp_codecs_and_limits():
    # RDP runs on the GPU path for p <= 23 (n <= 22); wider arrays are refused, not faked
    enc = G.encoder(G.CodingScheme.rdp(8))
    assert enc.n_out == 2 and enc.out_index == [8, 9] and not enc.specialised
    h = C.c_void_p()
    assert L.lib().gs_encoder_create(1, 30, 2, C.byref(h)) == L.GS_UNSUPPORTED
    for lost, outs in (([3], [3]), ([3, 8], [3]), ([3, 9], [3]), ([1, 5], [1, 5]), ([8, 9], [])):
        assert G.decoder(G.CodingScheme.rdp(6 if max(lost) < 8 else 8), G.ErasurePattern(lost)).out_index == outs
    with pytest.raises(G.UnrecoverableError):
        G.decoder(G.CodingScheme.rdp(4), G.ErasurePattern([0, 1, 2]))


def test_slice_bytes_and_seal(golden, port):
    from paper_2605_00831_b200 import kv_layout as K
    for rec in golden["slice_bytes"]:
        Lr, H, D, tp = rec["model"]
        assert K.slice_bytes(K.ModelConfig(Lr, H, D, 2, tp), rec["m"]) == rec["bytes"]
    with pytest.raises(G.InvalidArgument):
        K.slice_bytes(K.ModelConfig(2, 4, 8, 2, 3), 16)
    assert K.chunk_count(5000, 2048) == 3
    lib = L.lib()
    buf = np.frombuffer(b"foobar", np.uint8)
    assert f"{lib.gs_fnv1a64(buf.ctypes.data, 6, 0xCBF29CE484222325):016x}" == golden["fnv"]["foobar"]
    parity = [np.frombuffer(os.urandom(777), np.uint8) for _ in range(12)]
    out = (C.c_uint64 * 4)()
    assert lib.gs_parity_checksum_batch(L.ptr_array([p.ctypes.data for p in parity]), 4, 3, 777, 3,
                                        out) == 0
    for c in range(4):
        assert out[c] == port.parity_checksum(parity[3 * c: 3 * c + 3])
    # lockstep groups of 4..8 chains per thread (chunk counts that are not a
    # multiple of the group, one thread, more threads than chunks)
    rng = np.random.default_rng(5)
    for n_chunks, threads, ln in [(13, 2, 301), (9, 1, 64), (64, 14, 33), (7, 3, 1), (5, 16, 100)]:
        parity = [rng.integers(0, 256, ln, dtype=np.uint8) for _ in range(2 * n_chunks)]
        out = (C.c_uint64 * n_chunks)()
        assert lib.gs_parity_checksum_batch(L.ptr_array([p.ctypes.data for p in parity]), n_chunks, 2, ln,
                                            threads, out) == 0
        for c in range(n_chunks):
            assert out[c] == port.parity_checksum(parity[2 * c: 2 * c + 2]), (n_chunks, threads, c)


def test_stripe_ranges_partition_exactly():
    lib = L.lib()
    for total in [0, 1, 4095, 4096, 83886080, 262144 * 32 + 17]:
        for world in [1, 2, 3, 4, 8]:
            spans = []
            for r in range(world):
                off, ln = C.c_uint64(), C.c_uint64()
                assert lib.gs_stripe_range(total, r, world, C.byref(off), C.byref(ln)) == 0
                spans.append((off.value, ln.value))
            pos = 0
            for off, ln in spans:
                assert off == pos or ln == 0
                if ln:
                    assert off % 4096 == 0
                pos = max(pos, off + ln)
            assert sum(ln for _, ln in spans) == total


def test_row_ptrs_match_indexing():
    """row_ptrs (stride arithmetic) == per-row data_ptr() for contiguous,
    sliced and transposed-stripe views."""
    import torch
    from paper_2605_00831_b200.device import row_ptrs
    base = torch.zeros((6, 5, 64), dtype=torch.uint8)
    for t in (base, base[1:5], base[:, 1:4], base[:, :, 8:40], base.transpose(0, 1), base[2]):
        want = ([t[s, r].data_ptr() for s in range(t.shape[0]) for r in range(t.shape[1])] if t.dim() == 3
                else [t[r].data_ptr() for r in range(t.shape[0])])
        assert row_ptrs(t) == want


def test_fastdiv_magic_is_exact():
    """The kernels' invariant-divisor division (gs_kernels.cuh fdiv): exact
    for 32-bit numerators at the edges and at random, divisors 2 .. 2^32-1."""
    import random
    rnd = random.Random(7)
    divs = [2, 3, 5, 7, 16, 80, 4096, 65536, 16 * 256, 1 << 31, (1 << 32) - 1, 641, 6700417]
    divs += [rnd.randrange(2, 1 << 32) for _ in range(200)]
    for d in divs:
        m = ((1 << 64) - 1) // d + 1
        nums = [0, 1, d - 1, d, d + 1, (1 << 32) - 1, ((1 << 32) - 1) // d * d, ((1 << 32) - 1) // d * d - 1]
        nums += [rnd.randrange(0, 1 << 32) for _ in range(200)]
        for n in nums:
            if n < 0:
                continue
            r = n * (m >> 32) + ((n * (m & 0xFFFFFFFF)) >> 32)
            assert (r >> 32) == n // d, (n, d)


@pytest.mark.skipif(not O.have_ref(), reason="reference not compiled here (oracle/_ref)")
def test_random_schemes_decode_like_the_reference(port):
    """Arbitrary RS(n,k) (n+k up to 255) and random erasure patterns: the host
    decode plan of gs_decoder_create, applied with the CPU field math to random
    shards, returns exactly what the reference's own reconstruct returns
    (coding.hpp:458-571, compiled in place). Pins the host Gauss-Jordan /
    folding for schemes outside the compiled kernel set."""
    import random
    ref = O.ref()
    rng = random.Random(2024)
    mul = ref.mul_table()
    for trial in range(fuzz_trials(60)):
        k = rng.randint(1, 8)
        n = rng.randint(k, min(96, 255 - k))
        ln = rng.randint(1, 24)
        data = [np.frombuffer(rng.randbytes(ln), np.uint8).copy() for _ in range(n)]
        par = [np.zeros(ln, np.uint8) for _ in range(k)]
        ref.encode_timed(O.RS, n, k, data, par, 1)
        e = rng.randint(1, k)
        lost = sorted(rng.sample(range(n + k), e))
        shards = list(data) + list(par)
        slots = [None if j in lost else shards[j] for j in range(n + k)]
        lost_data = [j for j in lost if j < n]
        outs = [np.zeros(ln, np.uint8) for _ in lost_data]
        if lost_data:
            ref.reconstruct_timed(O.RS, n, k, slots, lost, outs, 1)
        c = G.codec_ex(G.CodingScheme.reed_solomon(n, k), G.ErasurePattern(lost))
        assert c.out_index == lost_data
        coef = c.coefficients()
        for b, j in enumerate(lost_data):
            acc = np.zeros(ln, np.uint8)
            for s in range(n + k):
                if coef[b, s]:
                    assert slots[s] is not None, (n, k, lost, s)
                    acc ^= mul[coef[b, s]][slots[s]]
            assert np.array_equal(acc, outs[b]), (trial, n, k, lost, j)
            assert np.array_equal(acc, data[j])


def test_reference_gf256_suite_runs_against_the_library():
    """The reference's own proj/tests/gf256_test.cpp (8 cases: known values,
    exhaustive schoolbook oracle, inverses, field laws, mul_row), compiled
    unmodified against the B200 library's GF(2^8) (tests/cpp/refsuite shims;
    built by build() into oracle/_ref when the reference is mounted)."""
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                       "ref_gf256_test_b200")
    if not os.path.exists(exe):
        pytest.skip("reference suites not built (no /root/reference at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "8 tests, 0 failed" in out.stdout


def test_host_fnv_bit_sliced_chain_matches_oracle(port):
    """The host FNV-1a (gs_fnv1a64, the checksums, the store's seal, the
    recovery verification) takes the bit-sliced AVX-512 chain of
    gs_fnv_simd.cpp when the CPU has it: bit-exact vs the oracle's serial
    chain (parity_store.hpp:19-25) at lengths around the 2 KiB super-block,
    from arbitrary chain states, at misaligned addresses, and over adversarial
    bytes (all-zero / all-0xFF runs keep the low-byte chain in short cycles)."""
    lib = L.lib()
    rng = np.random.default_rng(2026)
    big = rng.integers(0, 256, (1 << 20) + 4096, dtype=np.uint8)
    lens = [0, 1, 511, 2047, 2048, 2049, 4095, 4096, 6144 + 17, 65536, 65536 * 3 + 2048 + 5, 1 << 20]
    for ln in lens:
        for off in (0, 1, 63):
            buf = big[off: off + ln]
            for h0 in (0xCBF29CE484222325, int(rng.integers(0, 2**63)) * 2 + 1, 0):
                got = lib.gs_fnv1a64(buf.ctypes.data, ln, h0)
                assert got == port.fnv1a64(buf, h0), (ln, off, hex(h0))
    for fill in (0x00, 0xFF, 0x80, 0x01):
        buf = np.full(8192 + 100, fill, np.uint8)
        buf[4000] ^= 0x5A
        assert lib.gs_fnv1a64(buf.ctypes.data, buf.size, 0xCBF29CE484222325) == port.fnv1a64(buf)
    # the batch form (one chain per claim when the SIMD chain is present)
    parity = [rng.integers(0, 256, 40000, dtype=np.uint8) for _ in range(2 * 9)]
    out = (C.c_uint64 * 9)()
    assert lib.gs_parity_checksum_batch(L.ptr_array([p.ctypes.data for p in parity]), 9, 2, 40000, 4, out) == 0
    for c in range(9):
        assert out[c] == port.parity_checksum(parity[2 * c: 2 * c + 2])
    assert lib.gs_fnv_host_simd() in (0, 1)
    # the scalar chain (gs_fnv_host_set_simd(0), the A/B switch) gives the same sums
    buf = big[3: 3 + 70000]
    want = port.fnv1a64(buf)
    hw = lib.gs_fnv_host_simd()
    try:
        assert lib.gs_fnv_host_set_simd(0) == 0
        assert lib.gs_fnv1a64(buf.ctypes.data, buf.size, 0xCBF29CE484222325) == want
    finally:
        assert lib.gs_fnv_host_set_simd(1) == hw
    assert lib.gs_fnv1a64(buf.ctypes.data, buf.size, 0xCBF29CE484222325) == want


def test_process_wide_controls_without_a_gpu():
    """The small process-wide entry points behave without a device: ABI
    version, JIT switch (returns the previous state), JIT quiesce, zero-copy
    threshold setter, CUDA availability probe."""
    lib = L.lib()
    assert lib.gs_abi_version() >= 1
    prev = lib.gs_set_jit(0)
    assert prev in (0, 1)
    assert lib.gs_set_jit(prev) == 0          # the state set just before
    assert lib.gs_jit_quiesce() == 0
    assert lib.gs_set_zero_copy_bytes(2 << 20) == 0
    assert lib.gs_cuda_available() in (0, 1)
