"""K1/K2 on a paged KV cache: pages read / written in place,
partial blocks masked exactly like pad_partial; bytes checked against the
oracle on the gathered reference-layout slices."""
import numpy as np
import pytest
from fuzzutil import fuzz_trials

from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2605_00831_b200 import device as D  # noqa: E402
from paper_2605_00831_b200.coding import CodingScheme, ErasurePattern, InvalidArgument  # noqa: E402
from paper_2605_00831_b200.kv_layout import ModelConfig, make_ground_truth_slice  # noqa: E402
from paper_2605_00831_b200.paged import (PagedKVCache, checkpoint_blocks, encode_blocks,  # noqa: E402
                                         rebuild_blocks)


def build(model, n, S, block, valid, nblocks=64, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    caches = []
    for j in range(n):
        c = PagedKVCache(model, nblocks, block)
        c.buf.copy_(torch.randint(0, 256, c.buf.shape, dtype=torch.uint8, device="cuda", generator=g))
        caches.append(c)  # garbage everywhere, incl. past `valid`
    rng = np.random.default_rng(seed)
    perms = [rng.permutation(nblocks) for _ in range(n)]     # distinct blocks per worker across stripes
    tables = [[int(perms[j][s]) for j in range(n)] for s in range(S)]
    truth = []
    for s in range(S):
        row = []
        for j in range(n):
            sl = make_ground_truth_slice(3, s, 9, j, model, block, valid, device="cuda")
            caches[j].write_slice(tables[s][j], sl, valid)
            row.append(sl)
        truth.append(row)
    return caches, tables, truth


@pytest.mark.parametrize("valid", [16, 5, 0])
def test_paged_encode_equals_oracle_on_reference_slices(valid):
    model = ModelConfig(32, 8, 128, 2, 8)              # Llama-3-8B TP8: 4 KiB pages at block 16
    n, k, S = 8, 2, 6
    caches, tables, truth = build(model, n, S, 16, valid)
    scheme = CodingScheme.reed_solomon(n, k)
    par = torch.empty((S, k, caches[0].slice_bytes), dtype=torch.uint8, device="cuda")
    encode_blocks(scheme, caches, tables, valid, par)
    hp = par.cpu().numpy()
    for s in range(S):
        host = [t.cpu().numpy() for t in truth[s]]
        for j in range(n):
            assert np.array_equal(caches[j].read_slice(tables[s][j], valid).cpu().numpy(), host[j])
        want = O.port().encode(O.RS, n, k, host)
        for i in range(k):
            assert np.array_equal(hp[s, i], want[i]), (valid, s, i)


def test_paged_checkpoint_and_rebuild_into_replacement_cache():
    model = ModelConfig(2, 6, 64, 2, 6)                # 6-divisible geometry, RS(6,2)
    n, k, S, valid = 6, 2, 5, 11
    caches, tables, truth = build(model, n, S, 16, valid, nblocks=40, seed=3)
    scheme = CodingScheme.reed_solomon(n, k)
    pipe = D.Pipeline(0, 64 << 10)                     # tiny ring: many pieces across page boundaries
    h_par = torch.zeros((S, k, caches[0].slice_bytes), dtype=torch.uint8).pin_memory()
    comp, copy = torch.cuda.Stream(), torch.cuda.Stream()
    comp.wait_stream(torch.cuda.current_stream())
    checkpoint_blocks(pipe, scheme, caches, tables, valid, h_par, comp, copy)
    copy.synchronize()
    for s in range(S):
        want = O.port().encode(O.RS, n, k, [t.cpu().numpy() for t in truth[s]])
        for i in range(k):
            assert np.array_equal(h_par[s, i].numpy(), want[i])
    for lost in ([2], [0, 4], [5, 7]):
        pat = ErasurePattern(lost)
        reps = {}
        for w in lost:
            if w < n:
                reps[w] = PagedKVCache(model, 40, 16, fill=0xEE)
        rebuild_blocks(pipe, scheme, pat, [None if j in lost else caches[j] for j in range(n)], reps, tables,
                       valid, h_par, comp, copy)
        comp.synchronize()
        for w, rep in reps.items():
            for s in range(S):
                assert torch.equal(rep.read_slice(tables[s][w], valid), truth[s][w]), (lost, w, s)
                # tokens past `valid` of the page are never written
                assert bool((rep.buf[:, :, tables[s][w], valid:] == 0xEE).all())
    pipe.close()


def test_paged_rejects_bad_geometry():
    model = ModelConfig(2, 8, 8, 2, 8)                 # 16 B/token: fine
    c = PagedKVCache(model, 4, 16)
    with pytest.raises(InvalidArgument):
        c.page_map(17)
    bad = ModelConfig(2, 4, 2, 2, 1)                  # 16 B tokens but check odd strides via apply
    cb = PagedKVCache(bad, 4, 3)                       # 3-token pages of 16 B -> 48 B pages: ok (multiple of 16)
    par = torch.empty((1, 1, cb.slice_bytes), dtype=torch.uint8, device="cuda")
    encode_blocks(CodingScheme.xor_code(2), [cb, cb], [[0, 1]], 3, par)


@pytest.mark.parametrize("model,block,chunk", [
    (ModelConfig(32, 8, 128, 2, 8), 16, 64),     # 4 KiB blocks: CTA-uniform table lookups
    (ModelConfig(2, 8, 8, 2, 8), 16, 128),       # 256 B blocks: per-thread mapping path
])
@pytest.mark.parametrize("valid", [None, 37])
def test_paged_multi_block_chunks_with_block_table(model, block, chunk, valid):
    from paper_2605_00831_b200.paged import checkpoint_chunks, rebuild_chunks
    n, k, S = 8, 2, 3
    v = chunk if valid is None else valid
    nblk = chunk // block
    nblocks = S * nblk + 5
    g = torch.Generator(device="cuda").manual_seed(7)
    caches = []
    for j in range(n):
        c = PagedKVCache(model, nblocks, block)
        c.buf.copy_(torch.randint(0, 256, c.buf.shape, dtype=torch.uint8, device="cuda", generator=g))
        caches.append(c)
    perm = np.random.default_rng(5).permutation(nblocks)[: S * nblk].reshape(S, nblk)
    table = torch.from_numpy(perm.astype(np.int32)).cuda()
    truth = []
    for s in range(S):
        row = []
        for j in range(n):
            sl = make_ground_truth_slice(3, s, 2, j, model, chunk, v, device="cuda")
            caches[j].write_chunk(perm[s], sl, chunk, v)
            row.append(sl)
        truth.append(row)
    scheme = CodingScheme.reed_solomon(n, k)
    pipe = D.Pipeline(0, 256 << 10)
    slice_bytes = caches[0].chunk_slice_bytes(chunk)
    h_par = torch.zeros((S, k, slice_bytes), dtype=torch.uint8).pin_memory()
    st = torch.cuda.current_stream()
    checkpoint_chunks(pipe, scheme, caches, table, chunk, v, h_par, st, st)
    st.synchronize()
    for s in range(S):
        want = O.port().encode(O.RS, n, k, [t.cpu().numpy() for t in truth[s]])
        for i in range(k):
            assert np.array_equal(h_par[s, i].numpy(), want[i]), (s, i)
    lost = ErasurePattern([1, 6])
    reps = {w: PagedKVCache(model, nblocks, block, fill=0x5A) for w in (1, 6)}
    rebuild_chunks(pipe, scheme, lost, [None if j in (1, 6) else caches[j] for j in range(n)], reps, table, chunk, v,
                   h_par, st, st)
    st.synchronize()
    for w in (1, 6):
        for s in range(S):
            assert torch.equal(reps[w].read_chunk(perm[s], chunk, v), truth[s][w]), (w, s)
    pipe.close()


def test_paged_fuzz_geometries():
    """Random model geometries (layers, heads, head dim, tp), block sizes,
    chunk sizes (one or several blocks per chunk), valid-token counts, schemes
    and staging rings through checkpoint_chunks / rebuild_chunks: parity and
    rebuilt pages bit-exact vs the oracle on the reference-layout slices."""
    import random
    from paper_2605_00831_b200.paged import checkpoint_chunks, rebuild_chunks
    rng = random.Random(31337)
    for trial in range(fuzz_trials(30)):
        tp = rng.choice([2, 4, 6, 8])
        heads = tp * rng.choice([1, 2])
        model = ModelConfig(rng.choice([1, 2, 3, 5]), heads, rng.choice([8, 16, 64, 128]), 2, tp)
        block = rng.choice([1, 2, 8, 16])
        chunk = block * rng.choice([1, 2, 4])
        n = tp
        k = rng.randint(1, min(3, n))
        valid = rng.randint(0, chunk)
        S = rng.randint(1, 4)
        nblk = chunk // block
        nblocks = S * nblk + rng.randint(0, 4)
        g = torch.Generator(device="cuda").manual_seed(trial)
        caches = []
        for j in range(n):
            c = PagedKVCache(model, nblocks, block)
            c.buf.copy_(torch.randint(0, 256, c.buf.shape, dtype=torch.uint8, device="cuda", generator=g))
            caches.append(c)
        perm = np.random.default_rng(trial).permutation(nblocks)[: S * nblk].reshape(S, nblk)
        table = torch.from_numpy(perm.astype(np.int32)).cuda()
        truth = []
        for s in range(S):
            row = []
            for j in range(n):
                sl = make_ground_truth_slice(3, s, trial, j, model, chunk, valid, device="cuda")
                caches[j].write_chunk(perm[s], sl, chunk, valid)
                row.append(sl)
            truth.append(row)
        scheme = CodingScheme.reed_solomon(n, k)
        pipe = D.Pipeline(0, rng.choice([16 << 10, 64 << 10, 1 << 20]))
        slice_bytes = caches[0].chunk_slice_bytes(chunk)
        h_par = torch.zeros((S, k, slice_bytes), dtype=torch.uint8).pin_memory()
        st = torch.cuda.current_stream()
        ctx = (trial, model, block, chunk, valid, n, k, S)
        checkpoint_chunks(pipe, scheme, caches, table, chunk, valid, h_par, st, st)
        st.synchronize()
        for s in range(S):
            want = O.port().encode(O.RS, n, k, [t.cpu().numpy() for t in truth[s]])
            for i in range(k):
                assert np.array_equal(h_par[s, i].numpy(), want[i]), ctx
        lost_w = sorted(rng.sample(range(n), rng.randint(1, k)))
        reps = {w: PagedKVCache(model, nblocks, block, fill=0xA5) for w in lost_w}
        rebuild_chunks(pipe, scheme, ErasurePattern(lost_w), [None if j in lost_w else caches[j] for j in range(n)],
                       reps, table, chunk, valid, h_par, st, st)
        st.synchronize()
        for w in lost_w:
            for s in range(S):
                assert torch.equal(reps[w].read_chunk(perm[s], chunk, valid), truth[s][w]), ctx + (w, s)
        pipe.close()


@pytest.mark.parametrize("model,staging", [
    (ModelConfig(32, 8, 128, 2, 8), 16 << 10),    # 4 KiB pages, pieces of 16 KiB: logical0 > 0
    (ModelConfig(4, 16, 128, 2, 8), 64 << 10),    # 8 KiB pages (two tiles per page)
    (ModelConfig(3, 8, 128, 2, 8), 1 << 20),      # whole slice in one piece
])
def test_paged_tile_pages_path_pipelined(model, staging):
    """The page-per-tile paged K1 (single-block chunks, every token valid,
    pages a whole number of 4 KiB tiles: gs_kernels.cuh TileGeom.tile_pages)
    through the pipelined decode-block checkpoint, whose pieces start at
    logical offsets > 0: parity bit-exact vs the oracle."""
    n, k, S = 8, 2, 7
    caches, tables, truth = build(model, n, S, 16, 16, nblocks=48, seed=5)
    scheme = CodingScheme.reed_solomon(n, k)
    pipe = D.Pipeline(0, staging)
    h_par = torch.zeros((S, k, caches[0].slice_bytes), dtype=torch.uint8).pin_memory()
    st = torch.cuda.current_stream()
    checkpoint_blocks(pipe, scheme, caches, tables, 16, h_par, st, st)
    st.synchronize()
    for s in range(S):
        want = O.port().encode(O.RS, n, k, [t.cpu().numpy() for t in truth[s]])
        for i in range(k):
            assert np.array_equal(h_par[s, i].numpy(), want[i]), (s, i)


@pytest.mark.parametrize("model,block,chunk,staging", [
    (ModelConfig(4, 16, 128, 2, 8), 16, 64, 16 << 10),   # 8 KiB blocks (2 tiles each), pieces of 16 KiB
    (ModelConfig(32, 8, 128, 2, 8), 16, 128, 1 << 20),   # 4 KiB blocks, 8 blocks per chunk
])
def test_paged_tile_pages_with_block_table(model, block, chunk, staging):
    """The page-per-tile path through a block table (tiles inside one block,
    every token valid), pipelined so pieces start mid-block: parity bit-exact
    vs the oracle (gs_kernels.cuh TileGeom.tile_pages)."""
    from paper_2605_00831_b200.paged import checkpoint_chunks
    n, k, S = 8, 2, 5
    nblk = chunk // block
    nblocks = S * nblk + 3
    g = torch.Generator(device="cuda").manual_seed(11)
    caches = []
    for j in range(n):
        c = PagedKVCache(model, nblocks, block)
        c.buf.copy_(torch.randint(0, 256, c.buf.shape, dtype=torch.uint8, device="cuda", generator=g))
        caches.append(c)
    perm = np.random.default_rng(9).permutation(nblocks)[: S * nblk].reshape(S, nblk)
    table = torch.from_numpy(perm.astype(np.int32)).cuda()
    truth = []
    for s in range(S):
        row = []
        for j in range(n):
            sl = make_ground_truth_slice(3, s, 4, j, model, chunk, chunk, device="cuda")
            caches[j].write_chunk(perm[s], sl, chunk, chunk)
            row.append(sl)
        truth.append(row)
    scheme = CodingScheme.reed_solomon(n, k)
    pipe = D.Pipeline(0, staging)
    h_par = torch.zeros((S, k, caches[0].chunk_slice_bytes(chunk)), dtype=torch.uint8).pin_memory()
    st = torch.cuda.current_stream()
    checkpoint_chunks(pipe, scheme, caches, table, chunk, chunk, h_par, st, st)
    st.synchronize()
    for s in range(S):
        want = O.port().encode(O.RS, n, k, [t.cpu().numpy() for t in truth[s]])
        for i in range(k):
            assert np.array_equal(h_par[s, i].numpy(), want[i]), (s, i)
    pipe.close()
