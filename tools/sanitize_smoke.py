"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family once -- specialised (register + bulk-copy pipeline),
generic (aligned, ragged tail, misaligned), paged gather/scatter (incl. the
page-per-tile path), the
offload / upload pipelines (with live kernel timing stamps), RDP (pipelined
body + tile remainder + P/Q tail, two-column and single-column recovery) and
a runtime-specialised (NVRTC) kernel, the GPU FNV-1a seal and the split
parity verification -- at sizes that finish quickly under
instrumentation. Exits non-zero on any byte mismatch vs the oracle.

    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_2605_00831_b200 import _lib as L  # noqa: E402
from paper_2605_00831_b200 import device as D  # noqa: E402
from paper_2605_00831_b200.coding import CodingScheme, ErasurePattern, codec_ex  # noqa: E402
from paper_2605_00831_b200.kv_layout import ModelConfig, make_ground_truth_slice  # noqa: E402
from paper_2605_00831_b200.paged import PagedKVCache, encode_blocks, rebuild_blocks  # noqa: E402


def main():
    torch.cuda.set_device(0)
    g = torch.Generator(device="cuda").manual_seed(1)
    bad = 0
    for variant in (0, 1):
        L.lib().gs_set_kernel_variant(variant)
        for n, k, ln in ((8, 2, 3 * 4096 + 32), (4, 2, 4096 + 5), (9, 3, 1000)):
            sch = CodingScheme.reed_solomon(n, k)
            data = torch.randint(0, 256, (n, ln), dtype=torch.uint8, device="cuda", generator=g)
            par = D.encode(sch, data)
            want = O.port().encode(O.RS, n, k, list(data.cpu().numpy()))
            bad += sum(not np.array_equal(par[i].cpu().numpy(), want[i]) for i in range(k))
            lost = ErasurePattern([0, n])
            sh = {j: data[j] for j in range(1, n)}
            sh.update({n + i: par[i] for i in range(1, k)})
            got = D.reconstruct(sch, sh, lost)
            bad += not torch.equal(got[0], data[0])
    L.lib().gs_set_kernel_variant(2)
    # generic on misaligned pointers
    sch = CodingScheme.reed_solomon(8, 2)
    buf = torch.randint(0, 256, (8, 4096 + 64), dtype=torch.uint8, device="cuda", generator=g)
    out = torch.zeros((2, 4096 + 64), dtype=torch.uint8, device="cuda")
    c = codec_ex(sch, generic=True)
    D.apply(c, [[buf[j, 3:].data_ptr() for j in range(8)]], [[out[i, 3:].data_ptr() for i in range(2)]], 4096 + 17)
    want = O.port().encode(O.RS, 8, 2, [buf[j, 3:3 + 4096 + 17].cpu().numpy() for j in range(8)])
    bad += sum(not np.array_equal(out[i, 3:3 + 4096 + 17].cpu().numpy(), want[i]) for i in range(2))
    # pipelines
    pipe = D.Pipeline(0, 64 << 10)
    data = torch.randint(0, 256, (3, 8, 3 * 4096 + 16), dtype=torch.uint8, device="cuda", generator=g)
    h = torch.zeros((3, 2, data.shape[-1]), dtype=torch.uint8).pin_memory()
    st = torch.cuda.current_stream()
    pipe.encode_offload(sch, data, h, st, st)
    st.synchronize()
    bad += not torch.equal(h, D.encode(sch, data).cpu())
    outs = {2: torch.zeros((3, data.shape[-1]), dtype=torch.uint8, device="cuda")}
    pipe.reconstruct_upload(sch, ErasurePattern([2]), {j: data[:, j].contiguous() for j in range(8) if j != 2}, h,
                            outs, st, st)
    st.synchronize()
    bad += not torch.equal(outs[2], data[:, 2])
    # paged
    model = ModelConfig(2, 8, 8, 2, 8)
    caches = [PagedKVCache(model, 6, 16) for _ in range(8)]
    truth = []
    for j in range(8):
        caches[j].buf.zero_()
        sl = make_ground_truth_slice(3, 0, 0, j, model, 16, 9, device="cuda")
        caches[j].write_slice(j % 6, sl, 9)
        truth.append(sl)
    tables = [[j % 6 for j in range(8)]]
    par = torch.empty((1, 2, caches[0].slice_bytes), dtype=torch.uint8, device="cuda")
    encode_blocks(sch, caches, tables, 9, par)
    want = O.port().encode(O.RS, 8, 2, [t.cpu().numpy() for t in truth])
    bad += sum(not np.array_equal(par[0, i].cpu().numpy(), want[i]) for i in range(2))
    hp = par.cpu().pin_memory()
    rep = {4: PagedKVCache(model, 6, 16, fill=0)}
    rebuild_blocks(pipe, sch, ErasurePattern([4]), [None if j == 4 else caches[j] for j in range(8)], rep, tables,
                   9, hp, st, st)
    st.synchronize()
    bad += not torch.equal(rep[4].read_slice(4, 9), truth[4])
    # paged, page-per-tile path (4 KiB pages, every token valid: TileGeom.tile_pages)
    model4k = ModelConfig(4, 8, 128, 2, 8)
    caches4k = [PagedKVCache(model4k, 3, 16) for _ in range(8)]
    truth4k = []
    for j in range(8):
        sl = make_ground_truth_slice(3, 1, 0, j, model4k, 16, 16, device="cuda")
        caches4k[j].write_slice((j + 1) % 3, sl, 16)
        truth4k.append(sl)
    par4k = torch.empty((1, 2, caches4k[0].slice_bytes), dtype=torch.uint8, device="cuda")
    encode_blocks(sch, caches4k, [[(j + 1) % 3 for j in range(8)]], 16, par4k)
    want4k = O.port().encode(O.RS, 8, 2, [t.cpu().numpy() for t in truth4k])
    bad += sum(not np.array_equal(par4k[0, i].cpu().numpy(), want4k[i]) for i in range(2))
    # pipelines with live kernel timing (globaltimer stamps)
    import ctypes as C
    L.lib().gs_pipeline_set_timing(pipe.handle, 1)
    pipe.encode_offload(sch, data, h, st, st)
    st.synchronize()
    ev, dv, grp, nl = C.c_double(), C.c_double(), C.c_int(), C.c_uint64()
    L.lib().gs_pipeline_kernel_time(pipe.handle, C.byref(ev), C.byref(dv), C.byref(grp), C.byref(nl))
    L.lib().gs_pipeline_set_timing(pipe.handle, 0)
    bad += grp.value < 1 or dv.value <= 0
    bad += not torch.equal(h, D.encode(sch, data).cpu())
    # RDP(8): p = 11, two pipelined tiles + tile-kernel remainder + P/Q tail
    rdp = CodingScheme.rdp(8)
    ln = 2 * 1024 * 10 + 37 * 10 + 3
    data = torch.randint(0, 256, (2, 8, ln), dtype=torch.uint8, device="cuda", generator=g)
    par = D.encode(rdp, data)
    for s_ in range(2):
        want = O.port().encode(O.RDP, 8, 2, list(data[s_].cpu().numpy()))
        bad += sum(not np.array_equal(par[s_, i].cpu().numpy(), want[i]) for i in range(2))
    for lost in ([1, 6], [3, 8], [5]):
        sh = {j: data[:, j].contiguous() for j in range(8) if j not in lost}
        sh.update({8 + i: par[:, i].contiguous() for i in range(2) if 8 + i not in lost})
        got = D.reconstruct(rdp, sh, ErasurePattern(lost))
        bad += sum(not torch.equal(t, data[:, j]) for j, t in got.items())
    # runtime-specialised kernel (NVRTC), RS(9,2) is outside the compiled set
    from paper_2605_00831_b200.coding import encoder
    sch9 = CodingScheme.reed_solomon(9, 2)
    enc9 = encoder(sch9)
    js = C.c_int()
    L.lib().gs_codec_jit_status(enc9.handle, 1, C.byref(js))
    data = torch.randint(0, 256, (9, 3 * 4096), dtype=torch.uint8, device="cuda", generator=g)
    par = D.encode(sch9, data)
    want = O.port().encode(O.RS, 9, 2, list(data.cpu().numpy()))
    bad += sum(not np.array_equal(par[i].cpu().numpy(), want[i]) for i in range(2))
    # GPU FNV-1a seal (all 18 kernels: partial last block, several chains) and
    # the split verification (GPU-hashed rows continued by host threads)
    port = O.port()
    ln = 16384 * 2 + 4096 + 48
    rows = torch.randint(0, 256, (3, 2, ln), dtype=torch.uint8, device="cuda", generator=g)
    sums = torch.zeros(3, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    ptrs = L.ptr_array([rows[c, i].data_ptr() for c in range(3) for i in range(2)])
    assert L.lib().gs_fnv1a64_device(ptrs, 3, 2, ln, 0xCBF29CE484222325, sums.data_ptr(), st.cuda_stream) == 0
    host = rows.cpu()
    want = [port.parity_checksum([host[c, 0].numpy(), host[c, 1].numpy()]) for c in range(3)]
    bad += sum((int(v) & (2**64 - 1)) != w for v, w in zip(sums.cpu().tolist(), want))
    hp = host.pin_memory()
    dev = torch.zeros_like(rows)
    torch.cuda.synchronize()
    h = C.c_void_p()
    drows = [dev[c, i].data_ptr() if (c < 1 or i < 1) else None for c in range(3) for i in range(2)]
    assert L.lib().gs_verify_enqueue(L.ptr_array([hp[c, i].data_ptr() for c in range(3) for i in range(2)]), 3, 2,
                                     ln, 1, 1, L.ptr_array(drows), st.cuda_stream, st.cuda_stream, C.byref(h)) == 0
    out = (C.c_uint64 * 3)()
    assert L.lib().gs_verify_finish(h, 2, out) == 0
    bad += sum(out[c] != want[c] for c in range(3))
    # dynamic split (n_full = -1) with rates set, so idle host threads take whole
    # chains from the back and the feeder serves the rest
    dev.zero_()
    torch.cuda.synchronize()
    drows = [dev[c, i].data_ptr() for c in range(3) for i in range(2)]
    assert L.lib().gs_verify_enqueue(L.ptr_array([hp[c, i].data_ptr() for c in range(3) for i in range(2)]), 3, 2,
                                     ln, -1, 1, L.ptr_array(drows), st.cuda_stream, st.cuda_stream, C.byref(h)) == 0
    assert L.lib().gs_verify_set_rates(h, 0.5, 0.2) == 0
    out = (C.c_uint64 * 3)()
    assert L.lib().gs_verify_finish(h, 2, out) == 0
    bad += sum(out[c] != want[c] for c in range(3))
    # the N>1 checksum relay's GPU worker on a one-rank board: row 0 hashed on the
    # GPU (seeded window kernel), row 1 on host threads
    ln16 = ln - ln % 16
    board = (C.c_uint8 * L.lib().gs_relay_board_bytes(3, 2, 1))()
    sums_r = (C.c_uint64 * 3)()
    assert L.lib().gs_fnv_relay_device(board, 1, 0, 1, L.ptr_array([rows[c, 0].data_ptr() for c in range(3)]), 1,
                                       None, L.ptr_array([hp[c, i].data_ptr() for c in range(3) for i in range(2)]),
                                       ln16, 3, 2, 0xCBF29CE484222325, 2, 2, st.cuda_stream, 30.0, sums_r) == 0
    want16 = [port.parity_checksum([host[c, 0].numpy()[:ln16], host[c, 1].numpy()[:ln16]]) for c in range(3)]
    bad += sum(sums_r[c] != want16[c] for c in range(3))
    pipe.close()
    torch.cuda.synchronize()
    print("sanitize_smoke: mismatches =", bad, "kernels =", D.launches(), "jit status =", js.value)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
