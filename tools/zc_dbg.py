import sys, os
sys.path.insert(0, os.getcwd())
import ctypes as C, numpy as np, torch
from paper_2605_00831_b200 import _lib as L, coding as G
from oracle import oracle as O
from tests.golden.vectors import splitmix_bytes
lib = L.lib()
st = torch.cuda.current_stream()
for (n, k) in ((8, 2),):
    for ln in (4096 * 9 + 48, 4096*9, 65536, 4096):
        enc = C.c_void_p()
        G.check(lib.gs_codec_create(2, n, k, C.byref(enc)), "codec_create")
        host = [splitmix_bytes(700 + 13 * n + j, ln) for j in range(n)]
        want = O.port().encode(O.RS, n, k, host)
        data = torch.stack([torch.from_numpy(h) for h in host]).cuda()
        hp = torch.zeros((k, ln), dtype=torch.uint8).pin_memory()
        b0 = lib.gs_zero_copy_offloads()
        G.check(lib.gs_encode_async(enc, L.ptr_array([data[j].data_ptr() for j in range(n)]), ln,
                                    L.ptr_array([hp[i].data_ptr() for i in range(k)]), st.cuda_stream, st.cuda_stream), "e")
        G.check(lib.gs_sync(st.cuda_stream), "sync")
        torch.cuda.synchronize()
        for i in range(k):
            got = hp[i].numpy()
            bad = np.nonzero(got != want[i])[0]
            print(ln, i, "zc", lib.gs_zero_copy_offloads() - b0, "bad", len(bad), bad[:5], bad[-5:] if len(bad) else "", hp.data_ptr() % 4096, hp[1].data_ptr() - hp[0].data_ptr())
