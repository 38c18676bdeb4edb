"""K1 sensitivity to the shards' relative placement (not the bench): RS(8,2)
encode of S stripes x 8 shards of L bytes, the shards of one stripe spaced
L + pad bytes apart inside one allocation, for both kernel variants
(0 = LDG.128 register kernel, 1 = bulk TMA ring). Events on the launch
stream, 4 rotating sets."""
import json
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2605_00831_b200 import _lib as L  # noqa: E402
from paper_2605_00831_b200.coding import CodingScheme, check, encoder  # noqa: E402

lib = L.lib()
dev = torch.device("cuda", 0)
st = torch.cuda.Stream()
n, k = 8, 2
enc = encoder(CodingScheme.reed_solomon(n, k))
geos = [(32, 256 << 10), (1, 32 << 20)] if len(sys.argv) < 2 else [tuple(int(x) for x in a.split("x")) for a in sys.argv[1:]]
for S, ln in geos:
    for pad in (0, 16, 512, 4096, 65536, 12288):
        sets = 4
        pitch = ln + pad
        data = torch.randint(0, 256, (sets, S, n, pitch), dtype=torch.uint8, device=dev)
        out = torch.empty((sets, S, k, ln), dtype=torch.uint8, device=dev)
        slots = [L.ptr_array([data[b, s, j].data_ptr() for s in range(S) for j in range(n)]) for b in range(sets)]
        outs = [L.ptr_array([out[b, s, i].data_ptr() for s in range(S) for i in range(k)]) for b in range(sets)]
        row = {"stripes": S, "shard_bytes": ln, "pad": pad}
        for var in (0, 1):
            lib.gs_set_kernel_variant(var)

            def run(b):
                check(lib.gs_apply_device(enc.handle, S, slots[b], outs[b], ln, st.cuda_stream), "k1")
            for b in range(sets):
                run(b)
            st.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for r in range(5):
                for b in range(sets):
                    run(b)
            e1.record(st)
            e1.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / (5 * sets)
            row[f"v{var}_tbs"] = round(S * (n + k) * ln / us / 1e6, 3)
        lib.gs_set_kernel_variant(2)
        print(json.dumps(row), flush=True)
        del data, out
