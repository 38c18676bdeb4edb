"""K1 throughput by scheme and shard layout (not the bench): RS(4,2) /
RS(6,2) / RS(8,2) encodes over shards spaced exactly one shard apart (one
contiguous [n, L] tensor, as bench --configs allocates them) or with a 4 KiB
pad between shards, for each kernel variant (0 = LDG.128, 1 = bulk TMA ring,
2 = auto). Events on the launch stream over 4 rotating sets."""
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
for (n, k, ln) in [(4, 2, 128 << 20), (8, 2, 64 << 20), (6, 2, 80 << 20)]:
    for pad in (0, 4096):
        sets = 4
        pitch = ln + pad
        data = torch.randint(0, 256, (sets, n, pitch), dtype=torch.uint8, device=dev)
        out = torch.empty((sets, k, pitch), dtype=torch.uint8, device=dev)
        enc = encoder(CodingScheme.reed_solomon(n, k))
        slots = [L.ptr_array([data[s, j].data_ptr() for j in range(n)]) for s in range(sets)]
        outs = [L.ptr_array([out[s, i].data_ptr() for i in range(k)]) for s in range(sets)]
        for var in (0, 1):
            lib.gs_set_kernel_variant(var)

            def run(s):
                check(lib.gs_apply_device(enc.handle, 1, slots[s], outs[s], ln, st.cuda_stream), "k1")
            for s in range(sets):
                run(s)
            st.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for r in range(5):
                for s in range(sets):
                    run(s)
            e1.record(st)
            e1.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / (5 * sets)
            print(json.dumps({"rs": f"({n},{k})", "shard_mib": ln >> 20, "pad": pad, "variant": var,
                              "us": round(us, 1), "tbs": round((n + k) * ln / us / 1e6, 3)}), flush=True)
        lib.gs_set_kernel_variant(2)
        del data, out
