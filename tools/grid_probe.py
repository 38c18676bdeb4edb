"""K1 at the C2 launch (32 stripes x RS(8,2) x 256 KiB) under tuning env
overrides (GS_CTAS_PER_SM, GS_FULL_GRID, GS_PDL); CUDA-graph timed, 8 rotating
blocks. Prints us/launch and GB/s per configuration (child processes)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child():
    import torch
    from paper_2605_00831_b200 import _lib as L
    from paper_2605_00831_b200.coding import CodingScheme, check, encoder
    from tools.kernel_sweep import graph_time
    S, n, k, ln, B = 32, 8, 2, 262144, 8
    data = torch.randint(0, 256, (B, S, n, ln), dtype=torch.uint8, device="cuda")
    par = torch.empty((B, S, k, ln), dtype=torch.uint8, device="cuda")
    enc = encoder(CodingScheme.reed_solomon(n, k))
    sl = [L.ptr_array([data[b, s, j].data_ptr() for s in range(S) for j in range(n)]) for b in range(B)]
    ol = [L.ptr_array([par[b, s, i].data_ptr() for s in range(S) for i in range(k)]) for b in range(B)]
    st = torch.cuda.Stream()
    cnt = [0]

    def k1():
        b = cnt[0] % B
        cnt[0] += 1
        check(L.lib().gs_apply_device(enc.handle, S, sl[b], ol[b], ln, st.cuda_stream))
    best = min(graph_time(k1, 32, st) for _ in range(3))
    return {"us": round(best * 1e6, 2), "gbs": round(S * (n + k) * ln / best / 1e9, 1)}


if __name__ == "__main__":
    if "--child" in sys.argv:
        print(json.dumps(child()))
        sys.exit(0)
    confs = [{}, {"GS_FULL_GRID": "1"}] + [{"GS_CTAS_PER_SM": str(c)} for c in (2, 3, 4, 5)]
    if "--confs" in sys.argv:  # e.g. --confs '[{"GS_PDL": "0"}, {}]'
        confs = json.loads(sys.argv[sys.argv.index("--confs") + 1])
    for c in confs:
        out = subprocess.check_output([sys.executable, __file__, "--child"], cwd=ROOT,
                                      env=dict(os.environ, **c)).decode().strip().splitlines()[-1]
        print(json.dumps({"env": c, **json.loads(out)}), flush=True)
