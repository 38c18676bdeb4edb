"""e2e host-buffer encode (gs_encode_host) vs host-piece size, plus the raw
PCIe copy rates it is bounded by (H2D alone, D2H alone, both at once).

Runs one child process per GS_HOST_PIECE value (read at library load).
  python tools/e2e_sweep.py [--pieces 131072,262144,524288,1048576,2097152]
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(steps):
    import torch
    from paper_2605_00831_b200 import _lib as L, coding as G, device as D
    from paper_2605_00831_b200.coding import check
    per = 32 * 262144
    h_in = torch.randint(0, 256, (8, per), dtype=torch.uint8).pin_memory()
    h_out = torch.empty((2, per), dtype=torch.uint8).pin_memory()
    enc = G.encoder(G.CodingScheme.reed_solomon(8, 2))
    pipe = D.Pipeline(0, 256 << 20)
    lib = L.lib()
    pi = L.ptr_array([h_in[j].data_ptr() for j in range(8)])
    po = L.ptr_array([h_out[i].data_ptr() for i in range(2)])
    for _ in range(5):
        check(lib.gs_encode_host(pipe.handle, enc.handle, pi, po, per), "e2e")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        check(lib.gs_encode_host(pipe.handle, enc.handle, pi, po, per), "e2e")
    dt = (time.perf_counter() - t0) / steps
    ok = torch.equal(h_out.cuda(), D.encode(G.CodingScheme.reed_solomon(8, 2), h_in.cuda()))
    return {"ms_per_call": round(dt * 1e3, 4), "e2e_gbs": round(8 * per / dt / 1e9, 2), "parity_ok": ok}


def links(steps):
    import torch
    a = torch.empty(64 << 20, dtype=torch.uint8).pin_memory()
    b = torch.empty(16 << 20, dtype=torch.uint8).pin_memory()
    da = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    db = torch.empty(16 << 20, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def run(h2d, d2h):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            if h2d:
                with torch.cuda.stream(s1):
                    da.copy_(a, non_blocking=True)
            if d2h:
                with torch.cuda.stream(s2):
                    b.copy_(db, non_blocking=True)
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / steps

    run(True, True)
    t_h, t_d, t_b = run(True, False), run(False, True), run(True, True)
    return {"h2d_gbs": round(da.numel() / t_h / 1e9, 2), "d2h_gbs": round(db.numel() / t_d / 1e9, 2),
            "both_ms": round(t_b * 1e3, 4), "both_h2d_gbs": round(da.numel() / t_b / 1e9, 2),
            "ideal_e2e_ms": round(max(t_h, t_d) * 1e3, 4)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pieces", default="131072,262144,524288,1048576,2097152,4194304")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--links", action="store_true")
    a = ap.parse_args()
    if a.child:
        print(json.dumps(child(a.steps)))
        return
    if a.links:
        print(json.dumps(links(a.steps)))
        return
    print(json.dumps(dict(links=json.loads(subprocess.check_output(
        [sys.executable, __file__, "--links", "--steps", str(a.steps)], cwd=ROOT).decode().strip().splitlines()[-1]))),
        flush=True)
    for pc in a.pieces.split(","):
        out = subprocess.check_output([sys.executable, __file__, "--child", "--steps", str(a.steps)], cwd=ROOT,
                                      env=dict(os.environ, GS_HOST_PIECE=pc)).decode().strip().splitlines()[-1]
        print(json.dumps({"host_piece": int(pc), **json.loads(out)}), flush=True)


if __name__ == "__main__":
    main()
