"""bench.py's reference arm runs on the host alone (the driver launches it
on the GPU box next to our arm): its JSON line keeps the driver's contract
and carries the SAME `config` object as our arm for the workload, so the
driver's same-config check compares like with like (tools/ghostserve.cpp:238-290
is the reference's own bench this arm follows)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line_keeps_the_contract():
    sys.path.insert(0, ROOT)
    import bench
    from oracle import oracle as O
    if not O.have_ref():
        pytest.skip("oracle/_ref not built")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "c2",
                          "--steps", "1", "--warmup", "0"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"] == bench.METRIC and line["unit"] == "GB/s" and line["higher_is_better"] is True
    assert line["value"] > 0 and line["warmup"] >= 3 and line["n_gpus"] == 1
    assert line["config"] == bench.workload_config(bench.WORKLOADS["c2"], 1)
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_workload_configs_are_arm_independent():
    sys.path.insert(0, ROOT)
    import bench
    for key, W in bench.WORKLOADS.items():
        for world in (1, 2, 8):
            c = bench.workload_config(W, world)
            assert c["workload"].startswith(key.upper()) and c["n_ranks"] == world
            assert c["data_bytes_per_step"] == W.stripes * 8 * W.slice * world
            assert c["parity_d2h_bytes_per_step"] * 4 == c["data_bytes_per_step"]
            json.dumps(c)
