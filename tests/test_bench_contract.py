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


def test_reference_arm_under_two_ranks_prints_one_line():
    """`--impl reference --gpus 2` (re-exec under torch.distributed.run, as the
    driver's scaling run launches it): rank 0 alone runs the reference codec and
    prints the line with n_gpus = 2 and our arm's N=2 config; rank 1 exits 0."""
    sys.path.insert(0, ROOT)
    import bench
    from oracle import oracle as O
    if not O.have_ref():
        pytest.skip("oracle/_ref not built")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--workload", "c2", "--steps", "1", "--warmup", "0"], cwd=ROOT, capture_output=True,
                         text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"] == bench.workload_config(bench.WORKLOADS["c2"], 2)


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


@pytest.mark.gpu
def test_two_rank_bench_line_on_one_gpu():
    """`bench.py --gpus 2` re-execs itself under torch.distributed.run and
    prints one contract line for the whole job (ranks sharing the B200:
    GS_BENCH_SHARED_GPU=1, gloo plumbing; the C2 step striped over the two
    ranks with peer loads through CUDA IPC; functional, not a timing)."""
    sys.path.insert(0, ROOT)
    import bench
    env = dict(os.environ, GS_BENCH_SHARED_GPU="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--workload", "c2",
                          "--steps", "5", "--warmup", "3", "--no-cpu", "--no-overhead", "--no-c3", "--no-c4"],
                         cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["metric"] == bench.METRIC and line["value"] > 0
    assert line["parity_ok"] is True and line["failures"] == []
    assert line["comm"]["nranks"] == 2 and line["config"] == bench.workload_config(bench.WORKLOADS["c2"], 2)
    assert line["gpu_launches"] > 0
