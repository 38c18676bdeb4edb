# Closing confirmation on one B200: GPU suite, smoke, and the three bench
# lines the driver records (default C3, reference arm, C2).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --workload c2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
tail -2 gpurun_out/gpu_tests.log; tail -1 gpurun_out/smoke.log
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
r = json.loads(open("gpurun_out/bench_ref.json").read().strip().splitlines()[-1])
c = json.loads(open("gpurun_out/bench_c2.json").read().strip().splitlines()[-1])
o = d["recovery"]["c3_orchestrated"]
print("C3", d["value"], "recovery", d["recovery_ms"], o["plan"]["mode"], o["decoded_chunks"], "K1", d["roofline"]["frac"],
      "traffic", d["roofline"]["traffic"], "e2e", d["e2e"]["value"], "overhead", d["decode_overhead"]["overhead_pct_of_decode_step"],
      "ok", d["parity_ok"], "launches", d["gpu_launches"], "clocks", d["clocks"])
print("REF", r["value"], r["recovery_ms"], "same config", r["config"] == d["config"])
print("C2", c["value"], c["roofline"]["frac"], c["parity_ok"])
PY
