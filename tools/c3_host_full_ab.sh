mkdir -p gpurun_out
for mode in 1 0 1 0; do
  echo "== GS_VERIFY_HOST_FULL=$mode" >> gpurun_out/c3ab.log
  GS_VERIFY_HOST_FULL=$mode timeout 600 python tools/c3_probe.py 1 >> gpurun_out/c3ab.log 2>&1
done
timeout 900 python -m pytest tests/test_checkpoint.py tests/test_gpu_fnv.py -q -m gpu > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
tail -2 gpurun_out/ab_tests.log
python - <<'PY'
import json
mode=None
for line in open("gpurun_out/c3ab.log"):
    if line.startswith("=="): mode=line.strip(); continue
    if line.startswith("{"):
        d=json.loads(line)
        print(mode, d["recover_wall_ms_runs"], d["decode_device_ms"], [r["split"] for r in d["runs_detail"]][:1], d["verified"], d["decoded_chunks"])
PY
