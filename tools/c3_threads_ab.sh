# C3 verified recovery vs the number of host verification threads (A/B/A/B)
mkdir -p gpurun_out
: > gpurun_out/c3_threads.log
for t in 14 16 15 14 16 15; do
  echo "== GS_VERIFY_THREADS=$t" >> gpurun_out/c3_threads.log
  GS_VERIFY_THREADS=$t timeout 600 python tools/c3_probe.py 1 >> gpurun_out/c3_threads.log 2>&1
done
python - <<'PY'
import json
mode=None
for line in open("gpurun_out/c3_threads.log"):
    if line.startswith("=="): mode=line.strip(); continue
    if line.startswith("{"):
        d=json.loads(line)
        print(mode, d["recover_wall_ms_runs"], d["decode_device_ms"], d["runs_detail"][0]["split"])
PY
