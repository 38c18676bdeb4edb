# C3 verified recovery: K2 per group of landed chunks vs one K2 after every upload,
# and the launch tables built before / after the upload enqueue (A/B, 2 x 3 recoveries each)
mkdir -p gpurun_out
: > gpurun_out/c3_k2_ab.log
for rep in 1 2 3; do
  for cfg in "1 1"; do
    set -- $cfg
    echo "== GS_RECOVER_K2_GROUPS=$1 GS_RECOVER_TABLES_FIRST=$2" >> gpurun_out/c3_k2_ab.log
    GS_RECOVER_K2_GROUPS=$1 GS_RECOVER_TABLES_FIRST=$2 timeout 600 python tools/c3_probe.py 1 >> gpurun_out/c3_k2_ab.log 2>&1
  done
done
python - <<'PY'
import json
mode=None
for line in open("gpurun_out/c3_k2_ab.log"):
    if line.startswith("=="): mode=line.strip(); continue
    if line.startswith("{"):
        d=json.loads(line)
        print(mode, d["recover_wall_ms_runs"], "decode", d["decode_device_ms"], "enq", d["enqueue_ms"], d["runs_detail"][0]["split"]["hosts_done_ms"], d["runs_detail"][0]["split"]["chunks_gpu"])
PY
