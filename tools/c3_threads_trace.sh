# C3 verified recovery: verification thread-count A/B with the per-claim trace
# (GS_VERIFY_TRACE=1 -> gpurun_out/threads_<t>_<i>.err; summary in threads_ab.log).
mkdir -p gpurun_out
for i in 1 2; do for t in 14 16 15; do
  GS_VERIFY_TRACE=1 GS_VERIFY_THREADS=$t timeout 300 python tools/c3_probe.py 1 > gpurun_out/threads_${t}_$i.out 2> gpurun_out/threads_${t}_$i.err
  python - "$t" "gpurun_out/threads_${t}_$i.out" >> gpurun_out/threads_ab.log <<'PY'
import json, sys
for l in open(sys.argv[2]):
    if l.startswith("{"):
        d = json.loads(l)
        print("threads", sys.argv[1], "wall", d["recover_wall_ms_runs"], "decode", d["decode_device_ms"],
              [r["split"] for r in d["runs_detail"]][-1], d["verified"], d["decoded_chunks"])
PY
done; done
cat gpurun_out/threads_ab.log
