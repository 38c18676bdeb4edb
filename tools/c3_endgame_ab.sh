# C3 verified recovery: end-game hand-off A/B (GS_VERIFY_ENDGAME) x verification
# threads, with the per-claim trace; summary in gpurun_out/endgame_ab.log.
mkdir -p gpurun_out
# timeout 600 python -m pytest tests/test_gpu_fnv.py tests/test_checkpoint.py -q -m gpu > gpurun_out/eg_tests.log 2>&1; tail -1 gpurun_out/eg_tests.log
for i in 1 2 3; do for cfg in "0 14" "1 16" "1 15" "0 16"; do set -- $cfg
  GS_VERIFY_TRACE=1 GS_VERIFY_ENDGAME=$1 GS_VERIFY_THREADS=$2 timeout 300 python tools/c3_probe.py 1 > gpurun_out/eg_$1_$2_$i.out 2> gpurun_out/eg_$1_$2_$i.err
  python - "$1" "$2" "gpurun_out/eg_$1_$2_$i.out" >> gpurun_out/endgame_ab.log <<'PY'
import json, sys
for l in open(sys.argv[3]):
    if l.startswith("{"):
        d = json.loads(l)
        print("endgame", sys.argv[1], "threads", sys.argv[2], "wall", d["recover_wall_ms_runs"], "verify", [r["verify_ms"] for r in d["runs_detail"]],
              "decode", d["decode_device_ms"], "gpu/handed", [(r["split"]["chunks_gpu"], r["split"]["chunks_handed_over"]) for r in d["runs_detail"]], d["verified"], d["decoded_chunks"])
PY
done; done
cat gpurun_out/endgame_ab.log
