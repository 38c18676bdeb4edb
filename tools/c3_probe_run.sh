timeout 900 python -m pytest tests/test_checkpoint.py tests/test_gpu_fnv.py -q -m gpu > gpurun_out/ck_tests.log 2>&1; tail -1 gpurun_out/ck_tests.log
python tools/c3_probe.py 3 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['recover_wall_ms_runs'], d['decode_device_ms'], d['enqueue_ms'], d['runs_detail'][0]['split'], d['verified'], d['decoded_chunks'])
"
