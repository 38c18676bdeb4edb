mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
c=d['recovery']['c3_orchestrated']; print('value',d['value'],'recovery_ms',d['recovery_ms'], 'frac', d['roofline']['frac'], d['roofline']['traffic_source'])
print({k:c.get(k) for k in ['plan','decode_device_ms','recover_wall_ms','verify_host_ms','verify_gpu_chunks','verify_split','verified','decoded_chunks']})
print(c.get('runs_ms'), d['recovery'].get('c3_orchestrated_runs_ms'))
"
