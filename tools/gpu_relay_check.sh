# N>1 verified recovery (checksum relay) on one B200: the striping GPU tests and
# the bench with 2 and 4 ranks sharing the GPU (functional; timings shared-GPU).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_peer_striping.py -q > gpurun_out/striping_tests.log 2>&1; echo "rc=$?" >> gpurun_out/striping_tests.log
for n in 2 4 8; do
  GS_BENCH_SHARED_GPU=1 timeout 1200 python bench.py --gpus $n --steps 5 --warmup 3 --no-cpu --no-overhead > gpurun_out/bench_n${n}_shared.json 2> gpurun_out/bench_n${n}_shared.err
done
grep -q "rc=0" gpurun_out/striping_tests.log && tail -2 gpurun_out/striping_tests.log || tail -60 gpurun_out/striping_tests.log
for n in 2 4 8; do tail -1 gpurun_out/bench_n${n}_shared.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['recovery']
print($n, d['value'], d.get('recovery_ms'), d.get('failures'), {k:v for k,v in r.items() if k.startswith('c3_') and k not in ('c3_mode','c3_verify')})"; tail -3 gpurun_out/bench_n${n}_shared.err; done
