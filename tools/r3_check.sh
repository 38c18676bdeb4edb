make -s -C tests/cpp > gpurun_out/r3_make.log 2>&1
python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/r3_tests.log
python bench.py --workload c2 --steps 20 --warmup 5 --no-c3 --no-c4 --no-overhead > gpurun_out/r3_c2.json 2> gpurun_out/r3_c2.err
GS_BENCH_SHARED_GPU=1 timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu > gpurun_out/r3_n2.json 2> gpurun_out/r3_n2.err
echo done >> gpurun_out/r3_tests.log
