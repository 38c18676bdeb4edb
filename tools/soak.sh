# Seeded fuzz loops at 20x (GS_FUZZ_SCALE) on one B200; log -> gpurun_out/soak.txt
mkdir -p gpurun_out
out=gpurun_out/soak.txt
: > $out
echo "GS_FUZZ_SCALE=20 python -m pytest tests -m gpu -k fuzz (one B200): orchestration, pipelines, GPU FNV chains, paged geometries, the N>1 checksum relay on the GPUs" >> $out
GS_FUZZ_SCALE=20 timeout 2400 python -m pytest tests -q -m gpu -k fuzz 2>&1 | tail -1 >> $out
echo "GS_FUZZ_SCALE=20 -k random_schemes_on_the_gpu" >> $out
GS_FUZZ_SCALE=20 timeout 900 python -m pytest tests -q -m gpu -k random_schemes_on_the_gpu 2>&1 | tail -1 >> $out
echo "GS_FUZZ_SCALE=20 CPU: striped partition fuzz, random schemes vs the reference decode planner, checksum relay fuzz (3 ranks)" >> $out
GS_FUZZ_SCALE=20 timeout 1200 python -m pytest tests -q -m "not gpu" -k "fuzz or random" 2>&1 | tail -1 >> $out
cat $out
