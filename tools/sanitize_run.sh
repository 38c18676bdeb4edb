# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_smoke.py
# (every kernel family, the verification splits, the relay's GPU worker) and
# memcheck over the C++ drop-in consumers; log -> gpurun_out/sanitizer.txt
mkdir -p gpurun_out
out=gpurun_out/sanitizer.txt
: > $out
for tool in memcheck racecheck synccheck; do
  echo "== compute-sanitizer --tool $tool python tools/sanitize_smoke.py" >> $out
  GS_JIT=1 timeout 1200 compute-sanitizer --tool $tool python tools/sanitize_smoke.py 2>&1 | grep -E "COMPUTE-SANITIZER|sanitize_smoke|SUMMARY|Error|error" | head -20 >> $out
done
echo >> $out
echo "== compute-sanitizer --tool memcheck on the C++ drop-in consumers (LD_LIBRARY_PATH=paper_2605_00831_b200/_lib)" >> $out
for b in tests/cpp/facade_test oracle/_ref/ref_coding_test_b200 oracle/_ref/ref_recovery_test_b200; do
  echo "-- $b" >> $out
  LD_LIBRARY_PATH=paper_2605_00831_b200/_lib timeout 900 compute-sanitizer --tool memcheck $b 2>&1 | grep -E "tests,|SUMMARY" | tail -3 >> $out
done
cat $out
