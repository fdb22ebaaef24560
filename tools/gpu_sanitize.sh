# compute-sanitizer over small runs of every solver (tools/sanitize_run.py)
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"; timeout 900 $CS --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/san_$tool.log 2>&1; echo "exit $?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|error" gpurun_out/san_$tool.log | head -6
done
