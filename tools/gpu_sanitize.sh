# compute-sanitizer over tools/sanitize_workload.py; summaries into gpurun_out/
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
    python tools/sanitize_workload.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|error" gpurun_out/sanitize_$tool.log | tail -5 | tee -a gpurun_out/sanitize_summary.txt
done
