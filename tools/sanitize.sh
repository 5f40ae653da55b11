# compute-sanitizer over tools/sanitize_cases.py (run under gpurun); summaries -> gpurun_out/sanitize_*.txt
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitize_summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|worst parity" gpurun_out/sanitize_$tool.txt >> gpurun_out/sanitize_summary.txt
done
