# compute-sanitizer over scripts/sanitize_case.py (one tool per run, summaries to gpurun_out/)
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_case.py > gpurun_out/san_$tool.log 2>&1
  echo "== $tool rc=$?"; tail -4 gpurun_out/san_$tool.log
done
