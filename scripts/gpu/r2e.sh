# round 2 run e (after container restore): full gpu suite, bench N=1/2, reference arm, sanitizers, fmha timelines
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -q -s 2>&1 | grep -E "measured|wall-clock|relL2|diff|passed|failed|Error|error|assert" | tail -120 > gpurun_out/r2e_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2e_bench.log 2>&1
timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2e_bench2.log 2>&1
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r2e_ref.log 2>&1
for m in cross spatial 720; do DDIT_LIB=paper_2506_13497_b200/libddit_fmtrace.so timeout 300 python scripts/fmha_trace.py $m > gpurun_out/fmtrace_$m.log 2>&1; done
for tool in memcheck synccheck initcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_case.py > gpurun_out/san_$tool.log 2>&1
  echo "== $tool rc=$?" >> gpurun_out/san_summary.log; tail -4 gpurun_out/san_$tool.log >> gpurun_out/san_summary.log
done
tail -3 gpurun_out/r2e_*.log
