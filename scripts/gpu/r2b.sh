# round 2 run b: new step / boundary / executor tests + config-5 replay with pooled groups
python -m pytest tests/test_step_gpu.py tests/test_boundary_gpu.py tests/test_executor_gpu.py -m gpu -x -q -s 2>&1 | grep -E "measured|relL2|passed|failed|Error|error|assert" | tail -40 > gpurun_out/r2b_tests.log
timeout 900 python scripts/trace_replay.py --rates 0.5,1.0 --real-rates 0.5,1.0 --out gpurun_out/r2b_trace_replay.json > gpurun_out/r2b_trace.log 2>&1
tail -5 gpurun_out/r2b_trace.log
cat gpurun_out/r2b_tests.log
