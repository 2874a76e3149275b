# round 2 run c: full gpu suite + replay with one-call re-shard
python -m pytest tests -m gpu -x -q -s 2>&1 | grep -E "measured|wall-clock|relL2 z|passed|failed|Error|error|assert" | tail -40 > gpurun_out/r2c_tests.log
timeout 900 python scripts/trace_replay.py --rates 0.5,1.0 --real-rates 0.5,1.0 --out gpurun_out/r2c_trace_replay.json > gpurun_out/r2c_trace.log 2>&1
tail -3 gpurun_out/r2c_trace.log
cat gpurun_out/r2c_tests.log
