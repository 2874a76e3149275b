# config-5 trace replay with the split re-shard timing fields; executor GPU tests
set -x
timeout 900 python -m pytest tests/test_executor_gpu.py -m gpu -q -x > gpurun_out/r2w_executor_tests.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/r2w_executor_tests.log
timeout 2400 python scripts/trace_replay.py --out gpurun_out/r2w_trace_replay_c5.json > gpurun_out/r2w_trace_replay.log 2>&1; echo "replay rc=$?"
grep -E "B values|predicted|replayed" gpurun_out/r2w_trace_replay.log | cut -c1-400
