# HEAD evidence: config-5 trace replay (profile best of 5), config 4, reference arm
set -x
timeout 2400 python scripts/trace_replay.py --out gpurun_out/r2z_trace_replay_c5.json > gpurun_out/r2z_trace_replay.log 2>&1; echo "replay rc=$?"
timeout 900 python scripts/config4.py --out gpurun_out/r2z_config4.json > gpurun_out/r2z_config4.log 2>&1; echo "config4 rc=$?"
timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2z_reference_arm.log 2>&1; echo "ref rc=$?"
grep -E "B values|predicted|replayed" gpurun_out/r2z_trace_replay.log | cut -c1-200; tail -c 800 gpurun_out/r2z_reference_arm.log
