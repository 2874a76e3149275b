set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/test_parity_configs_gpu.py tests/test_attention_gpu.py -m gpu -x -q -s 2>&1 | grep -E "relL2|diff|passed|failed|Error|error" | tail -80 > gpurun_out/r2a_parity.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2a_bench.log 2>&1
timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_bench2.log 2>&1
tail -3 gpurun_out/*.log
