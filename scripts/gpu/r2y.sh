# HEAD evidence refresh: boundary test with the unmodified ditsim (baseline/_ref), 240p step launch list,
# ncu --set full of one block pair's kernels
set -x
timeout 900 python -m pytest tests/test_boundary_gpu.py -m gpu -q -rs > gpurun_out/r2y_boundary.log 2>&1; echo "boundary rc=$?"
tail -3 gpurun_out/r2y_boundary.log
K='regex:gemm|fmha|ln_mod|temporal|final_layer|patch_embed|gemv|modulation|timestep'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 700 -c 569 --csv --log-file gpurun_out/launches_r02h.csv python scripts/profile_step.py 240p 3 > /dev/null 2>&1; echo "launches rc=$?"
K2='regex:gemm|fmha|ln_mod|temporal'
timeout 1200 ncu --set full --clock-control none --import-source on -k "$K2" -s 600 -c 12 -o gpurun_out/block_r02h python scripts/profile_step.py 240p 2 > gpurun_out/r2y_ncu.log 2>&1; echo "ncu rc=$?"
