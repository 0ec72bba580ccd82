set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py 2>&1 | tail -3 | tee gpurun_out/bench_r01a.json
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv python tools/profile_step.py step > gpurun_out/ncu_step.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm -c 1 -o gpurun_out/gemm_gu python tools/profile_step.py gemm > gpurun_out/ncu_gemm.log 2>&1
tail -3 gpurun_out/ncu_step.log gpurun_out/ncu_gemm.log
