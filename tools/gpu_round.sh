# Round-end evidence run on one B200 (tests, smoke, bench, ncu launch list + full captures).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench.json
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv python tools/profile_step.py step > gpurun_out/ncu_step.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm -c 1 -o gpurun_out/gemm_gu python tools/profile_step.py gemm > gpurun_out/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 1 -c 1 -o gpurun_out/attn_tc_c4 python tools/attn_sweep.py --ctx 32768 --adapters 8 --chunk-pages 128 > gpurun_out/ncu_attn.log 2>&1
tail -n 3 gpurun_out/ncu_step.log gpurun_out/ncu_gemm.log gpurun_out/ncu_attn.log
timeout 600 python tools/attn_sweep.py --out gpurun_out/attn_sweep_auto.json > /dev/null 2>&1
timeout 300 python tools/attn_sweep.py --ctx 32768 --adapters 8 --chunk-pages 128 --pipelined > gpurun_out/attn_c4_pipelined.json 2>&1
timeout 900 python tools/c3_workflow.py --out gpurun_out/c3.json > gpurun_out/c3.log 2>&1; tail -2 gpurun_out/c3.log
