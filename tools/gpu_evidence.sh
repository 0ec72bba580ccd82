# Round evidence on one B200: full bench line, ncu launch list of one decode step, ncu --set full of
# the gate|up GEMM (in the step) and of the C4 attention launch, SASS opcode counts.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_full.json
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv python tools/profile_step.py step > gpurun_out/ncu_step.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:ILi16ELi3E -s 5 -c 1 -o gpurun_out/gemm_gu python tools/profile_step.py step > gpurun_out/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 1 -c 1 -o gpurun_out/attn_tc_c4 python tools/attn_sweep.py --ctx 32768 --adapters 8 --chunk-pages 128 > gpurun_out/ncu_attn.log 2>&1
tail -n 2 gpurun_out/ncu_step.log gpurun_out/ncu_gemm.log gpurun_out/ncu_attn.log
