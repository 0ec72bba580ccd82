# attention-focused iteration: kernel tests, C4 trace, C4 cold/pipelined, C2 bench
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python tools/attn_trace.py > gpurun_out/attn_trace.txt 2>&1; head -16 gpurun_out/attn_trace.txt
bash tools/gpu_attn_c4.sh 1 2 3
timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 128 2>&1 | tail -1 > gpurun_out/bench_iter.json
python -c "import json; d=json.load(open('gpurun_out/bench_iter.json')); print('tok/s', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'])"
