# Iteration run: GPU tests (optional: SKIP_TESTS=1), step trace phases, C2 bench line
if [ -z "$SKIP_TESTS" ]; then timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4; fi
timeout 300 python tools/trace_step.py gpurun_out/trace.csv > gpurun_out/trace.txt 2>&1
python tools/trace_phases.py gpurun_out/trace.csv x > gpurun_out/phases.txt 2>&1; cat gpurun_out/phases.txt | grep -v Warn
gzip -f gpurun_out/trace.csv
timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 128 2>&1 | tail -1 > gpurun_out/bench_iter.json
python -c "import json; d=json.load(open('gpurun_out/bench_iter.json')); print('tok/s', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'])"
