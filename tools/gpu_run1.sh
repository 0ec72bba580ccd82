nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench.json
timeout 300 python tools/trace_step.py gpurun_out/trace.csv > gpurun_out/trace.txt 2>&1
rm -f gpurun_out/trace.csv
