# One decode-step per-CTA trace (kept as CSV) + phase summary
timeout 300 python tools/trace_step.py gpurun_out/trace.csv > gpurun_out/trace.txt 2>&1
python tools/trace_phases.py gpurun_out/trace.csv > gpurun_out/phases.txt 2>&1
gzip -f gpurun_out/trace.csv
