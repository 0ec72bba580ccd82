timeout 600 python tools/profile_variants.py 2>&1 | tail -6
for w in 0 1 2; do timeout 300 python tools/trace_gemm.py $w 2>&1 | tail -7; cp gpurun_out/gemm_trace.csv gpurun_out/gemm_trace_$w.csv; done
