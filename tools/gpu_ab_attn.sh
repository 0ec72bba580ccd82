# A/B of the C4 attention span: in-tree library vs build/variants/$1, interleaved, N reps
for rep in 1 2 3 4; do
  for v in base $1; do
    if [ $v = base ]; then L=paper_2603_13281_b200/libicarus_b200.so; else L=build/variants/$v/libicarus_b200.so; fi
    ICR_LIB_PATH=$L timeout 300 python tools/attn_sweep.py --ctx 32768 --adapters 8 --chunk-pages 128 2>/dev/null | tail -1 > gpurun_out/ab.json
    python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$v', 'span', round(d['kernel_span_us'],2), 'frac', round(d['unique_kv_bytes']/d['kernel_span_us']/1e3/6540.5,3))"
  done
done
