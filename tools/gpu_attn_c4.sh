# C4 attention (cold device span and pipelined), repeated N times: bash tools/gpu_attn_c4.sh 1 2 3
for v in "$@"; do
  for mode in "" "--pipelined"; do
    timeout 300 python tools/attn_sweep.py --ctx 32768 --adapters 8 --chunk-pages 128 $mode 2>/dev/null | tail -1 > gpurun_out/apf.json
    python -c "import json; d=json.load(open('gpurun_out/apf.json')); print('run', d['mode'], 'ms', round(d['ms']*1e3,2), 'us', 'span', d.get('kernel_span_us'), 'frac_span', round(d['unique_kv_bytes']/d.get('kernel_span_us',1e9)/1e3/6540.5,3) if d.get('kernel_span_us') else '', 'frac_ev', round(d['gbs']/6540.5,3))"
  done
done
