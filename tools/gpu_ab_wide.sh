# A/B of the in-tree library vs build/variants/$1 on prefill and C3
for v in base $1; do
  if [ $v = base ]; then L=paper_2603_13281_b200/libicarus_b200.so; else L=build/variants/$v/libicarus_b200.so; fi
  echo "== $v"
  ICR_LIB_PATH=$L timeout 300 python tools/prefill_profile.py 2>&1 | tail -2 | cut -c1-200
  ICR_LIB_PATH=$L timeout 900 python tools/c3_workflow.py --out gpurun_out/c3_$v.json > gpurun_out/c3_$v.log 2>&1; python -c "import json; d=json.load(open('gpurun_out/c3_$v.json')); print('C3 tok/s', d['decode_tok_s'], 'p95', d['p95_request_latency_ms'])"
done
