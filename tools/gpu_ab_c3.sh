# A/B of the C3-regime step and the C2 step: in-tree library vs build/variants/$1, interleaved
for rep in 1 2; do
  for v in base $1; do
    if [ $v = base ]; then L=paper_2603_13281_b200/libicarus_b200.so; else L=build/variants/$v/libicarus_b200.so; fi
    echo "== $v"; ICR_LIB_PATH=$L timeout 500 python tools/c3_step_profile.py 2>&1 | grep marginal | cut -c1-60
    ICR_LIB_PATH=$L timeout 300 python tools/prefill_profile.py 2>&1 | grep "prefill 2048"
  done
done
