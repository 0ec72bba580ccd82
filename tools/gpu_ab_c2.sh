# A/B of the C2 decode step: in-tree library vs build/variants/$1, interleaved (GPU tests first)
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
for rep in 1 2 3; do
  for v in base $1; do
    if [ $v = base ]; then L=paper_2603_13281_b200/libicarus_b200.so; else L=build/variants/$v/libicarus_b200.so; fi
    echo "$v $(ICR_LIB_PATH=$L timeout 300 python tools/step_time.py 3 2>&1 | tail -1)"
  done
done
