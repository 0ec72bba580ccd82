# same-box A/B of the C2 decode step only: in-tree library vs build/variants/$1
for rep in 1 2 3; do
  for v in base $1; do
    if [ $v = base ]; then L=paper_2603_13281_b200/libicarus_b200.so; else L=build/variants/$v/libicarus_b200.so; fi
    echo "$v $(ICR_LIB_PATH=$L timeout 300 python tools/step_time.py 3 2>&1 | tail -1)"
  done
done
