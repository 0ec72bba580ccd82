# Step traces of the in-tree library and of build/variants/<name> libraries: fold timing per split tile
for v in base "$@"; do
  if [ $v = base ]; then L=paper_2603_13281_b200/libicarus_b200.so; else L=build/variants/$v/libicarus_b200.so; fi
  ICR_LIB_PATH=$L timeout 300 python tools/trace_step.py gpurun_out/trace_$v.csv > gpurun_out/trace_$v.log 2>&1; tail -3 gpurun_out/trace_$v.log
  echo "== $v"; python tools/trace_fold.py gpurun_out/trace_$v.csv
  rm -f gpurun_out/trace_$v.csv
done
