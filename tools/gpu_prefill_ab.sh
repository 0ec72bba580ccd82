# GPU tests, then prefill + C2 step A/B against build/variants/$1
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for v in base $1; do
  if [ $v = base ]; then L=paper_2603_13281_b200/libicarus_b200.so; else L=build/variants/$v/libicarus_b200.so; fi
  echo "== $v"
  ICR_LIB_PATH=$L timeout 300 python tools/prefill_profile.py 2>&1 | tail -2 | cut -c1-220
  echo "$(ICR_LIB_PATH=$L timeout 300 python tools/step_time.py 3 2>&1 | tail -1)"
done
