# same-box A/B/C: in-tree library vs build/variants/$1 and $2 (C2 step, C3-regime step, 2k prefill)
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
for rep in 1 2; do
  for v in base $1 $2; do
    if [ $v = base ]; then L=paper_2603_13281_b200/libicarus_b200.so; else L=build/variants/$v/libicarus_b200.so; fi
    c2=$(ICR_LIB_PATH=$L timeout 300 python tools/step_time.py 3 2>&1 | tail -1 | grep -o "min [0-9.]*")
    c3=$(ICR_LIB_PATH=$L timeout 500 python tools/c3_step_profile.py 2>&1 | grep marginal | grep -o "'full_step_ms': [0-9.]*")
    pf=$(ICR_LIB_PATH=$L timeout 300 python tools/prefill_profile.py 2>&1 | grep -o "prefill 2048 tokens: [0-9.]* ms")
    echo "$v | C2 $c2 | C3 $c3 | $pf"
  done
done
