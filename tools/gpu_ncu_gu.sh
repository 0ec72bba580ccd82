timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:ILi16ELi3E -s 5 -c 1 -o gpurun_out/gu_src python tools/profile_step.py step > gpurun_out/ncu_gu.log 2>&1
tail -3 gpurun_out/ncu_gu.log
