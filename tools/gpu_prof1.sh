timeout 300 ncu --set full --clock-control none --import-source on -k regex:sddmm_tc -s 1 -c 1 -o gpurun_out/prof_sddmm_tc python tools/prof_case.py sddmm 0.5 dense 2 > gpurun_out/ncu1.log 2>&1; echo ncu_rc=$?
tail -5 gpurun_out/ncu1.log
