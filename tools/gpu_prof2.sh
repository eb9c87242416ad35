timeout 300 ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none -k regex:sddmm_tc -s 2 -c 1 -o gpurun_out/prof_sddmm_tc2 python tools/prof_case.py sddmm 0.5 dense 3 > gpurun_out/ncu2.log 2>&1; echo ncu_rc=$?
tail -2 gpurun_out/ncu2.log
