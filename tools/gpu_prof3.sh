timeout 300 ncu --set full --import-source on --clock-control none -k regex:spmm_kernel -s 1 -c 1 -o gpurun_out/prof_spmm python tools/prof_case.py spmm 4096 512 4096 8 0.9 8 8 2 > gpurun_out/ncu3.log 2>&1; echo ncu_rc=$?
tail -2 gpurun_out/ncu3.log
