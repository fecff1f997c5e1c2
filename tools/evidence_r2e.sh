set -x
python tools/ncu_target.py 4 8192 8192 8192 2 > /dev/null && ncu --set full --clock-control none --import-source on -k regex:simt_mm_kernel -s 1 -c 1 -o gpurun_out/r2_minplus_tma python tools/ncu_target.py 4 8192 8192 8192 2 > gpurun_out/r2e_ncu1.log 2>&1
python tools/ncu_target.py 5 16384 16384 16384 1 > /dev/null && ncu --set full --clock-control none -k regex:simt_mm_kernel -s 0 -c 1 -o gpurun_out/r2_maxplus_tma python tools/ncu_target.py 5 16384 16384 16384 1 > gpurun_out/r2e_ncu2.log 2>&1
ls -la gpurun_out | grep tma
