set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/r2c_bench.log 2>&1; echo RC=$? >> gpurun_out/r2c_bench.log
python tools/fused_one.py 8192 raw > /dev/null && ncu --set full --clock-control none --import-source on -k regex:tc_pair_kernel -s 1 -c 1 -o gpurun_out/r2_tf32b2_raw python tools/fused_one.py 8192 raw > gpurun_out/r2_ncu7.log 2>&1
python tools/strassen_profile.py > /dev/null && ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c_strassen_launches.csv python tools/strassen_profile.py > gpurun_out/r2_ncu8.log 2>&1
