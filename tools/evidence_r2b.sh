set -x
python tools/fused_one.py 8192 split > /dev/null && ncu --set full --clock-control none --import-source on -k regex:tc_pair_kernel -s 1 -c 1 -o gpurun_out/r2_tf32x3_pair python tools/fused_one.py 8192 split > gpurun_out/r2_ncu5.log 2>&1
python -m pytest tests/test_gpu_tf32_fused.py tests/test_gpu_strassen.py tests/test_gpu_distributed_strassen.py -q > gpurun_out/r2_pytest_pair.log 2>&1; echo RC=$? >> gpurun_out/r2_pytest_pair.log
python tools/strassen_profile.py > gpurun_out/r2_strassen_prof.log 2>&1 && ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_strassen_launches.csv python tools/strassen_profile.py > gpurun_out/r2_ncu6.log 2>&1
