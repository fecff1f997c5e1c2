set -x
python -m pytest tests -m gpu -q > gpurun_out/r2_pytest.log 2>&1; echo RC=$? >> gpurun_out/r2_pytest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.log 2>&1; echo RC=$? >> gpurun_out/r2_bench.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2_bench_small.log 2>&1 && \
  timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2_ncu_launch.log 2>&1
python tools/ncu_target.py 4 8192 8192 8192 2 > /dev/null && ncu --set full --clock-control none --import-source on -k regex:simt_mm_kernel -s 1 -c 1 -o gpurun_out/r2_minplus python tools/ncu_target.py 4 8192 8192 8192 2 > gpurun_out/r2_ncu1.log 2>&1
python tools/ncu_target.py 5 16384 16384 16384 1 > /dev/null && ncu --set full --clock-control none -k regex:simt_mm_kernel -s 0 -c 1 -o gpurun_out/r2_maxplus python tools/ncu_target.py 5 16384 16384 16384 1 > gpurun_out/r2_ncu2.log 2>&1
python tools/ncu_target.py 7 65536 1024 256 3 > /dev/null && ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -s 2 -c 1 -o gpurun_out/r2_bf16 python tools/ncu_target.py 7 65536 1024 256 3 > gpurun_out/r2_ncu3.log 2>&1
python tools/fused_one.py 8192 split > /dev/null && ncu --set full --clock-control none -k regex:tc_gemm_kernel -s 1 -c 1 -o gpurun_out/r2_tf32x3 python tools/fused_one.py 8192 split > gpurun_out/r2_ncu4.log 2>&1
ls -la gpurun_out
