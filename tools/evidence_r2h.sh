set -x
python tools/tc_trace2.py > gpurun_out/r2h_trace2.log 2>&1
python -m pytest tests -m gpu -q > gpurun_out/r2h_pytest.log 2>&1; echo RC=$? >> gpurun_out/r2h_pytest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2h_bench.log 2>&1; echo RC=$? >> gpurun_out/r2h_bench.log
python tools/fused_one.py 8192 b3 > /dev/null && timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_pair_kernel -s 1 -c 1 -o gpurun_out/r2_bf16x3 python tools/fused_one.py 8192 b3 > gpurun_out/r2h_ncu_b3.log 2>&1
python tools/strassen_profile.py 16384 > gpurun_out/r2h_sp.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2h_strassen_launches.csv python tools/strassen_profile.py 16384 > gpurun_out/r2h_ncu_sp.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2h_bench_small.log 2>&1 && \
  timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2h_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2h_ncu_launch.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.log 2>&1; echo RC=$? >> gpurun_out/r2h_smoke.log
ls -la gpurun_out | grep r2h
