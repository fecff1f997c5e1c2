set -x
python -m pytest tests -m gpu -q > gpurun_out/r2j_pytest.log 2>&1; echo RC=$? >> gpurun_out/r2j_pytest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2j_bench.log 2>&1; echo RC=$? >> gpurun_out/r2j_bench.log
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2j_ref.log 2>&1; echo RC=$? >> gpurun_out/r2j_ref.log
python tools/strassen_profile.py 16384 > gpurun_out/r2j_sp.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2j_strassen_launches.csv python tools/strassen_profile.py 16384 > gpurun_out/r2j_ncu_sp.log 2>&1
python tools/fused_one.py 8192 b3n > /dev/null && timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_pair_kernel -s 1 -c 1 -o gpurun_out/r2_bf16x3n python tools/fused_one.py 8192 b3n > gpurun_out/r2j_ncu_b3n.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2j_bench_small.log 2>&1 && \
  timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2j_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2j_ncu_launch.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2j_smoke.log 2>&1; echo RC=$? >> gpurun_out/r2j_smoke.log
ls -la gpurun_out | grep r2j
