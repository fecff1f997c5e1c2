set -x
python -m pytest tests -m gpu -q > gpurun_out/r2d_pytest.log 2>&1; echo RC=$? >> gpurun_out/r2d_pytest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2d_bench.log 2>&1; echo RC=$? >> gpurun_out/r2d_bench.log
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2d_ref.log 2>&1; echo RC=$? >> gpurun_out/r2d_ref.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2d_bench_small.log 2>&1 && \
  timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2d_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2d_ncu_launch.log 2>&1
python tools/strassen_profile.py > /dev/null && ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d_strassen_launches.csv python tools/strassen_profile.py > gpurun_out/r2d_ncu8.log 2>&1
ls -la gpurun_out
