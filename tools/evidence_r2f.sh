set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/r2f_bench.log 2>&1; echo RC=$? >> gpurun_out/r2f_bench.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2f_bench_small.log 2>&1 && \
  timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2f_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2f_ncu_launch.log 2>&1
ls -la gpurun_out | grep r2f
