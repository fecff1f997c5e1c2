set -x
python -m pytest tests -m gpu -q > gpurun_out/r2g_pytest.log 2>&1; echo RC=$? >> gpurun_out/r2g_pytest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2g_bench.log 2>&1; echo RC=$? >> gpurun_out/r2g_bench.log
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2g_ref.log 2>&1; echo RC=$? >> gpurun_out/r2g_ref.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2g_bench_small.log 2>&1 && \
  timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2g_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2g_ncu_launch.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; echo RC=$? >> gpurun_out/r2g_smoke.log
ls -la gpurun_out | grep r2g
