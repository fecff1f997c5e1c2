set -x
for c in 2 3 4 5; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --cfg $c --steps 2 --warmup 3 > gpurun_out/r2k_torchrun_cfg$c.log 2>&1; echo RC=$? >> gpurun_out/r2k_torchrun_cfg$c.log
done
python -m pytest tests -m gpu -q > gpurun_out/r2k_pytest.log 2>&1; echo RC=$? >> gpurun_out/r2k_pytest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2k_bench.log 2>&1; echo RC=$? >> gpurun_out/r2k_bench.log
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2k_ref.log 2>&1; echo RC=$? >> gpurun_out/r2k_ref.log
python tools/strassen_profile.py 16384 > gpurun_out/r2k_sp.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2k_strassen_launches.csv python tools/strassen_profile.py 16384 > gpurun_out/r2k_ncu_sp.log 2>&1
python tools/fused_one.py 8192 b3n > /dev/null && timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_pair_kernel -s 1 -c 1 -o gpurun_out/r2_bf16x3n python tools/fused_one.py 8192 b3n > gpurun_out/r2k_ncu_b3n.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2k_bench_small.log 2>&1 && \
  timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2k_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2k_ncu_launch.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k_smoke.log 2>&1; echo RC=$? >> gpurun_out/r2k_smoke.log
ls -la gpurun_out | grep r2k
