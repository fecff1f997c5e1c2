set -x
timeout 600 python -m pytest tests/test_gpu_bf16x3.py -x -q > gpurun_out/b3_pytest.log 2>&1; echo RC=$? >> gpurun_out/b3_pytest.log
timeout 600 python tools/cfg5_variants.py > gpurun_out/b3_variants.log 2>&1; echo RC=$? >> gpurun_out/b3_variants.log
