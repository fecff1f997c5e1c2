# cfg3 kernel change check: bf16 correctness tests, graph/eager timing, back-to-back trace
timeout 900 python -m pytest tests/test_gpu_mm.py tests/test_gpu_fullsize.py tests/test_gpu_graph.py tests/test_gpu_guard.py tests/test_gpu_pdl.py tests/test_gpu_fuzz.py -q -x -k "bf16 or tc or graph or pdl or guard or fuzz or cfg3" > gpurun_out/c3_pytest.log 2>&1; echo RC=$? >> gpurun_out/c3_pytest.log
for i in 1 2 3; do python tools/tc_graph_vs_eager.py; done > gpurun_out/c3_time.log 2>&1
python tools/tc_trace2.py > gpurun_out/c3_trace.log 2>&1
