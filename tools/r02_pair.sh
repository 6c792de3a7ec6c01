mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm_pair.py tests/test_gpu_gemm.py -q -x > gpurun_out/pair_tests.log 2>&1; echo pair rc $?; tail -3 gpurun_out/pair_tests.log
timeout 600 python tools/gemm_pair_bench.py > gpurun_out/pair_bench.log 2>&1; echo bench rc $?
timeout 2400 python -m pytest tests/ -m gpu -q > gpurun_out/gputests.log 2>&1; tail -5 gpurun_out/gputests.log
