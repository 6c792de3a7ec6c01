mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm_pair.py tests/test_gpu_c4.py tests/test_gpu_gpt2.py tests/test_gpu_gemm.py -q -x > gpurun_out/fuse_tests.log 2>&1; echo tests rc $?; tail -3 gpurun_out/fuse_tests.log
timeout 300 python tools/step_time.py --config c4 > gpurun_out/step_time.log 2>&1; timeout 300 python tools/step_time.py --config c3 >> gpurun_out/step_time.log 2>&1
timeout 600 python tools/ptb_overhead.py --config c4 --chosen --out gpurun_out/ptb_overhead_c4.json > /dev/null 2>&1; echo ptbo $?
