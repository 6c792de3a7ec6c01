mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_gemm_pair.py tests/test_gpu_c4.py tests/test_gpu_gpt2.py -q -x > gpurun_out/f32_tests.log 2>&1; echo tests rc $?; tail -2 gpurun_out/f32_tests.log
timeout 600 python tools/ptb_overhead.py --config c4 --chosen --out gpurun_out/ptb_overhead_c4.json > gpurun_out/ptb_overhead_c4.log 2>&1; echo ptbo rc $?
timeout 600 python tools/gemm_pair_bench.py > gpurun_out/pair_bench.log 2>&1; echo pb rc $?
