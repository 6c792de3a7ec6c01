mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemm -o gpurun_out/ncu_pair python tools/ncu_pair.py ffn_down qkv > gpurun_out/ncu_pair.log 2>&1; echo ncu rc $?
timeout 600 python -m pytest tests/test_gpu_intercept.py -q > gpurun_out/intercept.log 2>&1; tail -2 gpurun_out/intercept.log
