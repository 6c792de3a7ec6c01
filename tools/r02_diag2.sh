mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_scheduler.py tests/test_gpu_irjit.py -q > gpurun_out/t_sched.log 2>&1; tail -2 gpurun_out/t_sched.log
timeout 600 python tools/c2_diag.py --ms 2000 --load 0.5 --burst 20 > gpurun_out/c2_diag.json 2> gpurun_out/c2_diag.err; echo diag $?
