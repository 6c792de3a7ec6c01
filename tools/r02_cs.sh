mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gpt2.py tests/test_gpu_c4.py tests/test_gpu_resnet.py -q -x > gpurun_out/cs_tests.log 2>&1; echo tests $?; tail -2 gpurun_out/cs_tests.log
for t in 296 128 64; do TALLY_COLSTATS_BLOCKS=$t timeout 300 python tools/step_time.py --config c4 | grep -o "step_ms_median.: [0-9.]*"; done
