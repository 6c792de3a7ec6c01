mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gpt2.py tests/test_gpu_c4.py -q -x > gpurun_out/ln_tests.log 2>&1; echo tests $?; tail -2 gpurun_out/ln_tests.log
for c in c4 c3; do timeout 300 python tools/step_time.py --config $c | grep -o "step_ms_median.: [0-9.]*"; done
timeout 600 python tools/ptb_overhead.py --config c4 --chosen --out gpurun_out/ptb_overhead_c4.json > /dev/null 2>&1; echo ptbo $?
