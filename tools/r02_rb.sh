mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_resnet.py tests/test_gpu_c4.py -q -x > gpurun_out/rb_tests.log 2>&1; echo tests rc $?; tail -2 gpurun_out/rb_tests.log
for c in c2 c4; do timeout 300 python tools/step_time.py --config $c; done > gpurun_out/step_time.log 2>&1
for c in c2 c4; do timeout 600 python tools/ptb_overhead.py --config $c --chosen --out gpurun_out/ptb_overhead_$c.json > /dev/null 2>&1; done
