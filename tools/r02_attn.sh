mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_c4.py -q -x -k fused_attention > gpurun_out/attn_tests.log 2>&1; echo t1 $?; tail -3 gpurun_out/attn_tests.log
timeout 900 python -m pytest tests/test_gpu_c4.py tests/test_gpu_gpt2.py -q -x > gpurun_out/attn_tests2.log 2>&1; echo t2 $?; tail -3 gpurun_out/attn_tests2.log
for f in 0 1; do TALLY_FUSE_ATTENTION=$f timeout 300 python tools/step_time.py --config c4; done > gpurun_out/step_time.log 2>&1
timeout 600 python tools/ptb_overhead.py --config c4 --chosen --out gpurun_out/ptb_overhead_c4.json > /dev/null 2>&1; echo ptbo $?
