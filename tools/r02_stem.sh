mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_conv.py -q 2>&1 | grep -E "Error|passed|failed" | head -8
for f in 0 1; do TALLY_IMPLICIT_STEM=$f timeout 300 python tools/step_time.py --config c2 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2 stem=$f', round(d['step_ms_median'],3), d['kernels'])"; done
timeout 900 python -m pytest tests/test_gpu_resnet.py tests/test_gpu_c4.py tests/test_gpu_gpt2.py -q -x 2>&1 | tail -2
