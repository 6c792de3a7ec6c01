mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_c4.py tests/test_gpu_gpt2.py tests/test_gpu_gemm_pair.py tests/test_gpu_resnet.py -q -x 2>&1 | tail -1
for c in c4 c3 c2; do timeout 300 python tools/step_time.py --config $c | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', round(d['step_ms_median'],3))"; done
