mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_c4.py tests/test_gpu_kernels.py tests/test_gpu_gemm_pair.py -q -x 2>&1 | tail -2
timeout 300 python tools/step_time.py --config c4 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4 fast erf', round(d['step_ms_median'],3))"
timeout 900 python tools/ptb_overhead.py --config c4 --reps 2 --out gpurun_out/ptb_overhead_c4_gelu.json > /dev/null 2>&1; python -c "
import json; d=json.load(open('gpurun_out/ptb_overhead_c4_gelu.json'))
for k in ['bn_act','gelu_bwd']: v=d['by_kind'][k]; print(k, v['n'], v['original_us'], v['achieved_TBps'])"
