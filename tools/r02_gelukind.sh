mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_c4.py tests/test_gpu_gpt2.py tests/test_gpu_kernels.py -q -x 2>&1 | tail -1
timeout 900 python tools/ptb_overhead.py --config c4 --chosen --reps 2 --out gpurun_out/ptb_gk_c4.json > /dev/null 2>&1; python -c "
import json; d=json.load(open('gpurun_out/ptb_gk_c4.json'))
for k in ['gelu_bwd_erf','bn_act']:
    v=d['by_kind'][k]; print(k, v['n'], v['original_us'], 'P/O', v['speed_ratio'], 'chosen', v['chosen_speed_ratio'])
print('step chosen/orig', round(d['chosen_vs_original_speed'],3))"
for c in c4 c3; do timeout 300 python tools/step_time.py --config $c | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', round(d['step_ms_median'],3))"; done
