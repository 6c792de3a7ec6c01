mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_resnet.py tests/test_gpu_c4.py -q -x 2>&1 | tail -1
for c in c2 c4; do timeout 900 python tools/ptb_overhead.py --config $c --chosen --reps 2 --out gpurun_out/ptb_bnact_$c.json > /dev/null 2>&1; python -c "
import json; d=json.load(open('gpurun_out/ptb_bnact_$c.json'))
v=d['by_kind']['bn_act']; print('$c bn_act', v['n'], v['original_us'], 'P/O', v['speed_ratio'], 'chosen', v['chosen_speed_ratio'], 'step chosen/orig', round(d['chosen_vs_original_speed'],3))"; done
timeout 300 python tools/step_time.py --config c4 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4', round(d['step_ms_median'],3))"
