mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_conv.py tests/test_gpu_c4.py -q -x 2>&1 | tail -3
timeout 300 python tools/bnfuse_bench.py --only x2
for o in 1 0; do if [ $o = 1 ]; then export TALLY_PAIR_TPB_OLD=1; else unset TALLY_PAIR_TPB_OLD; fi; timeout 300 python tools/step_time.py --config c2 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2 old=$o', round(d['step_ms_median'],3))"; timeout 900 python tools/ptb_overhead.py --config c2 --chosen --reps 2 --out gpurun_out/ptb_overhead_c2_old$o.json > /dev/null 2>&1; python -c "
import json; d=json.load(open('gpurun_out/ptb_overhead_c2_old$o.json')); print('old=$o chosen/orig', round(d['chosen_vs_original_speed'],3), 'x2', d['by_kind']['gemm_bf16_x2']['chosen_speed_ratio'])"; done
