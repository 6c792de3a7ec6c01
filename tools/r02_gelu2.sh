mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_c4.py tests/test_gpu_gpt2.py tests/test_gpu_resnet.py tests/test_gpu_intercept.py -q -x 2>&1 | tail -1
for c in c4 c3 c2; do timeout 300 python tools/step_time.py --config $c | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', round(d['step_ms_median'],3))"; done
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum --clock-control none -k "regex:k_original" python tools/ncu_prog.py --config c4 kernels bert.encoder.layer.3.intermediate.gelu_bwd bert.encoder.layer.3.intermediate.dense.bias 2>&1 | grep -E "GeluBwd|BnAct|duration|issue_active|bytes_read" | head -12
