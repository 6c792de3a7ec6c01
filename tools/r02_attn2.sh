mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_c4.py -q -x 2>&1 | tail -1
timeout 300 python tools/step_time.py --config c4 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4', round(d['step_ms_median'],3))"
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k "regex:k_original" python tools/ncu_prog.py --config c4 kernels bert.encoder.layer.3.attention.self.qk_softmax bert.encoder.layer.3.attention.self.dp_softmax_bwd 2>&1 | grep -E "AttnSoftmax|duration|issue_active" | head -8
