mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -m gpu -q > gpurun_out/gputests.log 2>&1; tail -2 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv python tools/ncu_c2.py step > gpurun_out/ncu_step.log 2>&1
N="layer2.0.conv1.gemm layer2.0.conv2.dgrad layer1.0.conv2.dgrad layer1.0.conv2.im2col layer1.0.bn3.bwd_stats layer1.0.conv2.wgrad"
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_gemm|k_original|k_ptb" -c 12 -o gpurun_out/ncu_c2_final python tools/ncu_c2.py kernels $N > gpurun_out/ncu_c2_final.log 2>&1
python -c "
import json;d=json.load(open('gpurun_out/bench_c2.json')); c=d['components']
print('ovh', round(d['value'],2), 'be', round(c['be_throughput_pct'],1), c['be_steps_per_s'], 'pre', c['preempt_latency_us_p50_p99_max'], 'KP', d['baselines'], 'e2e', round(d['e2e']['value'],2), c['window_p99_us_solo_co'], d['roofline']['kernel'], round(d['roofline']['frac'],3), d['roofline']['traffic'])"
