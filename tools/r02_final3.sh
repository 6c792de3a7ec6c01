# round-2 closing measurements: every GPU test, smoke, the three bench lines,
# per-kind roofline / transformation cost, the native steps
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/ -m gpu -q > gpurun_out/gputests.log 2>&1; echo tests $?; tail -2 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
for c in c2 c3 c4; do timeout 300 python tools/step_time.py --config $c; done > gpurun_out/step_time.log 2>&1; echo steps $?
timeout 1500 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4 rc $?
timeout 1500 python bench.py --config c2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2 rc $?
timeout 1500 python bench.py --config c3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo c3 rc $?
for c in c2 c3 c4; do timeout 900 python tools/ptb_overhead.py --config $c --chosen --out gpurun_out/ptb_overhead_$c.json > /dev/null 2>&1; echo ptb $c $?; done
