mkdir -p gpurun_out
timeout 2000 python -m pytest tests/ -m gpu -q > gpurun_out/gputests.log 2>&1; tail -2 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1500 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4 $?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref $?
for c in c2 c3 c4; do timeout 300 python tools/step_time.py --config $c; done > gpurun_out/step_time.log 2>&1
