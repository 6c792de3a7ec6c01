mkdir -p gpurun_out
timeout 1500 python bench.py --config c3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo c3 $?
timeout 1500 python bench.py --config c2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2 $?
for c in c2 c3 c4; do timeout 600 python tools/ptb_overhead.py --config $c --chosen --out gpurun_out/ptb_overhead_$c.json > /dev/null 2>&1; done; echo ptbo
for c in c2 c3 c4; do timeout 300 python tools/step_time.py --config $c; done > gpurun_out/step_time.log 2>&1
