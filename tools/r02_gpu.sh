# Round-2 measurement cycle on one B200 (run under gpurun from the repo root).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1800 python -m pytest tests/ -m gpu -q -x > gpurun_out/gputests.log 2>&1; tail -3 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench rc $?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc $?
timeout 600 python tools/ptb_overhead.py --config c4 --chosen --out gpurun_out/ptb_overhead_c4.json > gpurun_out/ptb_overhead_c4.log 2>&1; echo ptbo rc $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python tools/ncu_prog.py --config c4 step > gpurun_out/ncu_step.log 2>&1; echo ncu rc $?
