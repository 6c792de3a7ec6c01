mkdir -p gpurun_out
timeout 2400 python -m pytest tests/ -m gpu -q > gpurun_out/gputests.log 2>&1; tail -3 gpurun_out/gputests.log
timeout 300 python tools/dbg_sched.py > gpurun_out/dbg_sched.log 2>&1
timeout 600 python tools/ptb_overhead.py --config c4 --chosen --out gpurun_out/ptb_overhead_c4.json > gpurun_out/ptb_overhead_c4.log 2>&1; echo ptbo rc $?
