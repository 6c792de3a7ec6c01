mkdir -p gpurun_out
for t in 296 512; do TALLY_COLSTATS_BLOCKS=$t timeout 300 python tools/step_time.py --config c4 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4 colstats rows4 target=$t', round(d['step_ms_median'],3))"; done
TALLY_COLSTATS_BLOCKS=296 timeout 300 python tools/step_time.py --config c3 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 rows4', round(d['step_ms_median'],3))"
timeout 600 python -m pytest tests/test_gpu_c4.py tests/test_gpu_gpt2.py -q -x 2>&1 | tail -1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc $?
