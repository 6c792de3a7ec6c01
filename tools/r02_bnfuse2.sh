mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bnfuse.py -q -x > gpurun_out/bnfuse_tests.log 2>&1; echo bnfuse $?; tail -3 gpurun_out/bnfuse_tests.log
for r in 128 32; do echo rows=$r; TALLY_BNFUSE_ROWS=$r timeout 300 python tools/bnfuse_bench.py; done
for f in "0 128" "1 128" "1 32"; do set -- $f; TALLY_BN_FUSE=$1 TALLY_BNFUSE_ROWS=$2 timeout 300 python tools/step_time.py --config c2 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2', 'bnfuse=$1 rows=$2', round(d['step_ms_median'],3), d.get('kernels'))"; done
