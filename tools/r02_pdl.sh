mkdir -p gpurun_out
for c in c4 c3 c2; do for f in 0 1; do TALLY_PDL=$f timeout 300 python tools/step_time.py --config $c | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', 'pdl=$f', round(d['step_ms_median'],3))"; done; done
TALLY_PDL=1 timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_scheduler.py tests/test_gpu_gemm_pair.py tests/test_gpu_c4.py tests/test_gpu_irjit.py -q -x > gpurun_out/pdl_tests.log 2>&1; echo tests $?; tail -2 gpurun_out/pdl_tests.log
