mkdir -p gpurun_out
timeout 300 python tools/bnfuse_bench.py --only x2
for o in 1 0; do for c in c2 c4; do if [ $o = 1 ]; then export TALLY_PAIR_TPB_OLD=1; else unset TALLY_PAIR_TPB_OLD; fi; timeout 300 python tools/step_time.py --config $c | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', 'old=$o', round(d['step_ms_median'],3))"; done; done
unset TALLY_PAIR_TPB_OLD
timeout 600 python -m pytest tests/test_gpu_gemm_pair.py tests/test_gpu_bnfuse.py -q -x 2>&1 | tail -2
