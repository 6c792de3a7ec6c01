# fused batch-norm statistics: parity, then the C2 step with / without
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bnfuse.py -q -x > gpurun_out/bnfuse_tests.log 2>&1; echo bnfuse $?; tail -15 gpurun_out/bnfuse_tests.log
for f in 0 1; do TALLY_BN_FUSE=$f timeout 300 python tools/step_time.py --config c2 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2', 'bnfuse=$f', round(d['step_ms_median'],3), d.get('kernels'))"; done
timeout 900 python -m pytest tests/test_gpu_resnet.py -q -x > gpurun_out/bnfuse_resnet.log 2>&1; echo resnet $?; tail -5 gpurun_out/bnfuse_resnet.log
for f in 0 1; do TALLY_BN_FUSE=$f timeout 600 python tools/ptb_overhead.py --config c2 --reps 2 --launches gpurun_out/c2_launches_f$f.jsonl > /dev/null 2>&1; done
