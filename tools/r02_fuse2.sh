mkdir -p gpurun_out
for f in "" "bias" "bias,res" "bias,act" "bias,res,act"; do TALLY_FUSE_EPILOGUE=$f timeout 300 python tools/step_time.py --config c4 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$f', d['step_ms_median'])"; done > gpurun_out/fuse_ab.txt 2>&1
