mkdir -p gpurun_out
for S in 4 5 6; do
  TALLY_NVCC_DEFINES="-DTALLY_STAGES_PAIR=$S" python -c "from paper_2410_07381_b200 import build; build.build(force=True)" > /dev/null 2>&1
  for shp in "8192 8192 1024" "8192 8192 2048"; do
    timeout 120 python tools/gemm_worker_timeline.py $shp | python -c "
import sys,json; d=json.load(sys.stdin); r=d['runs'][1]
print('S=$S', '$shp', 'elapsed', round(r['elapsed_us'],1), 'step', [round(x,2) for x in r['block_step_us_p10_p50_p90']], 'exit', [round(x,1) for x in r['exit_us_p0_p50_max']])"
  done
done
