mkdir -p gpurun_out
for shp in "4096 3072 1024" "4096 1024 4096" "8192 8192 8192"; do
timeout 120 python tools/gemm_worker_timeline.py $shp > "gpurun_out/tl_pair_${shp// /x}.json" 2>&1
timeout 120 python tools/gemm_worker_timeline.py $shp --single > "gpurun_out/tl_single_${shp// /x}.json" 2>&1
done
timeout 300 python -m pytest tests/test_gpu_gemm_pair.py -q -x 2>&1 | tail -2
