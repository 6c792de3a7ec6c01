mkdir -p gpurun_out
timeout 600 python tools/c2_diag.py --ms 2000 --load 0.5 --burst 20 > gpurun_out/c2_diag.json 2> gpurun_out/c2_diag.err; echo diag $?
timeout 120 python tools/gemm_worker_timeline.py 4096 3072 1024 > gpurun_out/tl_pair_qkv.json 2>&1
timeout 120 python tools/gemm_worker_timeline.py 8192 8192 8192 > gpurun_out/tl_pair_8192.json 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_gemm" -c 2 -o gpurun_out/ncu_c4_decoder python tools/ncu_prog.py --config c4 kernels cls.predictions.decoder > gpurun_out/ncu_c4_decoder.log 2>&1; echo ncu $?
