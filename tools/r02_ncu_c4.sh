mkdir -p gpurun_out
timeout 300 python tools/ncu_prog.py --config c4 top > gpurun_out/c4_top.txt 2>&1
N="bert.encoder.layer.0.attention.self.qk bert.encoder.layer.0.intermediate.dense.wgrad bert.encoder.layer.0.output.dense.gemm"
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_gemm" -c 6 -o gpurun_out/ncu_c4_gemms python tools/ncu_prog.py --config c4 kernels $N > gpurun_out/ncu_c4_gemms.log 2>&1; echo ncu $?
