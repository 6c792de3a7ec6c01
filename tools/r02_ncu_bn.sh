mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_original|k_ptb" -c 4 -o gpurun_out/ncu_c2_bnstats python tools/ncu_prog.py --config c2 kernels layer1.0.bn1.stats layer1.0.bn3.stats > gpurun_out/ncu_c2_bnstats.log 2>&1; echo $?
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_original|k_ptb" -c 4 -o gpurun_out/ncu_c4_colstats python tools/ncu_prog.py --config c4 kernels layer.0.output.dense.dbias layer.0.output.LayerNorm.dparams > gpurun_out/ncu_c4_colstats.log 2>&1; echo $?
