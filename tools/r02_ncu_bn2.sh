# ncu --set full of the C2 batch-norm kernels after statistics fusion, plus the step's launch list
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_original" -o gpurun_out/ncu_c2_bn2 python tools/ncu_prog.py --config c2 kernels layer1.0.bn3.bwd_stats layer4.0.bn2.bwd_stats layer1.0.bn3.bwd layer1.0.conv1.gemm.bnfold layer1.0.bn3.act layer3.0.conv2.gemm.reduce > gpurun_out/ncu_c2_bn2.log 2>&1; echo full $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c2_launches.csv python tools/ncu_prog.py --config c2 step > gpurun_out/r02_c2_launches.log 2>&1; echo list $?
