LCMA_DEBUG=16 timeout 600 ncu --set full --clock-control none --import-source on -k regex:umma_gemm -s 2 -c 1 -o gpurun_out/s16 python tools/ncu_one.py strassen static > gpurun_out/ncu_s16.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:umma_gemm -s 2 -c 1 -o gpurun_out/sts python tools/ncu_one.py strassen static > gpurun_out/ncu_sts.log 2>&1
