LCMA_DEBUG=16 timeout 600 ncu --set full --clock-control none --import-source on -k regex:umma_gemm -s 2 -c 1 -o gpurun_out/s16b python tools/ncu_one.py strassen static > gpurun_out/ncu_s16b.log 2>&1
