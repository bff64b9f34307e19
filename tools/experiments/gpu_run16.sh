for d in 1 1920 0; do
LCMA_DEBUG=$d timeout 600 ncu --set full --clock-control none --import-source on -k regex:umma_gemm -s 2 -c 1 -o gpurun_out/d$d python tools/ncu_one.py strassen static > gpurun_out/ncu_d$d.log 2>&1
done
