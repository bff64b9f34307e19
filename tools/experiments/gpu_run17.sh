timeout 600 ncu --set full --clock-control none --import-source on -k regex:umma_gemm -s 2 -c 1 -o gpurun_out/r01f_umma_fusedH python tools/ncu_one.py strassen > gpurun_out/ncu_f.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:umma_gemm -s 2 -c 1 -o gpurun_out/r01f_umma_classical python tools/ncu_one.py classical > gpurun_out/ncu_c.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01f_launches.csv python bench.py --steps 3 --warmup 3 --no_large --no_e2e --no_cpu > gpurun_out/ncu_l.log 2>&1
ROUNDS=9 timeout 900 python tools/cmp.py 32768 28672 8192 cl:classical st:strassen sts:strassen:s > gpurun_out/r01f_cfg5_cmp.log 2>&1
ROUNDS=9 timeout 900 python tools/cmp.py 16384 28672 8192 cl:classical st:strassen sts:strassen:s >> gpurun_out/r01f_cfg5_cmp.log 2>&1
ROUNDS=9 timeout 900 python tools/cmp.py 8192 14336 4096 cl:classical st:strassen sts:strassen:s >> gpurun_out/r01f_cfg5_cmp.log 2>&1
