# FP8 kernels: ncu metrics of the block-scaled GEMM (classical, Strassen) at cfg2 / cfg5 and the quantizing combines
cd $GRAFT_REPO_ROOT
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__t_bytes.sum,launch__registers_per_thread"
for a in "classical static" "strassen static"; do
  DT=4 timeout 600 ncu --metrics $M --clock-control none -k regex:umma -s 2 -c 1 python tools/ncu_one.py $a 8192 14336 4096 > "gpurun_out/fp8_m_cfg2_${a// /_}.txt" 2>&1
  DT=4 timeout 900 ncu --metrics $M --clock-control none -k regex:umma -s 1 -c 1 python tools/ncu_one.py $a 32768 28672 8192 > "gpurun_out/fp8_m_cfg5_${a// /_}.txt" 2>&1
done
DT=4 timeout 600 ncu --metrics $M --clock-control none -k regex:group_combine -c 2 python tools/ncu_one.py strassen x 8192 14336 4096 > gpurun_out/fp8_m_cfg2_combines.txt 2>&1
DT=4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:umma -s 2 -c 1 -o gpurun_out/fp8_str_full python tools/ncu_one.py strassen static 8192 14336 4096 > /dev/null 2>&1
