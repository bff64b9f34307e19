cd $GRAFT_REPO_ROOT
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__t_bytes.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,launch__registers_per_thread"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --no_large --no_e2e --no_cpu > gpurun_out/r02_launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:umma -s 2 -c 1 -o gpurun_out/r02_str_full python tools/ncu_one.py strassen x 8192 14336 4096 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:umma -s 2 -c 1 -o gpurun_out/r02_cls_full python tools/ncu_one.py classical x 8192 14336 4096 > /dev/null 2>&1
for a in "classical x" "strassen x" "strassen static"; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:umma -s 2 -c 1 python tools/ncu_one.py $a 8192 14336 4096 > "gpurun_out/r02_m_cfg2_${a// /_}.txt" 2>&1
  timeout 900 ncu --metrics $M --clock-control none -k regex:umma -s 1 -c 1 python tools/ncu_one.py $a 32768 28672 8192 > "gpurun_out/r02_m_cfg5_${a// /_}.txt" 2>&1
done
timeout 600 ncu --metrics $M --clock-control none -k regex:group_combine -c 4 python tools/ncu_one.py strassen x 8192 14336 4096 > gpurun_out/r02_m_cfg2_combines.txt 2>&1
