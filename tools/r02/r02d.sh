cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/r02d_pytest.txt
export ROUNDS=5 REPS=2
python tools/cmp.py 32768 28672 8192 static:classical:sched=4 dyn:classical dyn_pf8:classical:pf=8 dyn_pf16:classical:pf=16 dyn_swz8:classical:swz=8 > gpurun_out/r02d_cfg5_classical.txt 2>&1
python tools/cmp.py 32768 28672 8192 static:strassen:s:sched=4 dyn:strassen:s dyn_pf8:strassen:s:pf=8 dyn_pf16:strassen:s:pf=16 dyn_swz4:strassen:s:swz=4 > gpurun_out/r02d_cfg5_strassen.txt 2>&1
export ROUNDS=7 REPS=5
python tools/cmp.py 8192 14336 4096 static:classical:sched=4 dyn:classical dyn_pf8:classical:pf=8 dyn_pf16:classical:pf=16 sstatic:strassen:s:sched=4 sdyn:strassen:s sdyn_pf8:strassen:s:pf=8 sdyn_pf16:strassen:s:pf=16 > gpurun_out/r02d_cfg2.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:umma -s 2 -c 1 python tools/ncu_one.py classical x 32768 28672 8192 > gpurun_out/r02d_ncu_cls_cfg5.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:umma -s 2 -c 1 python tools/ncu_one.py strassen static 32768 28672 8192 > gpurun_out/r02d_ncu_str_cfg5.txt 2>&1
