cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/r02h_bench.json 2> gpurun_out/r02h_bench.err; tail -c 300 gpurun_out/r02h_bench.json
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__t_bytes.sum"
timeout 600 ncu --metrics $M --clock-control none -k regex:umma -s 2 -c 1 python tools/ncu_one.py classical x 8192 14336 4096 > gpurun_out/r02h_m_cfg2_classical.txt 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:umma -s 1 -c 1 python tools/ncu_one.py classical x 32768 28672 8192 > gpurun_out/r02h_m_cfg5_classical.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02h_launches.csv python bench.py --steps 2 --warmup 1 --no_large --no_e2e --no_cpu > /dev/null 2>&1
for f in gpurun_out/r02h_m_*.txt; do echo "== $f"; grep -E "duration|dram__bytes|hit_rate|tensor_cycles|per_second" $f; done
