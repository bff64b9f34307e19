# round-2 final evidence: bench line, launch list, ncu metrics of the GEMM kernels (bf16 cfg2 / cfg5, FP8 cfg2), full capture of the fused Strassen GEMM
cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err; tail -c 600 gpurun_out/r02f_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02f_launches.csv python bench.py --steps 2 --warmup 1 --no_large --no_e2e --no_cpu > gpurun_out/r02f_launches_bench.log 2>&1
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__t_bytes.sum,launch__registers_per_thread"
for a in "classical x" "strassen x" "strassen static"; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:"umma|combine" -s 2 -c 3 python tools/ncu_one.py $a 8192 14336 4096 > "gpurun_out/r02f_m_cfg2_${a// /_}.txt" 2>&1
  timeout 900 ncu --metrics $M --clock-control none -k regex:umma -s 1 -c 1 python tools/ncu_one.py $a 32768 28672 8192 > "gpurun_out/r02f_m_cfg5_${a// /_}.txt" 2>&1
done
for a in "classical static" "strassen static"; do
  DT=4 timeout 600 ncu --metrics $M --clock-control none -k regex:umma -s 2 -c 1 python tools/ncu_one.py $a 8192 14336 4096 > "gpurun_out/r02f_m_fp8_cfg2_${a// /_}.txt" 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:umma -s 2 -c 1 -o gpurun_out/r02f_str_full python tools/ncu_one.py strassen static 8192 14336 4096 > /dev/null 2>&1
for f in gpurun_out/r02f_m_*.txt; do echo "== $f"; grep -E "umma_gemm|group_comb|duration|dram__bytes|hit_rate|tensor_cycles" $f | head -24; done
