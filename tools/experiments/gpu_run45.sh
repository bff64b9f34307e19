mkdir -p gpurun_out/ablation_r01g
timeout 900 python tools/ablation.py --static > gpurun_out/ablation_r01g/abl_g_cfg2_static.json 2> gpurun_out/ablation_r01g/err.txt
for s in classical alg1_unfused group_parallel split_group_paper cache_aware_lockstep product_order_slots_discard onchip_partial_homes variant3_producer_combine diag_mainloop_only; do
  ABL_ONE=$s timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:umma_gemm -s 2 -c 1 --csv python tools/ablation.py --static > gpurun_out/ablation_r01g/abl_g_ncu_$s.csv 2>&1
done
