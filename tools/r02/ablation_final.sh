cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/abl
timeout 900 python tools/ablation.py 8192 14336 4096 --static > gpurun_out/abl/ablation_cfg2.json 2> gpurun_out/abl/ablation_cfg2.err
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
for n in classical alg1_unfused group_parallel split_group_paper cache_aware_lockstep product_order_slots_discard onchip_partial_homes variant3_producer_combine diag_mainloop_only; do
  ABL_ONE=$n timeout 300 ncu --metrics $M --clock-control none -k regex:umma -s 2 -c 1 python tools/ablation.py 8192 14336 4096 --static > gpurun_out/abl/ncu_$n.txt 2>&1
done
python - <<'PY'
import json
d=json.load(open("gpurun_out/abl/ablation_cfg2.json"))
for n,v in d["steps"].items(): print(n, round(v["ms"]*1e3,1), v.get("sm_mhz_median"), v.get("power_w_median"))
PY
