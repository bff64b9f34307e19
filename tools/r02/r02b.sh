cd $GRAFT_REPO_ROOT
python tools/r02/drift.py classical 32768 28672 8192 > gpurun_out/r02b_drift.txt 2>&1
python tools/r02/drift.py strassen 32768 28672 8192 >> gpurun_out/r02b_drift.txt 2>&1
python tools/r02/drift.py classical 8192 14336 4096 >> gpurun_out/r02b_drift.txt 2>&1
python tools/r02/drift.py strassen 8192 14336 4096 >> gpurun_out/r02b_drift.txt 2>&1
cat > /tmp/cub.py <<'PY'
import torch
M,N,K=32768,28672,8192
A=torch.randn(M,K,device='cuda',dtype=torch.bfloat16); B=torch.randn(N,K,device='cuda',dtype=torch.bfloat16)
for _ in range(3): C=torch.matmul(A,B.t())
torch.cuda.synchronize()
PY
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__cluster_dim_x,launch__cluster_dim_y,launch__block_size,sm__cycles_elapsed.avg.per_second --clock-control none -s 2 -c 1 python /tmp/cub.py > gpurun_out/r02b_cublas_ncu.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:umma -s 2 -c 1 python tools/ncu_one.py classical x 32768 28672 8192 > gpurun_out/r02b_ours_ncu.txt 2>&1
