cd $GRAFT_REPO_ROOT
timeout 700 python -m pytest tests/test_gpu_fp8.py -q > gpurun_out/fp8_tests2.txt 2>&1; grep -E "passed|failed|^FAILED" gpurun_out/fp8_tests2.txt | tail -8
export BL=1 ROUNDS=5 REPS=3
DT=4 timeout 300 python tools/cmp.py 8192 14336 4096 cl:classical cls:classical:s st:strassen sts:strassen:s > gpurun_out/fp8_cfg2.txt 2>&1; cat gpurun_out/fp8_cfg2.txt
DT=0 timeout 300 python tools/cmp.py 8192 14336 4096 bcl:classical bsts:strassen:s > gpurun_out/bf16_cfg2_ref.txt 2>&1; cat gpurun_out/bf16_cfg2_ref.txt
DT=4 ROUNDS=3 timeout 600 python tools/cmp.py 32768 28672 8192 cl:classical cls:classical:s st:strassen sts:strassen:s > gpurun_out/fp8_cfg5.txt 2>&1; cat gpurun_out/fp8_cfg5.txt
for M in 1024 2048 4096 16384; do DT=4 timeout 200 python tools/cmp.py $M 14336 4096 cl:classical cls:classical:s st:strassen sts:strassen:s > gpurun_out/fp8_m$M.txt 2>&1; cat gpurun_out/fp8_m$M.txt; done
