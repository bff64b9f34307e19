timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "exact or float or determinism or cfg2" 2>&1 | tail -1
for rep in 1 2; do for env in "" "LCMA_SMEM_PARTIAL=0"; do
env $env timeout 120 python tools/env_one.py strassen static 8192 14336 4096 5 2>&1 | grep median
env $env timeout 200 python tools/env_one.py strassen static 16384 28672 8192 3 2>&1 | grep median
done; done
timeout 120 python tools/env_one.py classical dyn 8192 14336 4096 5 2>&1 | grep median
timeout 200 python tools/env_one.py classical dyn 16384 28672 8192 3 2>&1 | grep median
