set -x
nvidia-smi --query-gpu=name,clocks.sm,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for st in dyn static; do
timeout 300 python tools/env_exp.py classical $st 8192 14336 4096 ''
timeout 300 python tools/env_exp.py strassen $st 8192 14336 4096 'LCMA_QFULL=1' 'LCMA_QFULL=0' 'LCMA_QFULL=1,LCMA_REG_PARTIAL=0' 'LCMA_QFULL=0,LCMA_REG_PARTIAL=0,LCMA_SMEM_PARTIAL=0'
done
timeout 300 python tools/env_exp.py classical dyn 32768 28672 8192 ''
timeout 300 python tools/env_exp.py strassen static 32768 28672 8192 'LCMA_QFULL=1' 'LCMA_QFULL=0'
