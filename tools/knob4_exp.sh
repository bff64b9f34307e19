for env in "" "LCMA_OPERAND_HINT=1" "LCMA_OPERAND_HINT=2" "LCMA_PARTIAL_HINT=0" "LCMA_SWZ=16" "LCMA_SWZ=4" "LCMA_DISCARD=0"; do
env $env python tools/env_one.py strassen static 8192 14336 4096 5 2>&1 | grep median
done
for env in "" "LCMA_OPERAND_HINT=1" "LCMA_SWZ=16" "LCMA_SWZ=4"; do
env $env python tools/env_one.py classical dyn 8192 14336 4096 5 2>&1 | grep median
done
