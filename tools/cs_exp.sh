for rep in 1 2; do for env in "" "LCMA_C_CS=1"; do
env $env python tools/env_one.py strassen static 8192 14336 4096 5 2>&1 | grep median
env $env python tools/env_one.py classical dyn 8192 14336 4096 5 2>&1 | grep median
env $env python tools/env_one.py strassen static 16384 28672 8192 3 2>&1 | grep median
done; done
