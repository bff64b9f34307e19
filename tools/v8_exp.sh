for rep in 1 2; do
for env in "" "LCMA_NO_V8=1"; do
env $env python tools/env_one.py classical dyn 8192 14336 4096 2>&1 | grep median
env $env python tools/env_one.py strassen static 8192 14336 4096 2>&1 | grep median
done; done
