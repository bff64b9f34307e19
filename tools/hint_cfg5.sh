for rep in 1 2; do
python tools/env_one.py classical dyn 32768 28672 8192 5 2>&1 | grep median
LCMA_PARTIAL_HINT=0 python tools/env_one.py strassen static 32768 28672 8192 5 2>&1 | grep median
LCMA_PARTIAL_HINT=1 python tools/env_one.py strassen static 32768 28672 8192 5 2>&1 | grep median
LCMA_PARTIAL_HINT=0 python tools/env_one.py strassen dyn 32768 28672 8192 5 2>&1 | grep median
LCMA_PARTIAL_HINT=1 python tools/env_one.py strassen dyn 32768 28672 8192 5 2>&1 | grep median
done
