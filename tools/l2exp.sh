for shape in "8192 14336 4096" "16384 28672 8192"; do
for rep in 1 2; do
python tools/env_one.py classical dyn $shape 2>&1 | grep median
python tools/env_one.py strassen static $shape 2>&1 | grep median
LCMA_PARTIAL_HINT=1 python tools/env_one.py strassen static $shape 2>&1 | grep median
LCMA_L2PERSIST=64 python tools/env_one.py strassen static $shape 2>&1 | grep -E "median|Error"
LCMA_L2PERSIST=64 LCMA_PARTIAL_HINT=1 python tools/env_one.py strassen static $shape 2>&1 | grep -E "median|Error"
done; done
python -c "import torch; print(torch.cuda.get_device_properties(0))" 2>&1 | tail -1
