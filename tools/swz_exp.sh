for shape in "8192 14336 4096" "16384 28672 8192"; do
for swz in 16 8 4 32; do
LCMA_SWZ=$swz python tools/env_one.py strassen static $shape 5 2>&1 | grep median
done
LCMA_SWZ=16 python tools/env_one.py classical dyn $shape 5 2>&1 | grep median
LCMA_SWZ=8 python tools/env_one.py classical dyn $shape 5 2>&1 | grep median
done
