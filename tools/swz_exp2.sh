for algo in laderman strassen2; do
for swz in 16 8 4 2; do
LCMA_SWZ=$swz python tools/env_one.py $algo static 12288 12288 12288 3 2>&1 | grep median
done; done
for rep in 1 2; do
for swz in 16 8; do
LCMA_SWZ=$swz python tools/env_one.py strassen dyn 16384 28672 8192 5 2>&1 | grep median
LCMA_SWZ=$swz python tools/env_one.py strassen dyn 8192 14336 4096 5 2>&1 | grep median
done; done
python tools/env_one.py classical dyn 12288 12288 12288 3 2>&1 | grep median
