timeout 200 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "exact and not random" 2>&1 | tail -2
for env in "" "LCMA_B2D=1"; do
env $env timeout 100 python tools/tf32_layout.py 8192 14336 4096 2>&1 | grep "bl=0"
env $env timeout 100 python tools/layout_exp.py 2>&1 | grep -E "bl=0 (classical|strassen)" | head -2
done
