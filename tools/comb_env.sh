# Combine-B bandwidth under combine-kernel variants (one process each)
for env in "" "LCMA_COMB16_PQ4=1" "LCMA_COMB_BLOCKS=1184" "LCMA_COMB_BLOCKS=9472" "LCMA_COMB16_PQ4=1 LCMA_COMB_BLOCKS=9472" "LCMA_COMB_BLOCKS=100000"; do
  echo "== $env"; env $env python tools/combB_exp.py 2>&1 | grep -E "bl=1" | head -3
done
