for u in 1 2; do for cap in 2368 1184 4736 9472; do LCMA_COMB_U=$u LCMA_COMB_BLOCKS=$cap timeout 120 python tools/comb_u.py; done; done
