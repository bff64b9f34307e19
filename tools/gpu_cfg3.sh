CFG3_OUT=gpurun_out/r01g_cfg3_decision.json timeout 2400 python tools/cfg3_sweep.py > gpurun_out/cfg3g.log 2>&1; tail -1 gpurun_out/cfg3g.log
