timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_r01f.log 2>&1; tail -1 gpurun_out/bench_r01f.log
timeout 600 python tools/cfg4.py > gpurun_out/r01f_cfg4.json 2> gpurun_out/cfg4.err; tail -5 gpurun_out/r01f_cfg4.json
CFG3_OUT=gpurun_out/r01f_cfg3_decision.json timeout 1800 python tools/cfg3_sweep.py > gpurun_out/cfg3.log 2>&1; tail -1 gpurun_out/cfg3.log
