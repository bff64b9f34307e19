cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/r02k_pytest.txt
python bench.py --steps 20 --warmup 5 > gpurun_out/r02k_bench.json 2> gpurun_out/r02k_bench.err
python bench.py --workload cfg5 --steps 5 --warmup 3 > gpurun_out/r02k_cfg5.json 2>> gpurun_out/r02k_bench.err
