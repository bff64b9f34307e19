cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -5 > gpurun_out/r02w_pytest.txt
python bench.py --steps 20 --warmup 5 > gpurun_out/r02w_bench.json 2> gpurun_out/r02w_bench.err
