cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 200 -p no:cacheprovider > gpurun_out/r02y_pytest.txt 2>&1
