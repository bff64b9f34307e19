cd $GRAFT_REPO_ROOT
LCMA_LIB=$GRAFT_REPO_ROOT/paper_2605_06057_b200/liblcma_diag.so timeout 300 python -u tests/_diag_homes.py > gpurun_out/r02x_homes.txt 2>&1
echo "rc=$?" >> gpurun_out/r02x_homes.txt
timeout 900 python -m pytest tests -m gpu -v --timeout 120 -k "not diag_build" -p no:cacheprovider 2>&1 > gpurun_out/r02x_pytest.txt
