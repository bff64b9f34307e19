cd $GRAFT_REPO_ROOT
timeout 120 python tools/timeline.py strassen 8192 14336 4096
timeout 120 python tools/timeline.py classical 8192 14336 4096
