timeout 300 python tools/timeline.py strassen
timeout 300 python tools/timeline.py classical
