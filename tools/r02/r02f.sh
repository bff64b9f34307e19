cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/r02f_clocks.csv &
SMI=$!
python tools/r02/kwait.py 8192 14336 4096 > gpurun_out/r02f_kwait_cfg2.txt 2>&1
python tools/r02/kwait.py 32768 28672 8192 > gpurun_out/r02f_kwait_cfg5.txt 2>&1
kill $SMI
timeout 600 ncu --set full --clock-control base -k regex:umma -s 2 -c 1 -o gpurun_out/r02f_cls python tools/ncu_one.py classical x 8192 14336 4096 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control base -k regex:umma -s 2 -c 1 -o gpurun_out/r02f_str python tools/ncu_one.py strassen static 8192 14336 4096 > /dev/null 2>&1
ls gpurun_out
