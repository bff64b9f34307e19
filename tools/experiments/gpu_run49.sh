for cfg in "0 8" "3 8" "3 4" "4 16" "2 8" "1 8"; do set -- $cfg
  LCMA_OPERAND_HINT=$1 LCMA_SWZ=$2 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:umma_gemm -s 2 -c 1 --csv python tools/ncu_one.py strassen static > gpurun_out/h_$1_$2.csv 2>&1
  echo "hint=$1 swz=$2"; grep -E 'gpu__time_duration|dram__bytes_read|lts__t_sector_hit_rate' gpurun_out/h_$1_$2.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
