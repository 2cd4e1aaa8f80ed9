set -u
O=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:warp_beam -s 3 -c 1 -o $O/ncu_wb_c4 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_wb.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:frame_compact -s 3 -c 1 -o $O/ncu_cmp_c4 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_cmp.log 2>&1
ncu -i $O/ncu_wb_c4.ncu-rep --page source --csv --print-source cuda,sass > $O/ncu_wb_src.csv 2>&1
ncu -i $O/ncu_wb_c4.ncu-rep --page raw --csv > $O/ncu_wb_raw.csv 2>&1
ncu -i $O/ncu_cmp_c4.ncu-rep --page raw --csv > $O/ncu_cmp_raw.csv 2>&1
ncu -i $O/ncu_cmp_c4.ncu-rep --page source --csv --print-source cuda,sass > $O/ncu_cmp_src.csv 2>&1
echo done > $O/ncu_done
