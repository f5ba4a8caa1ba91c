CMD="python bench.py --config cfg4 --iterations 2 --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_box -s 2 -c 2 -o gpurun_out/prof_box3 $CMD > /dev/null 2>&1
FDG_FORCE_RECT=1 $CMD > /dev/null 2>&1 && FDG_FORCE_RECT=1 ncu --set full --clock-control none --import-source on -k regex:k_rect -s 2 -c 2 -o gpurun_out/prof_rect3 $CMD > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
