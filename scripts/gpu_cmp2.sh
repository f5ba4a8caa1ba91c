CMD="python bench.py --config cfg4b --iterations 1 --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_box -s 1 -c 1 -o gpurun_out/prof_box4b $CMD > /dev/null 2>&1
FDG_FORCE_RECT=1 $CMD > /dev/null 2>&1 && FDG_FORCE_RECT=1 ncu --set full --clock-control none --import-source on -k regex:k_rect -s 1 -c 1 -o gpurun_out/prof_rect4b $CMD > /dev/null 2>&1
ls -la gpurun_out/*4b*.ncu-rep
