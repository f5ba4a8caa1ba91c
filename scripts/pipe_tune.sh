#!/bin/bash
# Strip-pipeline tuning runs on one B200 (results: profiles/r02_pipeline_strip_tuning.txt,
# profiles/r02_pipeline_equal_strips.txt).  Every run prints the per-strip timeline
# (FDG_PIPE_DEBUG) and the wall time per call of scripts/pipe_probe.py.
#   layouts   strip heights (FDG_PIPE_STRIPS), 64-row last strip from the start
#   equal     equal strips, work-balanced vs plain grid (per-launch overhead)
#   tail      late-born last strip (FDG_PIPE_K0) with the default and other layouts
set -u
what=${1:-layouts}
run() { FDG_PIPE_DEBUG=1 python scripts/pipe_probe.py 16384 100 3 2>&1 | grep "fdg pipe\|pipeline=1" | tail -${1:-7}; }
case $what in
layouts)
  for s in "1024,4096,6144,5056" "2048,7168,7104" "1024,5120,10176" "2048,6144,8128" "1024,4096,11200" \
           "1536,6144,8640" "1024,3072,6144,6080" "2048,14272"; do
    echo "strips $s"; FDG_PIPE_STRIPS=$s run 6
  done ;;
equal)
  for s in "2048,2048,2048,2048,2048,2048,2048" "4096,4096,4096" "8192"; do
    for lin in 1 0; do echo "strips $s FDG_FUSED_LIN=$lin"; FDG_FUSED_LIN=$lin FDG_PIPE_STRIPS=$s run 9; done
  done ;;
tail)
  for k0 in 0 30 50 70; do echo "default strips, FDG_PIPE_K0=$k0"; FDG_PIPE_K0=$k0 run 6; done
  for s in "1024,4096,6144,3072" "1024,4096,5120,4096" "1024,4096,6144,3584,1024"; do
    echo "strips $s FDG_PIPE_K0=50"; FDG_PIPE_STRIPS=$s FDG_PIPE_K0=50 run 7
  done ;;
esac
