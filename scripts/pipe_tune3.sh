for k0 in 0 30 50 70; do
  echo "default strips, FDG_PIPE_K0=$k0"
  FDG_PIPE_K0=$k0 FDG_PIPE_DEBUG=1 python scripts/pipe_probe.py 16384 100 3 2>&1 | grep "fdg pipe\|pipeline=1" | tail -6
done
for s in "1024,4096,6144,3072" "1024,4096,5120,4096" "1024,4096,6144,3584,1024"; do
  echo "strips $s FDG_PIPE_K0=50"
  FDG_PIPE_STRIPS=$s FDG_PIPE_K0=50 FDG_PIPE_DEBUG=1 python scripts/pipe_probe.py 16384 100 3 2>&1 | grep "fdg pipe\|pipeline=1" | tail -7
done
