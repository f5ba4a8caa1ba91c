# per-strip iteration times for equal strips (middle strips keep their height)
for s in "2048,2048,2048,2048,2048,2048,2048" "4096,4096,4096" "8192"; do
  for lin in 1 0; do
    echo "strips $s FDG_FUSED_LIN=$lin"
    FDG_FUSED_LIN=$lin FDG_PIPE_DEBUG=1 FDG_PIPE_STRIPS=$s python scripts/pipe_probe.py 16384 100 2 2>&1 | grep "fdg pipe" | tail -9 | awk '{print $4,$5,$6,$13,$14}' 
  done
done
