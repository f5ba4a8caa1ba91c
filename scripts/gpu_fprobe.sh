mkdir -p gpurun_out
( for b in 60 128 256 512 4096; do FDG_FUSED_V=1 FDG_FUSED_BAND=$b python scripts/fused_probe.py; done
  for v in 0 2; do FDG_FUSED_V=$v python scripts/fused_probe.py; done
  FDG_FUSED_V=1 python scripts/fused_probe.py 1024 4096 10
  FDG_FUSED_V=1 python scripts/fused_probe.py 4096 1024 10
  FDG_NO_FUSED=1 python scripts/fused_probe.py ) > gpurun_out/fprobe.log 2>&1
