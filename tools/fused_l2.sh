# level 2: per-step kernels vs the fused solve (z_{n-1} in shared memory / global)
for env in "X=0" "WMC_FUSED_FORCE=1" "WMC_FUSED_ZP_GLOBAL=1" "WMC_FUSED_FORCE=1 WMC_FUSED_TMEM=0"; do
  env $env timeout 300 python tools/kernel_probe.py --level 2 --count 4096 --repeat 2 2>&1 | tail -1 | sed "s/^/$env /"
done
for env in "X=0" "WMC_FUSED_ZP_GLOBAL=1"; do
  env $env timeout 300 python tools/kernel_probe.py --level 3 --count 1024 --repeat 2 2>&1 | tail -1 | sed "s/^/$env /"
done
