# A/B of the fused lattice solve: tensor-memory vs shared-memory form (config-1 levels 0, 1)
for lv in 0 1; do
  for t in 0 1; do
    WMC_FUSED_TMEM=$t timeout 300 python tools/kernel_probe.py --level $lv --count 4096 --repeat 2 2>&1 | tail -1 | sed "s/^/tmem=$t /"
  done
done
