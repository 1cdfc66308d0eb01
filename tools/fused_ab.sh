# A/B of the fused lattice solve forms (config-1 levels 0-2):
# WMC_FUSED_TMEM = 0 shared memory, 1 weights + d_{m-1} in TMEM, 2 weights only
for lv in 0 1 2; do
  for t in ${FORMS:-0 1 2}; do
    WMC_FUSED_TMEM=$t timeout 300 python tools/kernel_probe.py --level $lv --count 4096 --repeat 2 2>&1 | tail -1 | sed "s/^/tmem=$t /"
  done
done
