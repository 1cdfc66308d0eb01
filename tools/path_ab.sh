# substep path A/B on config-1 levels 3 and 4 (bench batch sizes): lattice (on-chip, per-sample CTAs) vs global (HBM/L2-resident R rows)
for lv in 3 4; do
  cnt=$([ $lv = 3 ] && echo 1280 || echo 256)
  for p in lattice global; do
    if [ $p = global ]; then e="WMC_SUBSTEP_PATH=global"; else e="X=1"; fi
    env $e timeout 300 python tools/kernel_probe.py --level $lv --count $cnt --repeat 3 --profile 2>&1 | tail -2 | tr '\n' ' ' | sed "s/^/$p /"; echo
  done
done
