# sweep variants on config-1 levels 4 and 3 (per-kernel CUDA-event times):
# WMC_SWEEP_WIDE = 10 R + MINB of the 256-bit sweep, 0 = default sweep_rows_kernel
for lv in 4 3; do
for v in 23 14 15 33; do
  WMC_SWEEP_WIDE=$v timeout 120 python tools/kernel_probe.py --level $lv --count 1024 --repeat 3 --profile 2>&1 | tail -2 | tr '\n' ' ' | sed "s/^/wide=$v /"; echo
done
done

