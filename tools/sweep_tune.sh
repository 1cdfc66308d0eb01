set -x
for lv in 4 3; do
for v in 0 22 23 24 42 43 14; do
  WMC_SWEEP_AHEAD=$v timeout 120 python tools/kernel_probe.py --level $lv --count 1024 --repeat 3 --profile 2>&1 | tail -2
done
done
WMC_SWEEP_AHEAD=23 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
