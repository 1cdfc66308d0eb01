#!/bin/bash
# sweep-kernel variants: structured rows (two register budgets) vs generic gather
for v in lb0 lb6 generic; do
  lib=tune/$v.so; envs=""
  if [ $v = generic ]; then lib=tune/lb0.so; envs="WMC_SWEEP_GENERIC=1"; fi
  echo "== $v"
  env $envs WMC_LIB_PATH=$PWD/$lib python tools/kernel_probe.py --level 4 --count 1024 --steps 300 --profile --repeat 2 2>&1 | grep -E "profile|level" | tail -2
  env $envs WMC_LIB_PATH=$PWD/$lib python tools/kernel_probe.py --config2 --level 4 --count 2048 --steps 200 --profile --repeat 2 2>&1 | grep -E "profile|level" | tail -2
  env $envs WMC_LIB_PATH=$PWD/$lib python tools/kernel_probe.py --square 1024 8 --count 256 --steps 40 --profile --repeat 2 2>&1 | grep -E "profile|level" | tail -2
done
