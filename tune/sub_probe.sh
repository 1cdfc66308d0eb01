#!/bin/bash
for v in lb0 s2; do
  echo "== $v"
  WMC_LIB_PATH=$PWD/tune/$v.so python tools/kernel_probe.py --config2 --level 4 --count 2048 --steps 200 --profile --repeat 2 2>&1 | grep -E "profile|level" | tail -2
  WMC_LIB_PATH=$PWD/tune/$v.so python tools/kernel_probe.py --square 1024 8 --count 256 --steps 40 --profile --repeat 2 2>&1 | grep -E "profile|level" | tail -2
done
