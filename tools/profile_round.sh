#!/bin/bash
# Reproduces the profiles/ captures (run on the GPU box from the repo root):
#   launch lists (kernel share of the step) of the default bench and of
#   config 2 at 2 % of N_l, then one `ncu --set full` capture of each hot
#   kernel from tools/kernel_probe.py.  Every ncu command runs only after the
#   same command exited 0 without ncu.  Output: gpurun_out/<tag>_*.
tag=${1:-r1}
out=gpurun_out
small="--steps 1 --warmup 3 --scale 0.02 --no-cpu-baseline --no-profile"
python bench.py $small > $out/${tag}_b1.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $out/${tag}_launches_c1.csv \
    python bench.py $small > /dev/null 2>&1
python bench.py --config 2 $small > $out/${tag}_b2.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $out/${tag}_launches_c2.csv \
    python bench.py --config 2 $small > /dev/null 2>&1
cap() {  # name regex skip probe-args...
  local name=$1 rx=$2 skip=$3; shift 3
  python tools/kernel_probe.py "$@" > /dev/null 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 -o $out/${tag}_prof_$name -f \
      python tools/kernel_probe.py "$@" > /dev/null 2>&1
}
cap fused lattice_solve 0 --level 0 --count 296 --repeat 1
cap fused2 lattice_solve 0 --level 2 --count 296 --repeat 1
cap lattice lattice_substep 20 --level 2 --count 1184 --repeat 1
cap sweep sweep_wide 5 --level 4 --count 1024 --steps 20 --repeat 1
cap gsub global_substep 10 --square 1024 8 --count 192 --steps 6 --repeat 1
cap tier tier_stage 30 --config2 --level 4 --count 2048 --steps 10 --repeat 1
ls -la $out | grep $tag
