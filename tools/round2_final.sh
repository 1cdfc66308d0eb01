#!/bin/bash
# Round-2 record run (GPU box, repo root): GPU tests, the bench lines of every
# config (both arms where the driver runs them), launch lists and the full
# captures of the config-3 kernels.  Every ncu command runs only after the
# same command exited 0 without ncu.  Output: gpurun_out/r2f_*.
out=gpurun_out
mkdir -p $out
(timeout 1500 python -m pytest tests -m gpu -x -q > $out/r2f_gputests.log 2>&1; echo "rc=$?" >> $out/r2f_gputests.log)
python bench.py > $out/r2f_bench_config1.json 2> $out/r2f_bench_config1.err
python bench.py --integrator lf > $out/r2f_bench_config1_lf.json 2> $out/r2f_bench_config1_lf.err
python bench.py --config 0 > $out/r2f_bench_config0.json 2> $out/r2f_bench_config0.err
python bench.py --config 2 > $out/r2f_bench_config2.json 2> $out/r2f_bench_config2.err
python bench.py --config 4 > $out/r2f_bench_config4.json 2> $out/r2f_bench_config4.err
python bench.py --config 4 --field element > $out/r2f_bench_config4_element.json 2> $out/r2f_bench_config4_element.err
python bench.py --impl reference > $out/r2f_ref_config1.json 2> $out/r2f_ref_config1.err
python bench.py --config 4 --impl reference > $out/r2f_ref_config4.json 2> $out/r2f_ref_config4.err
python bench.py --config 4 --field element --impl reference > $out/r2f_ref_config4_element.json 2> $out/r2f_ref_config4_element.err
small="--steps 1 --warmup 3 --scale 0.02 --no-cpu-baseline --no-profile"
python bench.py $small > $out/r2f_b1.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $out/r2f_launches_c1.csv \
    python bench.py $small > /dev/null 2>&1
probe="tools/tile_probe.py --steps 4 --count 256 --reps 1"
python $probe > $out/r2f_probe.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/r2f_launches_c3.csv python $probe > /dev/null 2>&1
for k in stream_step tile_step sweep_sm_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 1 -c 1 -o $out/r2f_prof_$k -f python $probe > /dev/null 2>&1
done
python tools/tile_probe.py --steps 8 --count 256 > $out/r2f_probe8.log 2>&1
ls -la $out | grep r2f
