#!/bin/bash
for c in cfg1 cfg3; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/bench_$c.log 2>&1; echo $c=$?; done
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 1 > gpurun_out/bench_cfg5.log 2>&1; echo cfg5=$?
timeout 900 python bench.py --config cfg5 --impl reference --steps 1 --warmup 0 > gpurun_out/bench_cfg5_ref.log 2>&1; echo cfg5ref=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_cfg2_ref.log 2>&1; echo cfg2ref=$?
