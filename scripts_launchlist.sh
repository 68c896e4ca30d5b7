#!/bin/bash
B2="python bench.py --config cfg2 --steps 1 --warmup 1 --no-cpu-baseline --no-secondary"
B4="python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu-baseline --no-secondary"
timeout 300 $B2 > gpurun_out/plain2.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/ll2.csv $B2 > /dev/null 2>&1; echo a=$?
timeout 300 $B4 > gpurun_out/plain4.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/ll4.csv $B4 > /dev/null 2>&1; echo b=$?
