#!/bin/bash
B2="python bench.py --config cfg2 --steps 1 --warmup 1 --no-cpu-baseline --no-secondary"
timeout 300 $B2 > gpurun_out/plain2.log 2>&1 && timeout 600 ncu --set full --clock-control none -k regex:'k_occ_compact|k_rank_from|k_hist_count' -s 3 -c 3 -o gpurun_out/occ -f $B2 > gpurun_out/ncu_occ.log 2>&1; echo a=$?
