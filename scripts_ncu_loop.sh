#!/bin/bash
# helper for gpurun: one ncu --set full capture of k_wsm_loop (cfg given by $1, default cfg2)
CFG=${1:-cfg2}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_wsm_loop -c 1 \
  -o gpurun_out/ncu_loop_${CFG} -f python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-secondary \
  > gpurun_out/ncu_loop_${CFG}.log 2>&1; echo ncu=$?
