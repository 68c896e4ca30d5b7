#!/bin/bash
# helper for gpurun: launch list (cfg2) + ncu --set full of the loop (cfg2) and of the HBM kernels (cfg4).
# Every ncu command follows the same command line run plain with && (B200_PROFILING.md).
OUT=gpurun_out/prof_${TAG:-r01}
mkdir -p $OUT
B2="python bench.py --config cfg2 --steps 2 --warmup 1 --no-cpu-baseline --no-secondary"
B4="python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu-baseline --no-secondary"
timeout 300 $B2 > $OUT/plain_cfg2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_cfg2.csv $B2 > $OUT/ncu_launches.log 2>&1; echo launches=$?
timeout 300 $B2 > $OUT/plain_cfg2b.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wsm_loop -s 2 -c 1 \
    -o $OUT/loop_cfg2 -f $B2 > $OUT/ncu_loop_cfg2.log 2>&1; echo loop=$?
timeout 300 $B4 > $OUT/plain_cfg4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'k_hist_count|k_hist_compact|k_bins_compact|k_map_pixels|k_map_unique|k_init_centers' -s 6 -c 6 \
    -o $OUT/hbm_cfg4 -f $B4 > $OUT/ncu_hbm_cfg4.log 2>&1; echo hbm=$?
