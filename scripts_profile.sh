#!/bin/bash
# helper for gpurun: launch lists (cfg2, cfg4) + ncu --set full of the loop (cfg2, cfg4), of the
# fused small-image prep (cfg2) and of the HBM kernels (cfg4). Every ncu command follows the same
# command line run plain with && (B200_PROFILING.md).
OUT=gpurun_out/prof_${TAG:-r01}
mkdir -p $OUT
B2="python bench.py --config cfg2 --steps 2 --warmup 1 --no-cpu-baseline --no-secondary"
B4="python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu-baseline --no-secondary"
timeout 300 $B2 > $OUT/plain_cfg2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_cfg2.csv $B2 > $OUT/ncu_launches2.log 2>&1; echo launches2=$?
timeout 300 $B4 > $OUT/plain_cfg4.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_cfg4.csv $B4 > $OUT/ncu_launches4.log 2>&1; echo launches4=$?
timeout 300 $B2 > $OUT/plain_cfg2b.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_wsm_loop|k_prep_small|k_hist_count' \
    -s 6 -c 3 -o $OUT/small_cfg2 -f $B2 > $OUT/ncu_small_cfg2.log 2>&1; echo small=$?
timeout 300 $B4 > $OUT/plain_cfg4b.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on \
    -k regex:'k_wsm_loop|k_hist_count|k_bins_compact|k_bitmap_scan|k_rank_from|k_map_pixels|k_map_unique' -s 12 -c 10 \
    -o $OUT/large_cfg4 -f $B4 > $OUT/ncu_large_cfg4.log 2>&1; echo large=$?
