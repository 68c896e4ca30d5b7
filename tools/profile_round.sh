#!/bin/bash
# One round's profiling evidence (B200_PROFILING.md recipe): every ncu command
# follows the same command run plain with && and exit 0.
#   bash tools/profile_round.sh TAG     -> gpurun_out/prof_TAG/
OUT=gpurun_out/prof_${1:-r02}
mkdir -p $OUT
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-secondary"
timeout 600 $B > $OUT/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_cfg4.csv $B > $OUT/ncu_launches.log 2>&1; echo launches=$?
timeout 300 python tools/run_once.py cfg4 2 > $OUT/plain_once.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_wsm_loop -s 1 -c 1 \
    -o $OUT/loop_cfg4 -f python tools/run_once.py cfg4 2 > $OUT/ncu_loop.log 2>&1; echo loop=$?
timeout 300 python tools/run_once.py cfg4 2 > $OUT/plain_once2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:'k_hist_count|k_bins_compact|k_first|k_init_select|k_rank_pick|k_map_pixels|k_grid' -s 10 -c 12 \
    -o $OUT/hist_cfg4 -f python tools/run_once.py cfg4 2 > $OUT/ncu_hist.log 2>&1; echo hist=$?
timeout 300 python tools/run_once.py cfg2 2 > $OUT/plain_once3.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_wsm_loop|k_prep_small' -s 2 -c 2 \
    -o $OUT/small_cfg2 -f python tools/run_once.py cfg2 2 > $OUT/ncu_small.log 2>&1; echo small=$?
