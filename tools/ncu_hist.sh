# Launch list (duration + DRAM bytes) of the histogram / init / map kernels on a
# device-resident quantize: bash tools/ncu_hist.sh CONFIG DEBUG_FLAGS OUT.csv
CFG=${1:-cfg4}; FL=${2:-0}; OUT=${3:-gpurun_out/ncu_hist.csv}
timeout 300 python tools/run_once.py $CFG 2 256 $FL > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"k_part|k_first|k_bitmap|k_select|k_init|k_map|k_grid|k_hist|k_bins|k_rank" -c 60 --csv \
  python tools/run_once.py $CFG 2 256 $FL > $OUT 2>&1; echo ncu_$CFG_$FL=$?
