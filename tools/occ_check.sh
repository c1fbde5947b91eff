for lib in libgnb_base.so libgnb.so; do
  GNB_LIB=$lib timeout 300 ncu --metrics launch__occupancy_limit_shared_mem,launch__shared_mem_per_block_dynamic,launch__shared_mem_config_size,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,gpu__time_duration.sum \
    -k regex:predict_tma_kernel -s 3 -c 1 --csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-object-api 2>/dev/null | grep -E "launch__|sm__warps|gpu__time" | sed "s/^/$lib /"
done
