# select_kernel, one launch, full set with source-level sampling (cfg2)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'^select_kernel' -c 1 \
  -o gpurun_out/select_full python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 1 > gpurun_out/ncu_select.log 2>&1
echo done
